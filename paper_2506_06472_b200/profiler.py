"""Profiler: one training step of a PyTorch model -> a trace (the path's input).

The reference takes the trace as given (its JSONL format, trace.py:9-17,
is the profiler's output contract); the paper's profiler instruments
PyTorch's operator dispatch.  `TraceProfiler` is that
profiler on the B200: a TorchDispatchMode that records every aten operator
executed under it as one trace kernel, with its device time from CUDA events
around it, and every tensor storage it reads or writes.

Tensor identity (`StorageTracker`, shared with the migration engine's
executor so both number the tensors of a step identically):

  * a tensor is a storage (its StorageImpl, which survives the engine
    freeing and re-allocating its bytes); an output aliasing an input's
    storage (views, in-place ops) is the same tensor, any other output is a
    new tensor (allocator reuse never merges two tensors);
  * `globals` (name -> tensor: weights, optimizer states, persistent buffers)
    are registered before the step in name order, so they take ids
    0..G-1 independent of operator order, and are `global`; everything else
    is `intermediate`;
  * communication tensors (`comm` names, e.g. NCCL all-reduce buckets) are
    marked active on every kernel of the collective that touches them like
    any other input, so the planner never offloads them while a collective
    uses them;
  * a kernel's duration is ceil(device us), at least 1 (trace.py requires
    durations > 0).

`trace()` returns a validated Trace ready for `plan_migrations`.
"""

from __future__ import annotations

import math

import numpy as np
import torch
from torch.utils._python_dispatch import TorchDispatchMode

from .trace import KIND_GLOBAL, KIND_INTERMEDIATE, NONE_I64, Trace, TraceArrays, validate_arrays


def cuda_tensors(obj, out):
    """Append every CUDA tensor inside (nested lists/tuples/dicts of) obj."""
    if isinstance(obj, torch.Tensor):
        if obj.is_cuda:
            out.append(obj)
    elif isinstance(obj, (list, tuple)):
        for x in obj:
            cuda_tensors(x, out)
    elif isinstance(obj, dict):
        for x in obj.values():
            cuda_tensors(x, out)
    return out


class StorageTracker:
    """Tensor ids of a step: one per storage (see module docstring)."""

    def __init__(self, globals_: dict | None = None):
        self.live: dict[int, int] = {}           # StorageImpl address -> tensor id
        self.nbytes: list[int] = []              # tensor id -> storage bytes
        self.names: dict[int, str] = {}          # global tensor id -> name
        for name in sorted(globals_ or {}):
            t = globals_[name]
            st = t.untyped_storage()
            key = st._cdata
            if key in self.live:                 # two names for one storage
                continue
            tid = self._new(key, st.nbytes())
            self.names[tid] = name

    def _new(self, key: int, nbytes: int) -> int:
        tid = len(self.nbytes)
        self.nbytes.append(nbytes)
        self.live[key] = tid
        return tid

    def inputs(self, tensors):
        """(ids, keys) of the operator's input storages (new ids on first sight)."""
        ids, keys = [], set()
        for t in tensors:
            st = t.untyped_storage()
            nb = st.nbytes()
            key = st._cdata
            tid = self.live.get(key)
            if tid is None:
                if nb == 0:
                    continue
                tid = self._new(key, nb)
            elif nb > self.nbytes[tid]:
                self.nbytes[tid] = nb
            keys.add(key)
            ids.append(tid)
        return ids, keys

    def outputs(self, tensors, in_keys):
        """ids of the operator's output storages; fresh ones are new tensors.
        Returns (all ids, [(new id, tensor)])."""
        ids, new = [], []
        for t in tensors:
            st = t.untyped_storage()
            key = st._cdata
            if key in in_keys:
                ids.append(self.live[key])
                continue
            nb = st.nbytes()
            if nb == 0:
                continue
            tid = self._new(key, nb)
            ids.append(tid)
            new.append((tid, t))
            in_keys.add(key)
        return ids, new


class TraceProfiler(TorchDispatchMode):
    def __init__(self, timed: bool = True, globals_: dict | None = None):
        super().__init__()
        self.timed = timed
        self.tracker = StorageTracker(globals_)
        self.global_ids: set[int] = set(self.tracker.names)
        self.names: list[str] = []
        self.events: list = []
        self.accesses: list[list[int]] = []     # per op: tensor ids

    @property
    def size(self) -> list[int]:
        return self.tracker.nbytes

    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        ins, in_keys = self.tracker.inputs(cuda_tensors((args, kwargs), []))
        if self.timed:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        out = func(*args, **kwargs)
        if self.timed:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
        outs, _ = self.tracker.outputs(cuda_tensors(out, []), in_keys)
        self.names.append(str(func.overloadpacket.__name__))
        self.events.append((e0, e1) if self.timed else None)
        self.accesses.append(sorted(set(ins + outs)))
        return out

    def mark_global(self, tensors) -> None:
        """Tag the current tensors behind `tensors` (parameters, grads,
        optimizer states) as global (for steps profiled without `globals_`)."""
        for t in tensors:
            if t is None or not t.is_cuda:
                continue
            tid = self.tracker.live.get(t.untyped_storage()._cdata)
            if tid is not None:
                self.global_ids.add(tid)

    def trace(self, meta: dict | None = None) -> Trace:
        torch.cuda.synchronize()
        n = len(self.names)
        dur = np.ones(n, np.int64)
        if self.timed:
            for k, ev in enumerate(self.events):
                dur[k] = max(1, math.ceil(ev[0].elapsed_time(ev[1]) * 1000.0))
        size = self.tracker.nbytes
        per_tensor: list[list[int]] = [[] for _ in size]
        for k, ts in enumerate(self.accesses):
            for t in ts:
                per_tensor[t].append(k)
        keep = [t for t in range(len(size)) if per_tensor[t] and size[t] > 0]
        ptr = np.zeros(len(keep) + 1, np.int64)
        np.cumsum([len(per_tensor[t]) for t in keep], out=ptr[1:])
        acc = np.array([k for t in keep for k in per_tensor[t]], np.int64)
        names = sorted(set(self.names))
        code = {s: i for i, s in enumerate(names)}
        arrays = TraceArrays(
            duration_us=dur, kernel_index=np.arange(n, dtype=np.int64),
            kernel_name_code=np.array([code[s] for s in self.names], np.int32), name_table=names,
            kernel_stage=np.full(n, NONE_I64, np.int64), kernel_layer=np.full(n, NONE_I64, np.int64),
            tensor_id=np.array(keep, np.int64), size_bytes=np.array([size[t] for t in keep], np.int64),
            kind=np.array([KIND_GLOBAL if t in self.global_ids else KIND_INTERMEDIATE for t in keep], np.int8),
            tensor_layer=np.full(len(keep), NONE_I64, np.int64), access_ptr=ptr, accesses=acc)
        rep = validate_arrays(arrays)
        if not rep.ok:
            raise ValueError("profiled trace violates the trace model: " + "; ".join(rep.violations[:5]))
        m = dict(meta or {"generator": "TraceProfiler"})
        m.setdefault("globals", {str(t): self.tracker.names[t] for t in sorted(self.tracker.names)})
        return Trace.from_arrays(arrays, m)


def profile_step(step_fn, global_tensors_fn=None, meta: dict | None = None, globals_: dict | None = None) -> Trace:
    """Run `step_fn()` once under the profiler.  `globals_` (name -> tensor)
    registers the persistent tensors up front (stable ids, shared with the
    engine); `global_tensors_fn()` (called after the step) is the older form
    that only tags them."""
    prof = TraceProfiler(globals_=globals_)
    with prof:
        step_fn()
    if global_tensors_fn is not None:
        prof.mark_global(global_tensors_fn())
    return prof.trace(meta)
