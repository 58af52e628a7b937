"""Profiler: one training step of a PyTorch model -> a trace (the path's input).

The reference takes the trace as given (its JSONL format, trace.py:9-17,
is the profiler's output contract); the paper's profiler instruments
PyTorch's operator dispatch.  `TraceProfiler` is that
profiler on the B200: a TorchDispatchMode that records every aten operator
executed under it as one trace kernel, with its device time from CUDA events
around it, and every tensor storage it reads or writes:

  * an output aliasing an input's storage (views, in-place ops) is the same
    tensor; any other output is a new tensor (memory reuse by the caching
    allocator therefore never merges two tensors);
  * tensors marked with `mark_global` (parameters, gradients, optimizer
    states) are `global`, everything else `intermediate`;
  * a kernel's duration is ceil(device us), at least 1 (trace.py requires
    durations > 0).

`trace()` returns a validated Trace ready for `plan_migrations`.
"""

from __future__ import annotations

import math

import numpy as np
import torch
from torch.utils._python_dispatch import TorchDispatchMode
from torch.utils._pytree import tree_flatten

from .trace import KIND_GLOBAL, KIND_INTERMEDIATE, NONE_I64, Trace, TraceArrays, validate_arrays


def _storages(obj):
    out = []
    for x in tree_flatten(obj)[0]:
        if isinstance(x, torch.Tensor) and x.device.type == "cuda":
            st = x.untyped_storage()
            if st.nbytes() > 0:
                out.append((st.data_ptr(), st.nbytes()))
    return out


class TraceProfiler(TorchDispatchMode):
    def __init__(self, timed: bool = True):
        super().__init__()
        self.timed = timed
        self.names: list[str] = []
        self.events: list[tuple] = []
        self.accesses: list[list[int]] = []     # per op: tensor ids
        self.live: dict[int, int] = {}          # storage data_ptr -> tensor id
        self.size: list[int] = []               # tensor id -> bytes
        self.global_ids: set[int] = set()

    def _id_of(self, ptr: int, nbytes: int) -> int:
        tid = self.live.get(ptr)
        if tid is None:
            tid = len(self.size)
            self.size.append(nbytes)
            self.live[ptr] = tid
        else:
            self.size[tid] = max(self.size[tid], nbytes)
        return tid

    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        ins = _storages((args, kwargs))
        if self.timed:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        out = func(*args, **kwargs)
        if self.timed:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
        touched = [self._id_of(p, n) for p, n in ins]
        in_ptrs = {p for p, _ in ins}
        for p, n in _storages(out):
            if p in in_ptrs:                      # view / in-place: the same tensor
                touched.append(self._id_of(p, n))
            else:                                 # a fresh allocation: a new tensor
                tid = len(self.size)
                self.size.append(n)
                self.live[p] = tid
                touched.append(tid)
        self.names.append(str(func.overloadpacket.__name__))
        self.events.append((e0, e1) if self.timed else None)
        self.accesses.append(sorted(set(touched)))
        return out

    def mark_global(self, tensors) -> None:
        """Tag the current tensors behind `tensors` (parameters, grads,
        optimizer states) as global."""
        for t in tensors:
            if t is None or t.device.type != "cuda":
                continue
            st = t.untyped_storage()
            tid = self.live.get(st.data_ptr())
            if tid is not None:
                self.global_ids.add(tid)

    def trace(self, meta: dict | None = None) -> Trace:
        torch.cuda.synchronize()
        n = len(self.names)
        dur = np.ones(n, np.int64)
        if self.timed:
            for k, ev in enumerate(self.events):
                dur[k] = max(1, math.ceil(ev[0].elapsed_time(ev[1]) * 1000.0))
        per_tensor: list[list[int]] = [[] for _ in self.size]
        for k, ts in enumerate(self.accesses):
            for t in ts:
                per_tensor[t].append(k)
        keep = [t for t in range(len(self.size)) if per_tensor[t] and self.size[t] > 0]
        ptr = np.zeros(len(keep) + 1, np.int64)
        np.cumsum([len(per_tensor[t]) for t in keep], out=ptr[1:])
        acc = np.array([k for t in keep for k in per_tensor[t]], np.int64)
        names = sorted(set(self.names))
        code = {s: i for i, s in enumerate(names)}
        arrays = TraceArrays(
            duration_us=dur, kernel_index=np.arange(n, dtype=np.int64),
            kernel_name_code=np.array([code[s] for s in self.names], np.int32), name_table=names,
            kernel_stage=np.full(n, NONE_I64, np.int64), kernel_layer=np.full(n, NONE_I64, np.int64),
            tensor_id=np.array(keep, np.int64), size_bytes=np.array([self.size[t] for t in keep], np.int64),
            kind=np.array([KIND_GLOBAL if t in self.global_ids else KIND_INTERMEDIATE for t in keep], np.int8),
            tensor_layer=np.full(len(keep), NONE_I64, np.int64), access_ptr=ptr, accesses=acc)
        rep = validate_arrays(arrays)
        if not rep.ok:
            raise ValueError("profiled trace violates the trace model: " + "; ".join(rep.violations[:5]))
        return Trace.from_arrays(arrays, meta or {"generator": "TraceProfiler"})


def profile_step(step_fn, global_tensors_fn=None, meta: dict | None = None) -> Trace:
    """Run `step_fn()` once under the profiler; `global_tensors_fn()` (called
    after the step) returns the tensors to mark global."""
    prof = TraceProfiler()
    with prof:
        step_fn()
    if global_tensors_fn is not None:
        prof.mark_global(global_tensors_fn())
    return prof.trace(meta)
