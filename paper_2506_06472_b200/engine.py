"""Migration engine on the B200 — executes a plan for real.

`replay(trace, plan, capacity, rates)` runs one iteration of a trace under
a plan through libtio's executor (csrc/engine.cu): the engine scheduler
(csrc/engine_sched.cu, the reference engine semantics of simulator.py:178-528)
decides every transfer, and the executor carries it out with real copies
between stream-ordered device buffers and 4 KB-aligned pinned host extents on
one side stream per channel, gated by CUDA events, while a placeholder kernel
per trace kernel occupies the compute stream for its profiled duration.
Every prefetched tensor can be checked byte for byte (`verify=True`).

`pack` / `unpack` are the engine's TMA bulk copy kernels (gather tensors into
4 KB-aligned staging extents and back).  `measure_link` measures the pinned
host link the plan's rates should use.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .bandwidth import ChannelRates
from .planner import _rates_struct
from .simulator import _entries_of, entries_array
from .trace import Trace


class EngineConfigC(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_int64), ("rates", _native.Rates), ("time_scale", ctypes.c_double),
                ("verify", ctypes.c_int), ("measure_ideal", ctypes.c_int)]


class EngineStatsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("model_total_us", "model_ideal_us", "model_stall_us",
                                             "model_peak_resident", "emergency_offloads")] + [
        ("replay_ms", ctypes.c_double), ("ideal_ms", ctypes.c_double)] + [
        (n, ctypes.c_int64) for n in ("offload_bytes", "prefetch_bytes", "n_offloads", "n_prefetches")] + [
        ("offload_busy_ms", ctypes.c_double), ("prefetch_busy_ms", ctypes.c_double)] + [
        (n, ctypes.c_int64) for n in ("peak_device_bytes", "host_bytes", "verified_bytes", "verify_mismatches")]


@dataclass
class ReplayReport:
    model_total_us: int          # engine model (== simulate().total_time)
    model_ideal_us: int
    model_stall_us: int
    model_peak_resident: int
    emergency_offloads: int
    replay_ms: float             # measured device time of the iteration with migrations
    ideal_ms: float              # measured device time of the same kernels without migrations
    offload_bytes: int
    prefetch_bytes: int
    n_offloads: int
    n_prefetches: int
    offload_busy_ms: float
    prefetch_busy_ms: float
    peak_device_bytes: int
    host_bytes: int
    verified_bytes: int
    verify_mismatches: int

    @property
    def step_vs_ideal(self) -> float:
        return self.replay_ms / self.ideal_ms if self.ideal_ms else float("nan")

    @property
    def offload_gbs(self) -> float:
        return self.offload_bytes / (self.offload_busy_ms * 1e6) if self.offload_busy_ms else 0.0

    @property
    def prefetch_gbs(self) -> float:
        return self.prefetch_bytes / (self.prefetch_busy_ms * 1e6) if self.prefetch_busy_ms else 0.0


def replay(trace: Trace, plan, capacity: int, rates: ChannelRates, time_scale: float = 1.0,
           verify: bool = True, measure_ideal: bool = True, stream: int = 0) -> ReplayReport:
    _native.require_device()
    lib = _native.load()
    cols = _native.HostColumns(trace.arrays())
    desc = cols.desc()
    ents = entries_array(_entries_of(plan))
    cfg = EngineConfigC(capacity, _rates_struct(rates), time_scale, 1 if verify else 0, 1 if measure_ideal else 0)
    st = EngineStatsC()
    rc = lib.tio_engine_replay(ctypes.byref(desc), _native._ptr(ents), ctypes.c_int64(ents.shape[0]),
                               ctypes.byref(cfg), ctypes.c_void_p(stream), ctypes.byref(st))
    if rc == _native.TIO_ERR_SIMULATION:
        from .simulator import SimulationError
        raise SimulationError(_native.last_error())
    _native.check(rc)
    return ReplayReport(**{f: getattr(st, f) for f, _ in EngineStatsC._fields_})


def check_program(trace: Trace, plan, capacity: int, rates: ChannelRates, steps: int = 3) -> dict:
    """Walk the online engine's program for `steps` consecutive steps on the
    host (tio_engine_check_program: no device, fake addresses) — every
    offload finds its tensor resident, every prefetch finds it gone, every
    kernel finds its tensors on the GPU.  Returns the engine info."""
    lib = _native.load()
    cols = _native.HostColumns(trace.arrays())
    desc = cols.desc()
    ents = entries_array(_entries_of(plan))
    cfg = EngineConfigC(capacity, _rates_struct(rates), 1.0, 0, 0)
    info = EngineInfoC()
    rc = lib.tio_engine_check_program(ctypes.byref(desc), _native._ptr(ents), ctypes.c_int64(ents.shape[0]),
                                      ctypes.byref(cfg), ctypes.c_int64(steps), ctypes.byref(info))
    if rc == _native.TIO_ERR_SIMULATION:
        from .simulator import SimulationError
        raise SimulationError(_native.last_error())
    _native.check(rc)
    return {f: getattr(info, f) for f, _ in EngineInfoC._fields_}


def checksums(tensors) -> list[int]:
    """libtio's verification checksum of each CUDA tensor's storage bytes
    (one device pass each, on the current stream)."""
    import torch
    lib = _native.load()
    out = torch.zeros(max(1, len(tensors)), dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for i, t in enumerate(tensors):
        st = t.untyped_storage()
        _native.check(lib.tio_checksum(ctypes.c_void_p(st.data_ptr()), ctypes.c_int64(st.nbytes()),
                                       ctypes.c_void_p(out.data_ptr() + 8 * i), ctypes.c_void_p(s)))
    return [v & (2**64 - 1) for v in out.tolist()[:len(tensors)]]


def _scratch(n: int):
    import torch
    return torch.empty(64 * n + 64, dtype=torch.uint8, device="cuda")


def pack(tensors, staging, stream: int = 0) -> list[int]:
    """Copy each CUDA tensor's bytes into a 4 KB-aligned extent of `staging`
    (a uint8 CUDA tensor); returns the extent offsets."""
    lib = _native.load()
    n = len(tensors)
    src = (ctypes.c_void_p * max(1, n))(*[t.data_ptr() for t in tensors])
    nbytes = np.array([t.numel() * t.element_size() for t in tensors], np.int64)
    offs = np.zeros(max(1, n), np.int64)
    need = int(sum((int(b) + 4095) // 4096 * 4096 for b in nbytes))
    if staging.numel() < need:
        raise ValueError(f"staging buffer too small: {staging.numel()} < {need}")
    sc = _scratch(n)
    _native.check(lib.tio_pack(src, _native._ptr(nbytes), ctypes.c_int64(n), ctypes.c_void_p(staging.data_ptr()),
                               _native._ptr(offs), ctypes.c_void_p(sc.data_ptr()), ctypes.c_size_t(sc.numel()),
                               ctypes.c_void_p(stream)))
    return offs[:n].tolist()


def unpack(staging, offsets, tensors, stream: int = 0) -> None:
    lib = _native.load()
    n = len(tensors)
    dst = (ctypes.c_void_p * max(1, n))(*[t.data_ptr() for t in tensors])
    nbytes = np.array([t.numel() * t.element_size() for t in tensors], np.int64)
    offs = np.array(list(offsets) or [0], np.int64)
    sc = _scratch(n)
    _native.check(lib.tio_unpack(ctypes.c_void_p(staging.data_ptr()), _native._ptr(offs), dst,
                                 _native._ptr(nbytes), ctypes.c_int64(n), ctypes.c_void_p(sc.data_ptr()),
                                 ctypes.c_size_t(sc.numel()), ctypes.c_void_p(stream)))


def measure_link(nbytes: int = 1 << 30, reps: int = 5) -> dict:
    """Pinned host <-> device copy bandwidth (GB/s): H2D and D2H alone, and
    both at once on two streams (SURVEY §8d link measurement)."""
    import torch
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dev2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    host2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = float("inf")
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    def h2d():
        dev.copy_(host, non_blocking=True)

    def d2h():
        host.copy_(dev, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            dev.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2):
            host2.copy_(dev2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    gb = nbytes / 1e9
    return {"bytes": nbytes, "h2d_gbs": gb / (t_h2d / 1e3), "d2h_gbs": gb / (t_d2h / 1e3),
            "bidir_gbs_each": gb / (t_both / 1e3), "method": "pinned cudaMemcpyAsync, best of %d" % reps}


# ----------------------------------------------------------------------------
# Online engine: the plan executed on a REAL training step
# ----------------------------------------------------------------------------

_ALLOC_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                             ctypes.POINTER(ctypes.c_void_p))
_FREE_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)


class EngineInfoC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "num_kernels", "num_tensors", "num_transfers", "host_bytes", "model_total_us", "model_ideal_us",
        "model_stall_us", "model_peak_resident", "emergency_offloads", "model_offload_bytes",
        "model_prefetch_bytes", "model_offloads", "model_prefetches")]


class OnlineStatsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("steps", "offload_bytes", "prefetch_bytes", "n_offloads",
                                             "n_prefetches")] + [
        ("last_offload_busy_ms", ctypes.c_double), ("last_prefetch_busy_ms", ctypes.c_double),
        ("last_offload_bytes", ctypes.c_int64), ("last_prefetch_bytes", ctypes.c_int64),
        ("verify", ctypes.c_int64), ("verify_mismatches", ctypes.c_int64),
        ("reconcile_transfers", ctypes.c_int64), ("reconcile_bytes", ctypes.c_int64)]


class StepDivergence(RuntimeError):
    """The executed step does not match the profiled trace (different
    operators or tensors): the plan cannot be applied to it."""


class OffloadMode:
    """Runs a training step under a migration plan: a TorchDispatchMode over
    libtio's online engine (tio_engine_*, csrc/engine_online.cu).

        mode = OffloadMode(trace, plan, capacity, rates, globals_)
        for _ in range(steps):
            with mode.step():
                loss = step_fn()

    Every aten operator of the step is kernel k of the profiled trace: the
    mode numbers storages with the profiler's StorageTracker (same ids),
    checks that operator k touches exactly the trace's tensors of kernel k
    (`StepDivergence` otherwise), and calls tio_engine_before_kernel(k) /
    tio_engine_after_kernel(k) around it.  The engine moves tensors on its
    channel streams and asks this object to free (record_stream on the channel
    + storage resize to 0) and re-allocate (storage resize on the compute
    stream) their storages; the tensors' Python objects, views and autograd
    references stay valid throughout.
    """

    def __init__(self, trace: Trace, plan, capacity: int, rates: ChannelRates, globals_: dict,
                 verify: bool = False, check: bool = True, stream=None):
        import torch
        from .profiler import StorageTracker
        _native.require_device()
        self._torch = torch
        self.lib = _native.load()
        self.trace = trace
        self.globals_ = globals_
        self.check = check
        a = trace.arrays()
        self.N, self.T = a.num_kernels, a.num_tensors
        cols = _native.HostColumns(a)
        desc = cols.desc()
        ents = entries_array(_entries_of(plan))
        cfg = EngineConfigC(capacity, _rates_struct(rates), 1.0, 1 if verify else 0, 0)
        self.stream = stream or torch.cuda.current_stream()
        self._alloc_cb = _ALLOC_CB(self._on_alloc)
        self._free_cb = _FREE_CB(self._on_free)
        self.h = ctypes.c_void_p()
        rc = self.lib.tio_engine_create(ctypes.byref(desc), _native._ptr(ents), ctypes.c_int64(ents.shape[0]),
                                        ctypes.byref(cfg), ctypes.c_void_p(self.stream.cuda_stream),
                                        self._alloc_cb, self._free_cb, None, ctypes.byref(self.h))
        if rc == _native.TIO_ERR_SIMULATION:
            from .simulator import SimulationError
            raise SimulationError(_native.last_error())
        _native.check(rc)
        info = EngineInfoC()
        movable = np.zeros(max(1, self.T), np.uint8)
        _native.check(self.lib.tio_engine_info(self.h, ctypes.byref(info), _native._ptr(movable)))
        self.info = {f: getattr(info, f) for f, _ in EngineInfoC._fields_}
        self.movable = movable[:self.T].astype(bool)
        # tensor id -> trace position; per kernel: sorted positions it touches
        self.pos_of = {int(t): i for i, t in enumerate(a.tensor_id.tolist())}
        ptr, acc = a.access_ptr, a.accesses
        per_k = [[] for _ in range(self.N)]
        for t in range(self.T):
            for j in range(int(ptr[t]), int(ptr[t + 1])):
                per_k[int(acc[j])].append(t)
        self.k_tensors = [tuple(sorted(x)) for x in per_k]
        self.last_acc = np.array([int(acc[ptr[t + 1] - 1]) for t in range(self.T)], np.int64)
        self.is_global = a.kind == 1
        self.tracker_cls = StorageTracker
        self.refs: dict[int, object] = {}        # position -> a tensor on the storage (movable only)
        self.nbytes: dict[int, int] = {}
        self._streams: dict[int, object] = {}
        self.steps_done = 0
        self._bind_globals()

    # -- host side of the engine's memory callbacks ---------------------------
    def _on_free(self, user, pos, stream):
        try:
            stream = stream or 0                 # ctypes passes NULL (the legacy stream) as None
            t = self.refs[pos]
            s = self._streams.get(stream)
            if s is None:
                s = self._streams[stream] = self._torch.cuda.ExternalStream(stream)
            if stream != self.stream.cuda_stream:
                t.record_stream(s)
            t.untyped_storage().resize_(0)
            return 0
        except Exception as exc:  # pragma: no cover - reported through the engine
            self._cb_error = exc
            return 1

    def _on_alloc(self, user, pos, nbytes, out):
        try:
            t = self.refs[pos]
            st = t.untyped_storage()
            st.resize_(self.nbytes.get(pos, nbytes))
            out[0] = st.data_ptr()
            return 0
        except Exception as exc:  # pragma: no cover
            self._cb_error = exc
            return 1

    def _bind_globals(self):
        tr = self.tracker_cls(self.globals_)
        pos, ptrs = [], []
        for tid, name in tr.names.items():
            p = self.pos_of.get(tid)
            if p is None or not self.movable[p]:
                continue
            t = self.globals_[name]
            self.refs[p] = t
            self.nbytes[p] = t.untyped_storage().nbytes()
            pos.append(p)
            ptrs.append(t.untyped_storage().data_ptr())
        self._bind(pos, ptrs)

    def _bind(self, pos, ptrs):
        if not pos:
            return
        pa = np.array(pos, np.int64)
        va = (ctypes.c_void_p * len(ptrs))(*ptrs)
        _native.check(self.lib.tio_engine_bind(self.h, ctypes.c_int64(len(pos)), _native._ptr(pa), va))

    def _call(self, rc):
        if rc != 0:
            err = getattr(self, "_cb_error", None)
            msg = _native.last_error()
            if "diverges" in msg:
                raise StepDivergence(msg)
            if err is not None:
                raise RuntimeError(f"{msg} ({type(err).__name__}: {err})") from err
            _native.check(rc)

    # -- one step --------------------------------------------------------------
    def step(self, done_stream=None):
        """Context manager running one step under the engine; `done_stream`
        (optional) is made to wait for every transfer of the step."""
        self._cb_error = None
        return _EngineStep(self, done_stream)

    def set_verify(self, on: bool) -> None:
        _native.check(self.lib.tio_engine_set_verify(self.h, ctypes.c_int(1 if on else 0)))

    def stats(self) -> dict:
        st = OnlineStatsC()
        _native.check(self.lib.tio_engine_stats_get(self.h, ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in OnlineStatsC._fields_}

    def restore(self) -> None:
        """Bring every global tensor whose latest copy is off the GPU back
        (between steps; e.g. before a checkpoint or leaving the engine)."""
        self._cb_error = None
        self._call(self.lib.tio_engine_restore(self.h))

    def close(self, restore: bool = True):
        """Destroy the engine; by default first restore every global tensor to
        the device so the model is whole again."""
        if self.h:
            if restore:
                self.restore()
            self.lib.tio_engine_destroy(self.h)
            self.h = ctypes.c_void_p()
        self.refs.clear()
        self.globals_ = {}                     # the model's tensors are no longer the engine's

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _EngineStep:
    """The TorchDispatchMode of one step (see OffloadMode)."""

    def __init__(self, eng: OffloadMode, done_stream=None):
        from torch.utils._python_dispatch import TorchDispatchMode
        from .profiler import cuda_tensors
        self.eng = eng
        self.done_stream = done_stream
        outer = self

        class _Mode(TorchDispatchMode):
            def __torch_dispatch__(self, func, types, args=(), kwargs=None):
                return outer._op(func, args, kwargs or {}, cuda_tensors)
        self.mode = _Mode()

    def __enter__(self):
        e = self.eng
        self.tracker = e.tracker_cls(e.globals_)
        self.k = 0
        e._call(e.lib.tio_engine_step_begin(e.h))
        self.mode.__enter__()
        return self

    def __exit__(self, et, ev, tb):
        self.mode.__exit__(et, ev, tb)
        e = self.eng
        if et is not None:
            e.lib.tio_engine_step_abort(e.h)
            for p in [p for p in e.refs if not e.is_global[p]]:
                del e.refs[p]
            return False
        e._call(e.lib.tio_engine_step_end(e.h, ctypes.c_void_p(
            self.done_stream.cuda_stream if self.done_stream is not None else 0)))
        # drop what the step held: intermediates are the framework's again
        for p in [p for p in e.refs if not e.is_global[p]]:
            del e.refs[p]
        e.steps_done += 1
        return False

    def _op(self, func, args, kwargs, cuda_tensors):
        e = self.eng
        k = self.k
        if k >= e.N:
            raise StepDivergence(f"operator {k} ({func}) beyond the profiled trace's {e.N} kernels")
        tr = self.tracker
        ins_t = cuda_tensors((args, kwargs), [])
        ins, in_keys = tr.inputs(ins_t)
        pos_of = e.pos_of
        e._call(e.lib.tio_engine_before_kernel(e.h, ctypes.c_int64(k)))
        out = func(*args, **kwargs)
        outs_t = cuda_tensors(out, [])
        outs, new = tr.outputs(outs_t, in_keys)
        touched = sorted({pos_of[i] for i in ins + outs if i in pos_of})
        if e.check and tuple(touched) != e.k_tensors[k]:
            raise StepDivergence(f"operator {k} ({func}) touches tensors {touched[:8]} but the profiled kernel "
                                 f"touched {list(e.k_tensors[k])[:8]}")
        # keep a reference to every movable tensor until its last access; bind
        # the device address of movable tensors the engine has not seen yet
        movable, refs = e.movable, e.refs
        new_pos, new_ptr = [], []
        for t in ins_t:
            p = pos_of.get(tr.live.get(t.untyped_storage()._cdata, -1))
            if p is not None and movable[p] and p not in refs:
                refs[p] = t
                e.nbytes[p] = t.untyped_storage().nbytes()
                new_pos.append(p)
                new_ptr.append(t.untyped_storage().data_ptr())
        for tid, t in new:
            p = pos_of.get(tid)
            if p is not None and movable[p]:
                refs[p] = t
                e.nbytes[p] = t.untyped_storage().nbytes()
                new_pos.append(p)
                new_ptr.append(t.untyped_storage().data_ptr())
        if new_pos:
            pa = np.array(new_pos, np.int64)
            va = (ctypes.c_void_p * len(new_ptr))(*new_ptr)
            e._call(e.lib.tio_engine_after_kernel(e.h, ctypes.c_int64(k), ctypes.c_int64(len(new_pos)),
                                                  _native._ptr(pa), va))
        else:
            e._call(e.lib.tio_engine_after_kernel(e.h, ctypes.c_int64(k), ctypes.c_int64(0), None, None))
        for p in e.k_tensors[k]:
            if not e.is_global[p] and e.last_acc[p] == k:
                refs.pop(p, None)
        self.k = k + 1
        return out
