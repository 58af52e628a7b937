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
