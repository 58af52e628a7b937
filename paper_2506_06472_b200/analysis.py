"""Lifetime analysis — reference `offloader/analysis.py` API on the B200 path.

`compute_inactive_periods` (analysis.py:58-83), `compute_memory_timeline`
(:97-108) and `per_kernel_active_bytes` (:111-117) run as one cooperative
sm_100a kernel in libtio (csrc/lifetime.cu); this module only converts the
device results into the reference's dataclasses.  `lifetime_arrays` returns
the raw columns without building per-period Python objects (what large-trace
callers should use).

`period_interior_durations` (every period's interior duration, the
reference's only analogue of a "longest inactive gap") runs on the device;
`period_interior_duration` (one period), `characterize` and the CSV helpers
are the reference's Fig-1/Fig-2 reporting on the host over
the device-computed columns.
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass

import numpy as np

from . import _native
from .trace import Trace

DEFAULT_SIZE_BUCKETS = (10_000_000, 100_000_000, 1_000_000_000)
DEFAULT_DURATION_BUCKETS = (1_000, 10_000, 100_000)


@dataclass(frozen=True)
class InactivePeriod:
    tensor_id: int
    size_bytes: int
    start_kernel: int
    end_kernel: int
    wraps: bool = False


@dataclass
class MemoryTimeline:
    per_kernel_bytes: list[int]

    def peak(self) -> int:
        return max(self.per_kernel_bytes, default=0)

    def copy(self) -> "MemoryTimeline":
        return MemoryTimeline(list(self.per_kernel_bytes))


@dataclass
class LifetimeArrays:
    """Device lifetime products copied to host columns."""

    starts: np.ndarray          # int64[N+1]
    timeline: np.ndarray        # int64[N]
    active: np.ndarray          # int64[N]
    period_tensor: np.ndarray   # int64[P] tensor position
    period_start: np.ndarray    # int32[P]
    period_end: np.ndarray      # int32[P]
    period_wraps: np.ndarray    # int8[P]
    iteration: int


def _device_trace(trace: Trace) -> "_native.DeviceTrace":
    arrays = trace.arrays()          # drops every cached device product if the records changed
    dt = trace.device_cache.get("trace")
    if dt is None:
        dt = _native.DeviceTrace(arrays)
        trace.device_cache["trace"] = dt
    return dt


def lifetime_arrays(trace: Trace) -> LifetimeArrays:
    trace.arrays()                   # staleness check first (see Trace.arrays)
    cached = trace.device_cache.get("lifetime")
    if cached is None:
        r = _device_trace(trace).lifetime()
        cached = LifetimeArrays(r["starts"], r["timeline"], r["active"], r["period_tensor"],
                                r["period_start"], r["period_end"], r["period_wraps"], r["iteration"])
        trace.device_cache["lifetime"] = cached
    return cached


def compute_inactive_periods(trace: Trace) -> list[InactivePeriod]:
    """All inactive periods in (tensor order, period start) order."""
    if trace.num_tensors == 0:
        return []
    la = lifetime_arrays(trace)
    a = trace.arrays()
    tids = a.tensor_id[la.period_tensor].tolist()
    sizes = a.size_bytes[la.period_tensor].tolist()
    return [InactivePeriod(t, s, st, en, bool(w)) for t, s, st, en, w in
            zip(tids, sizes, la.period_start.tolist(), la.period_end.tolist(), la.period_wraps.tolist())]


def compute_memory_timeline(trace: Trace) -> MemoryTimeline:
    if trace.num_kernels == 0:
        return MemoryTimeline([])
    return MemoryTimeline(lifetime_arrays(trace).timeline.tolist())


def per_kernel_active_bytes(trace: Trace) -> list[int]:
    if trace.num_kernels == 0:
        return []
    return lifetime_arrays(trace).active.tolist()


def period_interior_duration(period: InactivePeriod, trace: Trace) -> int:
    """Sum of kernel durations strictly inside the period (analysis.py:86-94)."""
    a = trace.arrays()
    d = a.duration_us
    if not period.wraps:
        return int(d[period.start_kernel:period.end_kernel + 1].sum())
    pos = int(np.flatnonzero(a.tensor_id == period.tensor_id)[0])
    acc = a.accesses[a.access_ptr[pos]:a.access_ptr[pos + 1]]
    return int(d[int(acc[-1]) + 1:].sum() + d[:int(acc[0])].sum())


def period_interior_durations(trace: Trace) -> np.ndarray:
    """period_interior_duration (analysis.py:86-94) of every inactive period,
    in compute_inactive_periods order, computed on the device from the
    kernel start times (libtio `tio_period_interior`)."""
    import ctypes
    dt = _device_trace(trace)
    P = lifetime_arrays(trace).period_tensor.shape[0]
    out = np.zeros(P, np.int64)
    if P:
        _native.check(dt._lib.tio_period_interior(dt.handle, dt.stream, out.ctypes.data_as(ctypes.c_void_p)))
    return out


# --- characterization (reporting; reference analysis.py:120-188) -------------

def bucket_label(bounds: tuple[int, ...], value: int) -> str:
    if value < bounds[0]:
        return f"<{bounds[0]}"
    for lo, hi in zip(bounds, bounds[1:]):
        if lo <= value < hi:
            return f"[{lo},{hi})"
    return f">={bounds[-1]}"


@dataclass
class CharacterizationReport:
    capacity_bytes: int
    active_bytes: list[int]
    active_fraction: list[float]
    histogram: dict[tuple[str, str], int]
    mean_active_fraction: float
    max_active_fraction: float
    size_buckets: tuple[int, ...] = DEFAULT_SIZE_BUCKETS
    duration_buckets: tuple[int, ...] = DEFAULT_DURATION_BUCKETS
    total_periods: int = 0


def characterize(trace: Trace, capacity: int,
                 size_buckets: tuple[int, ...] = DEFAULT_SIZE_BUCKETS,
                 duration_buckets: tuple[int, ...] = DEFAULT_DURATION_BUCKETS) -> CharacterizationReport:
    if capacity <= 0:
        raise ValueError("capacity must be > 0")
    active = per_kernel_active_bytes(trace)
    fractions = [b / capacity for b in active]
    histogram: dict[tuple[str, str], int] = {}
    total = 0
    if trace.num_tensors:
        la = lifetime_arrays(trace)
        a = trace.arrays()
        tp = la.period_tensor
        interior = period_interior_durations(trace)
        sizes = a.size_bytes[tp]
        for s, dur in zip(sizes.tolist(), interior.tolist()):
            cell = (bucket_label(size_buckets, s), bucket_label(duration_buckets, dur))
            histogram[cell] = histogram.get(cell, 0) + 1
        total = int(tp.shape[0])
    return CharacterizationReport(
        capacity_bytes=capacity, active_bytes=active, active_fraction=fractions,
        histogram=histogram,
        mean_active_fraction=sum(fractions) / len(fractions) if fractions else 0.0,
        max_active_fraction=max(fractions, default=0.0),
        size_buckets=size_buckets, duration_buckets=duration_buckets, total_periods=total)


def fractions_csv(report: CharacterizationReport) -> str:
    out = io.StringIO()
    w = csv.writer(out)
    w.writerow(["kernel", "active_bytes", "active_fraction"])
    for k, (b, f) in enumerate(zip(report.active_bytes, report.active_fraction)):
        w.writerow([k, b, f"{f:.6f}"])
    return out.getvalue()


def histogram_csv(report: CharacterizationReport) -> str:
    out = io.StringIO()
    w = csv.writer(out)
    w.writerow(["size_class_bytes", "duration_class_us", "count"])
    for (size_cls, dur_cls), count in sorted(report.histogram.items()):
        w.writerow([size_cls, dur_cls, count])
    return out.getvalue()
