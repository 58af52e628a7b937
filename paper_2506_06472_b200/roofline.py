"""Roofline study — reference `offloader/roofline.py` API.

Normalized training throughput as a function of migration bandwidth under
the reference's roofline policy (roofline.py:1-12: every inactive period is
migrated when the trace oversubscribes capacity, serial offload and prefetch
channels at one rate).  The sweep runs in libtio (`tio_roofline`,
csrc/roofline.cu, host C++): the two bandwidth-independent processing orders
are built once and each bandwidth is one max/+ pass, on its own thread.
"""

from __future__ import annotations

import csv
import ctypes
import io
from dataclasses import dataclass

import numpy as np

from . import _native
from .trace import Trace


@dataclass(frozen=True)
class RooflinePoint:
    bandwidth: float            # bytes per microsecond, both directions
    normalized_throughput: float


def _sweep(trace: Trace, capacity: int, bandwidths) -> tuple[np.ndarray, "_native.RooflineInfoC"]:
    lib = _native.load()
    cols = _native.HostColumns(trace.arrays())
    desc = cols.desc()
    bw = np.ascontiguousarray(bandwidths, dtype=np.float64)
    tot = np.zeros(bw.shape[0], np.int64)
    info = _native.RooflineInfoC()
    _native.check(lib.tio_roofline(ctypes.byref(desc), ctypes.c_int64(capacity), _native._ptr(bw),
                                   ctypes.c_int64(bw.shape[0]), _native._ptr(tot), ctypes.byref(info)))
    return tot, info


def roofline_curve(trace: Trace, capacity: int, bandwidth_list: list[float]) -> list[RooflinePoint]:
    """One point per bandwidth; the list must be positive and ascending
    (roofline.py:90-110)."""
    if not bandwidth_list:
        raise ValueError("bandwidth list must be non-empty")
    if any(b <= 0 for b in bandwidth_list):
        raise ValueError("bandwidths must be positive")
    if list(bandwidth_list) != sorted(bandwidth_list):
        raise ValueError("bandwidths must be ascending")
    tot, info = _sweep(trace, capacity, [float(b) for b in bandwidth_list])
    ideal = int(info.ideal_us)
    points = []
    for b, t in zip(bandwidth_list, tot.tolist()):
        if not info.pressured or ideal == 0:
            points.append(RooflinePoint(b, 1.0))
        else:
            points.append(RooflinePoint(b, 1.0 if t == ideal else ideal / t))
    return points


def saturation_bandwidth(trace: Trace) -> int:
    """A bandwidth past the curve's knee (roofline.py:113-125): the largest
    period size times the period count."""
    _, info = _sweep(trace, 0, [])
    return int(info.max_period_bytes) * max(1, int(info.num_periods))


def roofline_csv(points: list[RooflinePoint]) -> str:
    out = io.StringIO()
    w = csv.writer(out)
    w.writerow(["bandwidth_gbps", "normalized_throughput"])
    for p in points:
        w.writerow([p.bandwidth / 1000, f"{p.normalized_throughput:.6f}"])
    return out.getvalue()
