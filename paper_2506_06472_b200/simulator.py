"""Migration-engine model — reference `offloader/simulator.py` API.

`simulate` / `simulate_on_demand` / `simulate_ideal` (simulator.py:539-547)
run the engine scheduler of libtio (csrc/engine_sched.cu, host C++): the
exact `_Engine` semantics (simulator.py:178-528) — location table, four
serial channels with urgent/front queueing, capacity-gated prefetches,
Belady emergency eviction, steady-state plan folding.  The same scheduler
drives the GPU executor (`paper_2506_06472_b200.engine`), so this is also
the step-time predictor of a plan before it runs.

The layer-granularity baseline (`simulate_layer_granularity`, :549-560,
policy :95-177) runs on the same scheduler with the
layer-batch hooks (`tio_simulate_layers`).
"""

from __future__ import annotations

import csv
import ctypes
import io
import json
from dataclasses import dataclass

import numpy as np

from . import _native
from .bandwidth import ChannelRates
from .planner import MigrationPlan, PlanEntry, _rates_struct
from .trace import NONE_I64, Trace


class SimulationError(RuntimeError):
    """The trace cannot execute under the given capacity/channel setup."""


class ConfigurationError(ValueError):
    """The policy's inputs are incomplete (e.g. missing layer ids)."""


@dataclass
class SimReport:
    total_time: int
    ideal_time: int
    per_kernel_start: list[int]
    stall_per_kernel: list[int]
    per_kernel_resident: list[int]
    stall_time_total: int
    peak_resident_bytes: int
    channel_utilization: dict[str, float]
    emergency_offloads: int
    throughput_vs_ideal: float


def simulate_ideal(trace: Trace) -> int:
    """Iteration time with infinite GPU memory: the sum of kernel durations."""
    return int(trace.arrays().duration_us.sum())


def _entries_of(plan) -> list[PlanEntry]:
    if plan is None:
        return []
    if isinstance(plan, MigrationPlan):
        return plan.entries
    return list(plan)


def entries_array(entries) -> np.ndarray:
    out = np.zeros(len(entries), _native.ENTRY_DTYPE)
    for i, e in enumerate(entries):
        out[i]["tensor_id"] = e.tensor_id
        out[i]["trigger_us"] = e.trigger_time
        out[i]["deadline_us"] = e.deadline
        out[i]["action"] = 0 if e.action == "offload" else 1
        out[i]["target"] = {"SSD": 1, "CPU": 2}.get(e.target, 0)
        out[i]["urgent"] = 1 if e.urgent else 0
    return out


_CHANNELS = ("ssd.offload", "ssd.prefetch", "host.offload", "host.prefetch")


def _run(trace: Trace, entries: np.ndarray, capacity: int, rates: ChannelRates, layers=None) -> SimReport:
    lib = _native.load()
    cols = _native.HostColumns(trace.arrays())
    desc = cols.desc()
    n = cols.dur.shape[0]
    start = np.zeros(n, np.int64)
    stall = np.zeros(n, np.int64)
    resid = np.zeros(n, np.int64)
    rep = _native.SimReportC()
    r = _rates_struct(rates)
    if layers is None:
        rc = lib.tio_simulate(ctypes.byref(desc), _native._ptr(entries), ctypes.c_int64(entries.shape[0]),
                              ctypes.c_int64(capacity), ctypes.byref(r), ctypes.byref(rep), _native._ptr(start),
                              _native._ptr(stall), _native._ptr(resid))
    else:
        kl, tl = layers
        rc = lib.tio_simulate_layers(ctypes.byref(desc), _native._ptr(kl), _native._ptr(tl), ctypes.c_int64(capacity),
                                     ctypes.byref(r), ctypes.byref(rep), _native._ptr(start), _native._ptr(stall),
                                     _native._ptr(resid))
    if rc == _native.TIO_ERR_SIMULATION:
        raise SimulationError(_native.last_error())
    if rc == _native.TIO_ERR_CONFIG:
        raise ConfigurationError(_native.last_error())
    if rc == _native.TIO_ERR_CHANNEL_CONFIG:
        from .bandwidth import ChannelConfigError
        raise ChannelConfigError(_native.last_error())      # "channel ssd.offload: rate must be > 0"
    _native.check(rc)
    total = int(rep.total_time)
    ideal = int(rep.ideal_time)
    util = {}
    for c, name in enumerate(_CHANNELS[:4 if rates.has_host else 2]):
        util[name] = int(rep.channel_busy[c]) / total if total > 0 else 0.0
    return SimReport(
        total_time=total, ideal_time=ideal, per_kernel_start=start.tolist(), stall_per_kernel=stall.tolist(),
        per_kernel_resident=resid.tolist(), stall_time_total=int(rep.stall_time_total),
        peak_resident_bytes=int(rep.peak_resident_bytes), channel_utilization=util,
        emergency_offloads=int(rep.emergency_offloads),
        throughput_vs_ideal=1.0 if total == ideal else ideal / total)


def schedule(trace: Trace, plan, capacity: int, rates: ChannelRates):
    """The engine program the GPU executor runs: (transfers as a
    TRANSFER_DTYPE array in start order, kernel start times, kernel launch
    positions in the processing order, initial tensor locations)."""
    lib = _native.load()
    cols = _native.HostColumns(trace.arrays())
    desc = cols.desc()
    ents = entries_array(_entries_of(plan))
    r = _rates_struct(rates)
    n = ctypes.c_int64()
    args = (ctypes.byref(desc), _native._ptr(ents), ctypes.c_int64(ents.shape[0]), ctypes.c_int64(capacity),
            ctypes.byref(r))
    rc = lib.tio_schedule(*args, None, ctypes.c_int64(0), ctypes.byref(n), None, None, None)
    if rc == _native.TIO_ERR_SIMULATION:
        raise SimulationError(_native.last_error())
    _native.check(rc)
    xs = np.zeros(n.value, _native.TRANSFER_DTYPE)
    starts = np.zeros(cols.dur.shape[0], np.int64)
    kseq = np.zeros(cols.dur.shape[0], np.int64)
    loc = np.zeros(cols.tid.shape[0], np.int8)
    _native.check(lib.tio_schedule(*args, _native._ptr(xs), ctypes.c_int64(n.value), ctypes.byref(n),
                                   _native._ptr(starts), _native._ptr(kseq), _native._ptr(loc)))
    return xs, starts, kseq, loc


def simulate(trace: Trace, plan, capacity: int, rates: ChannelRates) -> SimReport:
    """Execute the trace under a migration plan (a MigrationPlan, a list of
    entries, or None for no planned transfers) in the engine model."""
    return _run(trace, entries_array(_entries_of(plan)), capacity, rates)


def simulate_on_demand(trace: Trace, capacity: int, rates: ChannelRates) -> SimReport:
    """Baseline: no planning at all, every migration happens at point of need."""
    return _run(trace, entries_array([]), capacity, rates)


def simulate_layer_granularity(trace: Trace, capacity: int, rates: ChannelRates, layer_map=None) -> SimReport:
    """Baseline: batch offload/prefetch at whole-layer granularity
    (simulator.py:549-560, policy :95-177), run by the native scheduler
    (`tio_simulate_layers`).  Engages only when the trace oversubscribes
    capacity; `layer_map` ({tensor id: layer}) overrides tensor layers."""
    a = trace.arrays()
    kl = np.ascontiguousarray(a.kernel_layer, dtype=np.int64)
    tl = np.array(a.tensor_layer, dtype=np.int64, copy=True)
    if layer_map:
        for i, tid in enumerate(a.tensor_id.tolist()):
            if tid in layer_map:
                tl[i] = NONE_I64 if layer_map[tid] is None else int(layer_map[tid])
    return _run(trace, entries_array([]), capacity, rates, layers=(kl, tl))


# --- report serialization (reference simulator.py:565-585) ----------------------

def report_json(report: SimReport) -> str:
    return json.dumps({
        "total_time_us": report.total_time,
        "ideal_time_us": report.ideal_time,
        "throughput_vs_ideal": report.throughput_vs_ideal,
        "stall_time_total_us": report.stall_time_total,
        "peak_resident_bytes": report.peak_resident_bytes,
        "emergency_offloads": report.emergency_offloads,
        "channel_utilization": report.channel_utilization,
    }, indent=2)


def timeline_csv(report: SimReport) -> str:
    out = io.StringIO()
    w = csv.writer(out)
    w.writerow(["kernel", "start_us", "stall_us", "resident_bytes"])
    for k, row in enumerate(zip(report.per_kernel_start, report.stall_per_kernel, report.per_kernel_resident)):
        w.writerow([k, *row])
    return out.getvalue()
