"""Lifetime-aware migration planning — reference `offloader/planner.py` API.

`plan_migrations` (planner.py:267-370) runs entirely on the B200: the
lifetime stage, candidate construction in (tensor_id, start_kernel) order,
the greedy benefit/cost round loop (csrc/planner.cu, one persistent
cooperative kernel), the entry sort and `mark_urgent` (csrc/plan_setup.cu).
This module converts the device results to the reference's dataclasses and
maps libtio status codes back to the reference exceptions.

`candidate_window`, `candidate_benefit` and `select_destination` are the
reference's per-candidate helpers over `BandwidthChannel` objects
(planner.py:147-262); they are host-side inspection helpers that the device
planner does not use.
"""

from __future__ import annotations

import ctypes

import json
import logging
from collections.abc import Sequence
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from .analysis import InactivePeriod, MemoryTimeline, _device_trace
from .bandwidth import BandwidthChannel, ChannelConfigError, ChannelPair, ChannelRates, Reservation
from .trace import KIND_GLOBAL, Trace

log = logging.getLogger("offloader.planner")

PLAN_FORMAT_VERSION = 1
SSD = "SSD"
CPU = "CPU"
GPU = "GPU"
_TARGET = {1: SSD, 2: CPU}


class UnsatisfiableTraceError(ValueError):
    """Some kernel's actively-used bytes alone exceed capacity."""

    def __init__(self, kernel_index: int, active_bytes: int, capacity: int):
        super().__init__(
            f"kernel {kernel_index} uses {active_bytes} bytes actively, "
            f"more than capacity {capacity}; no offloading plan can help")
        self.kernel_index = kernel_index


@dataclass(frozen=True)
class PlanEntry:
    tensor_id: int
    action: str           # "offload" | "prefetch"
    trigger_time: int     # scheduled transfer start (us)
    deadline: int         # scheduled transfer completion (us)
    target: str           # SSD | CPU for offloads, GPU for prefetches
    urgent: bool = False


@dataclass
class CandidateWindow:
    t_offloaded: int
    t_prefetch: int
    offload_reservation: Reservation
    prefetch_reservation: Reservation
    destination: str


@dataclass(frozen=True)
class Benefit:
    value: int
    critical_kernels: frozenset[int]


@dataclass(frozen=True)
class CommittedMigration:
    tensor_id: int
    start_kernel: int
    end_kernel: int
    wraps: bool
    destination: str
    offload_interval: tuple[int, int]
    prefetch_interval: tuple[int, int]
    benefit: int
    cost: int
    relieved_kernels: tuple[int, ...]


def _commit_of(row) -> CommittedMigration:
    rel = []
    for lo, hi in ((int(row["rel0_lo"]), int(row["rel0_hi"])), (int(row["rel1_lo"]), int(row["rel1_hi"]))):
        if lo <= hi:
            rel.extend(range(lo, hi + 1))
    return CommittedMigration(
        tensor_id=int(row["tensor_id"]), start_kernel=int(row["start_kernel"]),
        end_kernel=int(row["end_kernel"]), wraps=bool(row["wraps"]),
        destination=_TARGET[int(row["destination"])],
        offload_interval=(int(row["off_start"]), int(row["off_end"])),
        prefetch_interval=(int(row["pre_start"]), int(row["pre_end"])),
        benefit=(int(row["benefit_hi"]) << 64) | int(row["benefit_lo"]),
        cost=int(row["cost"]), relieved_kernels=tuple(rel))


class CommitLog(Sequence):
    """Commit records of a device plan, materialised per item on access
    (a 10^4-round plan relieves ~10^7 kernel slots in total)."""

    def __init__(self, rows: np.ndarray):
        self.rows = rows

    def __len__(self) -> int:
        return int(self.rows.shape[0])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [_commit_of(self.rows[j]) for j in range(*i.indices(len(self)))]
        return _commit_of(self.rows[i])

    def __eq__(self, other) -> bool:
        if isinstance(other, CommitLog):
            return np.array_equal(self.rows, other.rows)
        if isinstance(other, Sequence):
            return len(other) == len(self) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __repr__(self) -> str:
        return f"CommitLog({len(self)} commits)"


@dataclass
class MigrationPlan:
    entries: list[PlanEntry]
    residual_timeline: MemoryTimeline
    planned_host_bytes: int
    over_capacity_kernels: list[int]
    capacity_bytes: int
    committed: Sequence
    rounds: int = 0

    @property
    def warning(self) -> bool:
        return bool(self.over_capacity_kernels)


# --- per-candidate helpers (host-side inspection API) -----------------------------

def _period_times(period: InactivePeriod, trace: Trace, starts: list[int], iteration: int) -> tuple[int, int]:
    if not period.wraps:
        return starts[period.start_kernel], starts[period.end_kernel + 1]
    a = trace.arrays()
    pos = int(np.flatnonzero(a.tensor_id == period.tensor_id)[0])
    first = int(a.accesses[a.access_ptr[pos]])
    last = int(a.accesses[a.access_ptr[pos + 1] - 1])
    return starts[last] + int(a.duration_us[last]), iteration + starts[first]


def _starts_full(trace: Trace) -> list[int]:
    d = trace.arrays().duration_us
    s = np.zeros(d.shape[0] + 1, np.int64)
    np.cumsum(d, out=s[1:])
    return s.tolist()


def candidate_window(period: InactivePeriod, trace: Trace, offload_channel: BandwidthChannel,
                     prefetch_channel: BandwidthChannel, destination: str) -> CandidateWindow | None:
    """Book a trial offload/prefetch pair (planner.py:147-176, libtio
    `tio_candidate_window`); on success the bookings stay live in the
    channels, on failure nothing stays booked."""
    starts = _starts_full(trace)
    iteration = starts[-1]
    ready, deadline = _period_times(period, trace, starts, iteration)
    ok, oid, oend, pid, pstart = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), \
        ctypes.c_int64()
    _native.check(_native.load().tio_candidate_window(
        offload_channel._h, prefetch_channel._h, ctypes.c_int64(ready), ctypes.c_int64(deadline),
        ctypes.c_int64(period.size_bytes), ctypes.c_int64(iteration), ctypes.c_int64(period.tensor_id),
        ctypes.byref(ok), ctypes.byref(oid), ctypes.byref(oend), ctypes.byref(pid), ctypes.byref(pstart)))
    if not ok.value:
        return None
    d_off = offload_channel.transfer_duration(period.size_bytes)
    d_pre = prefetch_channel.transfer_duration(period.size_bytes)
    off = offload_channel._booked(oid.value, oend.value - d_off, oend.value, period.tensor_id)
    pre = prefetch_channel._booked(pid.value, pstart.value, pstart.value + d_pre, period.tensor_id)
    return CandidateWindow(off.end, pre.start, off, pre, destination)


def _host_peak_occupancy(intervals, lo: int, hi: int) -> int:
    """planner.py:179-186 (libtio `tio_host_peak_occupancy`)."""
    iv = np.asarray([(s, e, z) for s, e, z in intervals], np.int64).reshape(-1, 3)
    cols = [np.ascontiguousarray(iv[:, j]) for j in range(3)]
    out = ctypes.c_int64()
    _native.check(_native.load().tio_host_peak_occupancy(
        *(c.ctypes.data_as(ctypes.c_void_p) for c in cols), ctypes.c_int64(iv.shape[0]), ctypes.c_int64(lo),
        ctypes.c_int64(hi), ctypes.byref(out)))
    return out.value


def _release(window: CandidateWindow, ssd: ChannelPair, host: ChannelPair | None) -> None:
    pair = ssd if window.destination == SSD else host
    pair.offload.release(window.offload_reservation)
    pair.prefetch.release(window.prefetch_reservation)


def _attempt(period, trace, ssd, host, host_cap, host_occupancy):
    w = candidate_window(period, trace, ssd.offload, ssd.prefetch, SSD)
    if w is not None or host is None:
        return w
    w = candidate_window(period, trace, host.offload, host.prefetch, CPU)
    if w is None:
        return None
    if _host_peak_occupancy(host_occupancy, w.t_offloaded, w.t_prefetch) + period.size_bytes > host_cap:
        _release(w, ssd, host)
        return None
    return w


def select_destination(period: InactivePeriod, trace: Trace, ssd_channels: ChannelPair,
                       host_channels: ChannelPair | None, host_cap: int,
                       host_occupancy: list[tuple[int, int, int]]) -> str | None:
    w = _attempt(period, trace, ssd_channels, host_channels, host_cap, host_occupancy)
    if w is None:
        return None
    _release(w, ssd_channels, host_channels)
    return w.destination


def candidate_benefit(window: CandidateWindow, period: InactivePeriod, residual: MemoryTimeline,
                      capacity: int, trace: Trace) -> Benefit:
    """size x duration of over-capacity kernels fully inside the window
    (planner.py:232-262, libtio `tio_candidate_benefit`)."""
    a = trace.arrays()
    N = a.num_kernels
    starts = np.zeros(N + 1, np.int64)
    np.cumsum(a.duration_us, out=starts[1:])
    dur = np.ascontiguousarray(a.duration_us, np.int64)
    resid = np.ascontiguousarray(np.asarray(residual.per_kernel_bytes, np.int64))
    first = last = 0
    if period.wraps:
        pos = int(np.flatnonzero(a.tensor_id == period.tensor_id)[0])
        first = int(a.accesses[a.access_ptr[pos]])
        last = int(a.accesses[a.access_ptr[pos + 1] - 1])
    crit = np.zeros(max(N, 1), np.int8)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _native.check(_native.load().tio_candidate_benefit(
        vp(starts), vp(dur), vp(resid), ctypes.c_int64(N), ctypes.c_int64(capacity),
        ctypes.c_int32(1 if period.wraps else 0), ctypes.c_int64(period.start_kernel),
        ctypes.c_int64(period.end_kernel), ctypes.c_int64(first), ctypes.c_int64(last),
        ctypes.c_int64(window.t_offloaded), ctypes.c_int64(window.t_prefetch), ctypes.c_int64(period.size_bytes),
        ctypes.byref(lo), ctypes.byref(hi), vp(crit)))
    return Benefit(value=(hi.value << 64) | lo.value,
                   critical_kernels=frozenset(np.flatnonzero(crit[:N]).tolist()))


# --- the device planner --------------------------------------------------------------

def _rates_struct(rates: ChannelRates) -> _native.Rates:
    for v in (rates.ssd_offload, rates.ssd_prefetch):
        if v is None:
            raise ChannelConfigError("ssd rates are required")
    host = rates.has_host
    return _native.Rates(float(rates.ssd_offload), float(rates.ssd_prefetch), 1 if host else 0,
                         float(rates.host_offload) if host else 0.0,
                         float(rates.host_prefetch) if host else 0.0)


def _raise_for(err: _native.TioError, capacity: int, rates: ChannelRates) -> None:
    if err.code == _native.TIO_ERR_UNSATISFIABLE:
        info = err.info
        raise UnsatisfiableTraceError(info.unsat_kernel, info.unsat_bytes, capacity) from None
    if err.code == _native.TIO_ERR_CHANNEL_CONFIG:
        # reference names the first channel it builds with a bad rate
        for name, direction, v in (("ssd", "offload", rates.ssd_offload), ("ssd", "prefetch", rates.ssd_prefetch),
                                   ("host", "offload", rates.host_offload),
                                   ("host", "prefetch", rates.host_prefetch)):
            if v is not None and not v > 0:
                raise ChannelConfigError(f"channel {name}.{direction}: rate must be > 0") from None
        raise ChannelConfigError(err.message) from None
    raise err


def plan_device(trace: Trace, capacity: int, rates: ChannelRates, host_cap: int = 0, max_rounds: int = 0) -> dict:
    """Run the device planner; return its raw columns (commits, entries,
    residual, over) plus the info struct — no per-entry Python objects.
    max_rounds > 0 stops after that many commits (a prefix of the plan)."""
    dt = _device_trace(trace)
    try:
        p = dt.plan(capacity, _rates_struct(rates), host_cap, max_rounds)
    except _native.TioError as err:
        _raise_for(err, capacity, rates)
    try:
        out = p.copy_out()
        out["info"] = p.info
        out["plan_bytes"] = p.write()
    finally:
        p.close()
    return out


def plan_device_virtual(trace: Trace, capacity: int, rates: ChannelRates, host_cap: int = 0, nranks: int = 2,
                        max_rounds: int = 0) -> list[dict]:
    """The sharded planner run by `nranks` virtual ranks on this
    GPU (tio_plan_create_virtual): each rank evaluates only its candidate
    tiles, the ranks exchange their round's best through device mailboxes and
    apply the same commit.  Returns every rank's raw output (plan_device
    format); all must equal the single-rank plan."""
    dt = _device_trace(trace)
    try:
        plans = dt.plan_virtual(capacity, _rates_struct(rates), host_cap, nranks, max_rounds)
    except _native.TioError as err:
        _raise_for(err, capacity, rates)
    outs = []
    for p in plans:
        try:
            o = p.copy_out()
            o["info"] = p.info
            o["plan_bytes"] = p.write()
            outs.append(o)
        finally:
            p.close()
    return outs


def plan_migrations(trace: Trace, capacity: int, rates: ChannelRates, host_cap: int = 0) -> MigrationPlan:
    """Greedy Algorithm-1 plan computed on the GPU (planner.py:267-370).

    Raises UnsatisfiableTraceError when some kernel's active bytes exceed
    capacity; leftover pressure is reported in `over_capacity_kernels`.
    """
    raw = plan_device(trace, capacity, rates, host_cap)
    info = raw["info"]
    ents = raw["entries"]
    entries = [PlanEntry(int(t), "prefetch" if a else "offload", int(tr), int(dl),
                         GPU if a else _TARGET.get(int(tg), SSD), bool(u))
               for t, a, tr, dl, tg, u in zip(ents["tensor_id"].tolist(), ents["action"].tolist(),
                                              ents["trigger_us"].tolist(), ents["deadline_us"].tolist(),
                                              ents["target"].tolist(), ents["urgent"].tolist())]
    rows = raw["commits"]
    committed = [_commit_of(r) for r in rows] if len(rows) <= 4096 else CommitLog(rows)
    for c in (committed if isinstance(committed, list) else []):
        log.debug("committed tensor %d period [%d,%d] to %s, benefit %d cost %d",
                  c.tensor_id, c.start_kernel, c.end_kernel, c.destination, c.benefit, c.cost)
    return MigrationPlan(entries=entries, residual_timeline=MemoryTimeline(raw["residual"].tolist()),
                         planned_host_bytes=int(info.planned_host_bytes),
                         over_capacity_kernels=raw["over"].tolist(), capacity_bytes=capacity,
                         committed=committed, rounds=int(info.rounds))


def mark_urgent(plan: MigrationPlan, trace: Trace) -> MigrationPlan:
    """Flag zero-slack prefetches (planner.py:373-397).  plan_migrations
    already marks its entries on the device; this re-marks any entry list."""
    a = trace.arrays()
    d = a.duration_us
    starts = np.zeros(d.shape[0] + 1, np.int64)
    np.cumsum(d, out=starts[1:])
    iteration = int(starts[-1])
    pos_of = {int(t): i for i, t in enumerate(a.tensor_id.tolist())}
    flagged = []
    for e in plan.entries:
        if e.action != "prefetch":
            flagged.append(replace(e, urgent=False))
            continue
        i = pos_of[e.tensor_id]
        ts = starts[a.accesses[a.access_ptr[i]:a.access_ptr[i + 1]]]
        j = int(np.searchsorted(ts, e.deadline, side="left"))
        need = int(ts[j]) if j < ts.shape[0] else None
        if a.kind[i] == KIND_GLOBAL:
            wrap = iteration + int(ts[0])
            if wrap >= e.deadline and (need is None or wrap < need):
                need = wrap
        flagged.append(replace(e, urgent=(need == e.deadline)))
    plan.entries = flagged
    return plan


# --- plan file (planner.py:402-442) --------------------------------------------------

def write_plan(plan: MigrationPlan) -> bytes:
    lines = [json.dumps({
        "version": PLAN_FORMAT_VERSION,
        "capacity_bytes": plan.capacity_bytes,
        "residual_peak_bytes": plan.residual_timeline.peak(),
        "planned_host_bytes": plan.planned_host_bytes,
        "over_capacity_kernels": plan.over_capacity_kernels,
    })]
    for e in plan.entries:
        lines.append(json.dumps({"tensor": e.tensor_id, "action": e.action, "trigger_us": e.trigger_time,
                                 "deadline_us": e.deadline, "target": e.target, "urgent": e.urgent}))
    return ("\n".join(lines) + "\n").encode("utf-8")


def parse_plan(data: bytes | str) -> tuple[dict, list[PlanEntry]]:
    text = data.decode("utf-8") if isinstance(data, bytes) else data
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise ValueError("empty plan file")
    header = json.loads(lines[0])
    if header.get("version") != PLAN_FORMAT_VERSION:
        raise ValueError(f"unsupported plan version {header.get('version')!r}")
    entries = []
    for ln in lines[1:]:
        o = json.loads(ln)
        entries.append(PlanEntry(o["tensor"], o["action"], o["trigger_us"], o["deadline_us"],
                                 o["target"], o["urgent"]))
    return header, entries
