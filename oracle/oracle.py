"""ctypes wrapper around the CPU oracle (tio_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product.

Restates the reference planning path on column arrays (see the C file's
header for the file:line map).  Output is plain Python data so tests can
compare it with both the reference (`offloader`, via tests/golden fixtures)
and the CUDA product.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libtio_oracle.so")
_lib = None

OR_ERR_UNSAT = -2
OR_ERR_RATE = -3


class _Commit(ctypes.Structure):
    _fields_ = [("cand", ctypes.c_int64), ("dest", ctypes.c_int64),
                ("off_s", ctypes.c_int64), ("off_e", ctypes.c_int64),
                ("pre_s", ctypes.c_int64), ("pre_e", ctypes.c_int64),
                ("benefit_lo", ctypes.c_uint64), ("benefit_hi", ctypes.c_uint64),
                ("cost", ctypes.c_int64),
                ("r0_lo", ctypes.c_int64), ("r0_hi", ctypes.c_int64),
                ("r1_lo", ctypes.c_int64), ("r1_hi", ctypes.c_int64),
                ("_tail", ctypes.c_int64)]  # struct padded to 16-byte alignment (u128 member)


class _Result(ctypes.Structure):
    _fields_ = [("n_commits", ctypes.c_int64), ("commits", ctypes.POINTER(_Commit)),
                ("planned_host", ctypes.c_int64), ("rounds", ctypes.c_int64),
                ("unsat_kernel", ctypes.c_int64), ("unsat_bytes", ctypes.c_int64)]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        _lib.tio_oracle_plan.restype = ctypes.c_int
        _lib.tio_oracle_count_periods.restype = ctypes.c_int64
        _lib.tio_oracle_periods.restype = ctypes.c_int64
        _lib.tio_oracle_commit_size.restype = ctypes.c_int64
        _lib.tio_oracle_threads.restype = ctypes.c_int
        assert _lib.tio_oracle_commit_size() == ctypes.sizeof(_Commit), "commit_t layout mismatch"
        del i64p
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _cols(arrays):
    a = arrays
    n = a.num_kernels
    t = a.num_tensors
    dur = np.ascontiguousarray(a.duration_us, dtype=np.int64)
    kind = np.ascontiguousarray(a.kind, dtype=np.int8)
    size = np.ascontiguousarray(a.size_bytes, dtype=np.int64)
    ptr = np.ascontiguousarray(a.access_ptr, dtype=np.int64)
    acc = np.ascontiguousarray(a.accesses, dtype=np.int64)
    return n, t, dur, kind, size, ptr, acc


def lifetime(arrays):
    """(periods, timeline, active) for a validated trace's columns.

    periods: dict of arrays in reference order (analysis.py:58-83):
      tensor (position), tensor_id, size, start, end, wraps.
    """
    L = lib()
    n, t, dur, kind, size, ptr, acc = _cols(arrays)
    cnt = L.tio_oracle_count_periods(ctypes.c_int64(n), ctypes.c_int64(t), _p(kind), _p(ptr), _p(acc))
    pt = np.zeros(cnt, np.int64)
    ps = np.zeros(cnt, np.int64)
    pe = np.zeros(cnt, np.int64)
    pw = np.zeros(cnt, np.int8)
    got = L.tio_oracle_periods(ctypes.c_int64(n), ctypes.c_int64(t), _p(kind), _p(ptr), _p(acc),
                               _p(pt), _p(ps), _p(pe), _p(pw))
    assert got == cnt
    timeline = np.zeros(n, np.int64)
    active = np.zeros(n, np.int64)
    L.tio_oracle_timeline(ctypes.c_int64(n), ctypes.c_int64(t), _p(kind), _p(size), _p(ptr), _p(acc),
                          _p(timeline))
    L.tio_oracle_active(ctypes.c_int64(n), ctypes.c_int64(t), _p(size), _p(ptr), _p(acc), _p(active))
    periods = {"tensor": pt, "tensor_id": arrays.tensor_id[pt], "size": size[pt],
               "start": ps, "end": pe, "wraps": pw.astype(bool)}
    return periods, timeline, active


class OracleUnsatisfiable(Exception):
    def __init__(self, kernel, nbytes):
        super().__init__(f"kernel {kernel} uses {nbytes} bytes")
        self.kernel = kernel
        self.nbytes = nbytes


def plan(arrays, capacity: int, ssd_off: float, ssd_pre: float, host_off=None, host_pre=None,
         host_cap: int = 0, lifetime_out=None, verbose: bool = False, max_rounds: int = 0) -> dict:
    """Algorithm 1 restated (planner.py:267-370) + mark_urgent + entry sort.

    Returns a dict with `committed` (list of tuples matching the reference
    CommittedMigration fields, relieved kernels as (lo, hi) ranges), `residual`,
    `planned_host_bytes`, `over_capacity_kernels`, `entries`
    (tensor_id, action, trigger, deadline, target, urgent) and `plan_bytes`
    (write_plan, planner.py:402-420).
    """
    L = lib()
    n, t, dur, kind, size, ptr, acc = _cols(arrays)
    periods, timeline, active = lifetime_out if lifetime_out is not None else lifetime(arrays)
    order = np.lexsort((periods["start"], periods["tensor_id"]))
    ptensor = periods["tensor"][order]
    p_size = np.ascontiguousarray(size[ptensor])
    p_start = np.ascontiguousarray(periods["start"][order])
    p_end = np.ascontiguousarray(periods["end"][order])
    p_wraps = np.ascontiguousarray(periods["wraps"][order].astype(np.int8))
    p_first = np.ascontiguousarray(acc[ptr[ptensor]]) if len(ptensor) else np.zeros(0, np.int64)
    p_last = np.ascontiguousarray(acc[ptr[ptensor + 1] - 1]) if len(ptensor) else np.zeros(0, np.int64)
    P = len(ptensor)
    has_host = host_off is not None and host_pre is not None
    residual = np.zeros(n, np.int64)
    res = _Result()
    rc = L.tio_oracle_plan(
        ctypes.c_int64(n), _p(dur), _p(active), _p(timeline), ctypes.c_int64(capacity),
        ctypes.c_double(ssd_off), ctypes.c_double(ssd_pre), ctypes.c_int(1 if has_host else 0),
        ctypes.c_double(host_off if has_host else 0.0), ctypes.c_double(host_pre if has_host else 0.0),
        ctypes.c_int64(host_cap), ctypes.c_int64(P), _p(p_size), _p(p_start), _p(p_end), _p(p_wraps),
        _p(p_first), _p(p_last), _p(residual), ctypes.byref(res), ctypes.c_int(1 if verbose else 0),
        ctypes.c_int64(max_rounds))
    if rc == OR_ERR_UNSAT:
        raise OracleUnsatisfiable(res.unsat_kernel, res.unsat_bytes)
    if rc != 0:
        raise RuntimeError(f"oracle plan failed rc={rc}")
    tensor_ids = arrays.tensor_id
    committed = []
    for j in range(res.n_commits):
        c = res.commits[j]
        i = c.cand
        tp = int(ptensor[i])
        ranges = tuple((lo, hi) for lo, hi in ((c.r0_lo, c.r0_hi), (c.r1_lo, c.r1_hi)) if lo <= hi)
        committed.append((int(tensor_ids[tp]), int(p_start[i]), int(p_end[i]), bool(p_wraps[i]),
                          "SSD" if c.dest == 1 else "CPU", (c.off_s, c.off_e), (c.pre_s, c.pre_e),
                          (c.benefit_hi << 64) | c.benefit_lo, c.cost, ranges, tp))
    if res.commits:
        L.tio_oracle_free(ctypes.cast(res.commits, ctypes.c_void_p))
    over = np.flatnonzero(residual > capacity).tolist()
    # entries in commit order (offload, prefetch), then stable sort (planner.py:360-361)
    raw = []
    for c in committed:
        raw.append((c[0], "offload", c[5][0], c[5][1], c[4], c[10]))
        raw.append((c[0], "prefetch", c[6][0], c[6][1], "GPU", c[10]))
    raw.sort(key=lambda e: (e[2], e[0], 0 if e[1] == "offload" else 1))
    starts = np.zeros(n + 1, np.int64)
    np.cumsum(dur, out=starts[1:])
    iteration = int(starts[n])
    entries = []
    for tid, action, trig, dl, target, tp in raw:
        urgent = False
        if action == "prefetch":   # mark_urgent (planner.py:373-397)
            ts = starts[acc[ptr[tp]:ptr[tp + 1]]]
            j = int(np.searchsorted(ts, dl, side="left"))
            need = int(ts[j]) if j < len(ts) else None
            if kind[tp] == 1:
                wrap = iteration + int(ts[0])
                if wrap >= dl and (need is None or wrap < need):
                    need = wrap
            urgent = need == dl
        entries.append((tid, action, trig, dl, target, urgent))
    peak = int(residual.max()) if n else 0
    return {"committed": committed, "residual": residual, "planned_host_bytes": res.planned_host,
            "over_capacity_kernels": over, "entries": entries, "rounds": res.rounds,
            "plan_bytes": format_plan(capacity, peak, res.planned_host, over, entries)}


def format_plan(capacity, residual_peak, planned_host, over, entries) -> bytes:
    """write_plan byte format (planner.py:402-420)."""
    lines = ['{"version": 1, "capacity_bytes": %d, "residual_peak_bytes": %d, '
             '"planned_host_bytes": %d, "over_capacity_kernels": [%s]}'
             % (capacity, residual_peak, planned_host, ", ".join(map(str, over)))]
    for tid, action, trig, dl, target, urgent in entries:
        lines.append('{"tensor": %d, "action": "%s", "trigger_us": %d, "deadline_us": %d, '
                     '"target": "%s", "urgent": %s}'
                     % (tid, action, trig, dl, target, "true" if urgent else "false"))
    return ("\n".join(lines) + "\n").encode("utf-8")
