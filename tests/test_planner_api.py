"""Planner building blocks (reference planner.py:130-262): candidate_window,
candidate_benefit, select_destination — the reference's test_planner.py
known answers restated.  The periods are written out (EX1's single period,
analysis.py:58-83) so these run without a GPU."""

from __future__ import annotations

from conftest import mk_trace
from paper_2506_06472_b200 import (CandidateWindow, ChannelRates, InactivePeriod, MemoryTimeline, candidate_benefit,
                                   candidate_window, select_destination)
from paper_2506_06472_b200.bandwidth import build_channels

MB100 = 100_000_000
CAP = 150_000_000
SSD = "SSD"
A = InactivePeriod(tensor_id=0, size_bytes=MB100, start_kernel=1, end_kernel=3, wraps=False)   # EX1's period


def ssd_pair(rate=20_000, period=50_000):
    return build_channels(ChannelRates.symmetric(rate), period)["ssd"]


def host_pair():
    return build_channels(ChannelRates.symmetric(1, host=20_000), 50_000)["host"]


def test_candidate_window(ex1):
    pair = ssd_pair()
    w = candidate_window(A, ex1, pair.offload, pair.prefetch, SSD)
    assert w.t_offloaded == 15_000 and w.offload_reservation.interval() == (10_000, 15_000)
    assert w.t_prefetch == 35_000 and w.prefetch_reservation.interval() == (35_000, 40_000)
    pair = ssd_pair()
    pair.offload.reserve_earliest(10_000, 560_000_000)             # occupies [10000, 38000]
    assert candidate_window(A, ex1, pair.offload, pair.prefetch, SSD) is None
    assert len([r for r in pair.offload.reservations if not r.shadow]) == 1   # trial bookings rolled back
    assert [r for r in pair.prefetch.reservations if not r.shadow] == []
    tiny = mk_trace([10] * 3, [(0, MB100, "intermediate", [0, 2])])
    pair = ssd_pair(rate=20_000, period=30)
    assert candidate_window(InactivePeriod(0, MB100, 1, 1, False), tiny, pair.offload, pair.prefetch, SSD) is None


def test_candidate_benefit(ex1):
    w = CandidateWindow(15_000, 35_000, None, None, SSD)
    b = candidate_benefit(w, A, MemoryTimeline([MB100, MB100, 2 * MB100, MB100, MB100]), CAP, ex1)
    assert b.critical_kernels == frozenset({2}) and b.value == MB100 * 10_000
    b = candidate_benefit(w, A, MemoryTimeline([MB100] * 5), CAP, ex1)
    assert b.value == 0 and b.critical_kernels == frozenset()
    tr = mk_trace([10_000] * 4, [(0, 50_000_000, "intermediate", [0, 3])])
    b = candidate_benefit(CandidateWindow(10_000, 30_000, None, None, SSD), InactivePeriod(0, 50_000_000, 1, 2, False),
                          MemoryTimeline([0, CAP + 1, CAP + 1, 0]), CAP, tr)
    assert b.critical_kernels == frozenset({1, 2}) and b.value == 50_000_000 * 20_000


def test_select_destination(ex1):
    assert select_destination(A, ex1, ssd_pair(), host_pair(), 10**9, []) == "SSD"
    assert select_destination(A, ex1, ssd_pair(rate=1), host_pair(), 10**9, []) == "CPU"
    assert select_destination(A, ex1, ssd_pair(rate=1), host_pair(), MB100 - 1, []) is None
    assert select_destination(A, ex1, ssd_pair(rate=1), host_pair(), CAP, [(0, 50_000, 60_000_000)]) is None
