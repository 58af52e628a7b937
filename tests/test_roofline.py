"""Roofline sweep (reference roofline.py:39-125) through libtio's
`tio_roofline` (host C++): the reference's own test_roofline.py known answers
and its outputs on a golden corpus (tests/golden/roofline.json.gz, made by
tests/golden/make_golden.py from the reference).  Host-only: no GPU."""

from __future__ import annotations

import hashlib

import pytest

from conftest import load_golden, mk_trace, regen
from paper_2506_06472_b200 import (TransformerGenConfig, gen_random_trace, gen_transformer_trace, roofline_curve,
                                   saturation_bandwidth, write_trace)
from paper_2506_06472_b200.roofline import roofline_csv

CAP = 150_000_000


def test_golden_corpus_matches_reference():
    cases = load_golden("roofline")
    assert len(cases) >= 120
    for rec in cases:
        if rec["gen"].get("c1"):
            tr = gen_transformer_trace(TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8,
                                                            seq_len=1024, bytes_per_element=4,
                                                            compute_rate=1_000_000_000, seed=0))
            assert hashlib.sha256(write_trace(tr)).hexdigest() == rec["trace_sha256"]
        else:
            tr = regen(rec)
        pts = roofline_curve(tr, rec["capacity"], rec["grid"])
        assert [p.normalized_throughput for p in pts] == rec["points"]
        assert [p.bandwidth for p in pts] == rec["grid"]
        assert saturation_bandwidth(tr) == rec["saturation"]


# reference test_roofline.py:11-68
def test_no_pressure_is_flat_one(ex1):
    assert [p.normalized_throughput for p in roofline_curve(ex1, 250_000_000, [1_000, 20_000])] == [1.0, 1.0]


def test_ex1_channels(ex1):
    assert roofline_curve(ex1, CAP, [20_000])[0].normalized_throughput == 1.0
    assert roofline_curve(ex1, CAP, [1_000])[0].normalized_throughput == pytest.approx(50_000 / 220_000)


def test_bandwidth_list_validation(ex1):
    for bad in ([], [5, 1], [0]):
        with pytest.raises(ValueError):
            roofline_curve(ex1, CAP, bad)


def test_monotone_and_bounded_on_random_traces():
    grid = [10, 30, 100, 300, 1_000, 10_000]
    for seed in range(30):
        trace = gen_random_trace(seed, 10, 8, size_range=(1_000, 80_000), duration_range=(50, 500))
        capacity = max(1, sum(int(s) for s in trace.arrays().size_bytes) // 2)
        values = [p.normalized_throughput for p in roofline_curve(trace, capacity, grid)]
        assert all(0 < v <= 1.0 for v in values)
        assert values == sorted(values)


def test_saturation_reaches_exactly_one(ex1):
    assert roofline_curve(ex1, CAP, [saturation_bandwidth(ex1)])[0].normalized_throughput == 1.0


def test_wrap_traffic_does_not_stall_the_iteration():
    trace = mk_trace([10_000] * 4, [(0, 100_000_000, "global", [1]), (1, 90_000_000, "intermediate", [0, 3])])
    assert roofline_curve(trace, 120_000_000, [20_000])[0].normalized_throughput == 1.0


def test_csv_reports_gbps(ex1):
    lines = roofline_csv(roofline_curve(ex1, CAP, [16_000])).splitlines()
    assert lines[0] == "bandwidth_gbps,normalized_throughput"
    assert lines[1].startswith("16.0,")


def test_criterion_4_roofline_properties():
    """Reference test_acceptance.py:134-150 (the timeline peak from the
    oracle: this test runs without a GPU)."""
    import random

    from oracle import oracle as O
    rng = random.Random(11)
    grid = [5, 20, 80, 320, 1_280, 20_000]
    for case in range(100):
        trace = gen_random_trace(rng.randint(0, 10**9), rng.randint(2, 12), rng.randint(1, 8),
                                 size_range=(10_000, 500_000), duration_range=(500, 5_000))
        tl = O.lifetime(trace.arrays())[1]
        capacity = max(1, (int(tl.max()) if len(tl) else 0) // 2)
        values = [p.normalized_throughput for p in roofline_curve(trace, capacity, grid)]
        assert values == sorted(values), case
        assert all(0 < v <= 1.0 for v in values), case
        (top,) = roofline_curve(trace, capacity, [saturation_bandwidth(trace)])
        assert top.normalized_throughput == 1.0, case
