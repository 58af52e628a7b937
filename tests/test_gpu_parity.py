"""GPU parity: the sm_100a lifetime + planner path (libtio, through the C ABI)
against the reference's golden vectors and the CPU oracle.

Bar: bit-exact.  Periods, timeline, active bytes, committed rounds, residual
timeline and write_plan bytes must equal the reference's (tests/golden,
produced by the reference itself) and, at sizes the reference cannot reach,
the oracle's (oracle/tio_oracle.c, itself pinned by test_oracle_golden.py).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import load_golden, mk_trace, rates_of, regen
from oracle import oracle as O
from paper_2506_06472_b200 import (
    ChannelConfigError, ChannelRates, InactivePeriod, PlanEntry, TransformerGenConfig,
    UnsatisfiableTraceError, compute_inactive_periods, compute_memory_timeline, gen_random_trace,
    gen_transformer_trace, lifetime_arrays, mark_urgent, per_kernel_active_bytes, plan_device,
    plan_migrations, write_plan, write_trace)
from paper_2506_06472_b200 import _native

pytestmark = pytest.mark.gpu

MB100 = 100_000_000
CAP = 150_000_000


def _committed_rows(raw):
    out = []
    for r in raw["commits"]:
        rel = []
        for lo, hi in ((int(r["rel0_lo"]), int(r["rel0_hi"])), (int(r["rel1_lo"]), int(r["rel1_hi"]))):
            if lo <= hi:
                rel.extend(range(lo, hi + 1))
        out.append([int(r["tensor_id"]), int(r["start_kernel"]), int(r["end_kernel"]), int(r["wraps"]),
                    {1: "SSD", 2: "CPU"}[int(r["destination"])], [int(r["off_start"]), int(r["off_end"])],
                    [int(r["pre_start"]), int(r["pre_end"])],
                    str((int(r["benefit_hi"]) << 64) | int(r["benefit_lo"])), int(r["cost"]), rel])
    return out


def _check_case(tr, rec):
    periods = [[p.tensor_id, p.size_bytes, p.start_kernel, p.end_kernel, int(p.wraps)]
               for p in compute_inactive_periods(tr)]
    assert periods == rec["periods"]
    assert compute_memory_timeline(tr).per_kernel_bytes == rec["timeline"]
    assert per_kernel_active_bytes(tr) == rec["active"]
    rates = rates_of(rec)
    if "unsat_kernel" in rec:
        with pytest.raises(UnsatisfiableTraceError) as ei:
            plan_device(tr, rec["capacity"], rates, rec["host_cap"])
        assert ei.value.kernel_index == rec["unsat_kernel"]
        return
    raw = plan_device(tr, rec["capacity"], rates, rec["host_cap"])
    assert raw["plan_bytes"].decode() == rec["plan"]
    assert raw["residual"].tolist() == rec["residual"]
    assert _committed_rows(raw) == rec["committed"]


# ---------------------------------------------------------------- golden corpora

@pytest.mark.parametrize("corpus", ["crit2", "crit3", "extreme"])
def test_fuzz_corpus_bit_exact_vs_reference(corpus):
    for rec in load_golden(corpus):
        _check_case(regen(rec), rec)


def test_c1_bit_exact_vs_reference():
    for rec in load_golden("c1"):
        cfg = TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8, seq_len=1024,
                                   bytes_per_element=4, compute_rate=rec["gen"]["compute_rate"], seed=0)
        tr = gen_transformer_trace(cfg)
        _check_case(tr, rec)
        plan = plan_migrations(tr, rec["capacity"], rates_of(rec), rec["host_cap"])
        assert hashlib.sha256(write_plan(plan)).hexdigest() == rec["plan_sha256"]


def test_llama1_bit_exact_vs_reference():
    from paper_2506_06472_b200 import LlamaTraceConfig, gen_llama_trace
    rec = load_golden("llama1")[0]
    tr = gen_llama_trace(LlamaTraceConfig(microbatches=1))
    assert hashlib.sha256(write_trace(tr)).hexdigest() == rec["trace_sha256"]
    _check_case(tr, rec)


def test_c2_lifetime_and_plan_bit_exact_vs_oracle():
    """Config C2 (E=1,001,836): the reference planner would take ~8 h per
    round here, so the checker is the pinned oracle (plan fingerprint in
    tests/golden/c2.json.gz, made by tests/golden/make_c2.py)."""
    from paper_2506_06472_b200 import LLAMA3_8B, gen_llama_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    rec = load_golden("c2")
    tr = gen_llama_trace(LLAMA3_8B)
    a = tr.arrays()
    assert a.num_events == rec["num_events"]
    per, tl, act = O.lifetime(a)
    la = lifetime_arrays(tr)
    assert np.array_equal(la.timeline, tl) and np.array_equal(la.active, act)
    assert np.array_equal(la.period_tensor, per["tensor"])
    assert np.array_equal(la.period_start, per["start"]) and np.array_equal(la.period_end, per["end"])
    assert np.array_equal(la.period_wraps.astype(bool), per["wraps"])
    cap = llama_peak_bytes(tr) // 2
    assert cap == rec["capacity"]
    raw = plan_device(tr, cap, ChannelRates.symmetric(16_000), 0)
    assert hashlib.sha256(raw["plan_bytes"]).hexdigest() == rec["plan_sha256"]
    assert int(raw["info"].num_commits) == rec["num_commits"]
    assert hashlib.sha256(raw["residual"].tobytes()).hexdigest() == rec["residual_sha256"]


def test_random_traces_vs_oracle_wide_fuzz():
    """Wider fuzz than the reference's corpora (bigger traces, fractional
    rates, shuffled / negative ids) against the oracle."""
    import random
    rng = random.Random(99)
    for case in range(120):
        nk = rng.randint(2, 400)
        nt = rng.randint(1, 300)
        tr = gen_random_trace(rng.randint(0, 10**9), nk, nt, size_range=(1_000, 80_000_000),
                              duration_range=(1, 3_000), global_fraction=rng.choice((0.0, 0.3, 0.9)))
        if rng.random() < 0.5:      # arbitrary unique ids, not in trace order
            a = tr.arrays()
            ids = rng.sample(range(-10**12, 10**12), a.num_tensors)
            a.tensor_id[:] = np.array(ids, dtype=np.int64)
            tr.device_cache.clear()
        a = tr.arrays()
        per, tl, act = O.lifetime(a)
        cap = max(int(act.max()), int(tl.max() * rng.choice((0.4, 0.6, 0.8, 0.95))))
        ssd = rng.choice((500.0, 7_777.5, 20_000.0, 123_456.0))
        host = rng.choice((None, ssd * 2.5, 3.0))
        hc = rng.choice((0, 10**8, 10**10)) if host else 0
        rates = ChannelRates.symmetric(ssd, host=host)
        o = O.plan(a, cap, ssd, ssd, host, host, hc, lifetime_out=(per, tl, act))
        g = plan_device(tr, cap, rates, hc)
        assert g["plan_bytes"] == o["plan_bytes"], case
        assert np.array_equal(g["residual"], o["residual"]), case


def test_random_traces_vs_oracle_many_blocks():
    """Larger random traces (hundreds of warp tiles spread over the grid's
    blocks), so refits queued by one block run on others and the owners'
    summaries leave them out for a round; SSD-only and with a host tier."""
    import random
    rng = random.Random(2718)
    for case in range(6):
        nk = rng.randint(2_000, 6_000)
        nt = rng.randint(3_000, 9_000)
        tr = gen_random_trace(rng.randint(0, 10**9), nk, nt, size_range=(1_000_000, 400_000_000),
                              duration_range=(10, 5_000), global_fraction=rng.choice((0.05, 0.3)))
        a = tr.arrays()
        per, tl, act = O.lifetime(a)
        cap = max(int(act.max()), int(tl.max() * rng.choice((0.5, 0.7))))
        ssd = rng.choice((20_000.0, 60_000.0))
        host = None if case % 2 == 0 else ssd * 2.0
        hc = 10**11 if host else 0
        rates = ChannelRates.symmetric(ssd, host=host)
        o = O.plan(a, cap, ssd, ssd, host, host, hc, lifetime_out=(per, tl, act), max_rounds=400)
        g = plan_device(tr, cap, rates, hc, max_rounds=400)
        assert len(o["committed"]) > 20, case
        assert g["plan_bytes"] == o["plan_bytes"], case
        assert np.array_equal(g["residual"], o["residual"]), case


# ---------------------------------------------------------------- known answers
# reference tests/test_analysis.py:18-69 and test_planner.py:108-234

def test_ex1_known_answers(ex1, rates20k):
    assert compute_inactive_periods(ex1) == [InactivePeriod(0, MB100, 1, 3, False)]
    assert compute_memory_timeline(ex1).per_kernel_bytes == [MB100, MB100, 2 * MB100, MB100, MB100]
    plan = plan_migrations(ex1, CAP, rates20k)
    assert plan.entries == [PlanEntry(0, "offload", 10_000, 15_000, "SSD", False),
                            PlanEntry(0, "prefetch", 35_000, 40_000, "GPU", True)]
    assert plan.residual_timeline.per_kernel_bytes == [MB100] * 5
    assert not plan.warning and plan.planned_host_bytes == 0
    c = plan.committed[0]
    assert (c.benefit, c.cost, c.relieved_kernels) == (10**12, 10_000, (2,))
    assert write_plan(plan) == (
        b'{"version": 1, "capacity_bytes": 150000000, "residual_peak_bytes": 100000000, '
        b'"planned_host_bytes": 0, "over_capacity_kernels": []}\n'
        b'{"tensor": 0, "action": "offload", "trigger_us": 10000, "deadline_us": 15000, '
        b'"target": "SSD", "urgent": false}\n'
        b'{"tensor": 0, "action": "prefetch", "trigger_us": 35000, "deadline_us": 40000, '
        b'"target": "GPU", "urgent": true}\n')


def test_global_wrap_periods():
    assert compute_inactive_periods(mk_trace([10] * 5, [(0, 7, "global", [0])])) == [
        InactivePeriod(0, 7, 1, 4, True)]
    assert compute_inactive_periods(mk_trace([10] * 5, [(0, 7, "global", [1, 2])])) == [
        InactivePeriod(0, 7, 3, 0, True)]
    assert compute_inactive_periods(mk_trace([10, 10], [(0, 5, "global", [0, 1])])) == []
    assert compute_inactive_periods(mk_trace([10, 10], [(0, 5, "intermediate", [0, 1])])) == []
    assert compute_memory_timeline(mk_trace([1, 1, 1], [(0, 7, "global", [1])])).per_kernel_bytes == [7, 7, 7]


def test_empty_trace():
    tr = mk_trace([], [])
    assert compute_memory_timeline(tr).per_kernel_bytes == []
    assert compute_inactive_periods(tr) == []
    plan = plan_migrations(tr, 100, ChannelRates.symmetric(10))
    assert plan.entries == [] and not plan.warning


def test_kernels_without_tensors():
    tr = mk_trace([5, 6, 7], [])
    assert compute_memory_timeline(tr).per_kernel_bytes == [0, 0, 0]
    assert plan_migrations(tr, 0, ChannelRates.symmetric(10)).entries == []


def test_no_pressure_infeasible_unsat(ex1, rates20k):
    assert plan_migrations(ex1, 250_000_000, rates20k).entries == []
    p = plan_migrations(ex1, CAP, ChannelRates.symmetric(1_000))
    assert p.entries == [] and p.warning and p.over_capacity_kernels == [2]
    with pytest.raises(UnsatisfiableTraceError, match="kernel 0"):
        plan_migrations(ex1, 90_000_000, rates20k)


def test_bad_rate_raises_channel_config_error(ex1):
    with pytest.raises(ChannelConfigError):
        plan_migrations(ex1, CAP, ChannelRates.symmetric(0))
    with pytest.raises(ChannelConfigError):
        plan_migrations(ex1, CAP, ChannelRates(20_000, 20_000, -1, 5))


def test_mark_urgent_zero_slack_only():
    tr = mk_trace([10_000] * 5, [(0, MB100, "intermediate", [0, 4]), (1, MB100, "intermediate", [0, 4]),
                                 (2, 220_000_000, "intermediate", [2])])
    plan = plan_migrations(tr, 230_000_000, ChannelRates.symmetric(20_000))
    pre = {e.tensor_id: e for e in plan.entries if e.action == "prefetch"}
    assert pre[0].deadline == 40_000 and pre[0].urgent
    assert pre[1].deadline == 35_000 and not pre[1].urgent
    assert mark_urgent(plan, tr).entries == plan.entries


def test_host_destination_and_cap(ex1):
    rates = ChannelRates(1, 1, 20_000, 20_000)
    plan = plan_migrations(ex1, CAP, rates, host_cap=MB100)
    assert [e.target for e in plan.entries] == ["CPU", "GPU"]
    assert plan.planned_host_bytes == MB100
    starved = plan_migrations(ex1, CAP, rates, host_cap=MB100 - 1)
    assert starved.entries == [] and starved.warning


def test_wrap_period_global_plan():
    tr = mk_trace([10_000] * 5, [(0, MB100, "global", [1]), (1, MB100, "intermediate", [3])])
    plan = plan_migrations(tr, CAP, ChannelRates.symmetric(20_000))
    assert plan.residual_timeline.per_kernel_bytes == [MB100, MB100, MB100, MB100, 0]
    off = [e for e in plan.entries if e.action == "offload"][0]
    pre = [e for e in plan.entries if e.action == "prefetch"][0]
    assert (off.trigger_time, off.deadline) == (20_000, 25_000)
    assert (pre.trigger_time, pre.deadline) == (55_000, 60_000) and pre.urgent


def test_invalid_trace_is_rejected():
    from paper_2506_06472_b200 import KernelRecord, TensorKind, TensorRecord, Trace
    bad = Trace([KernelRecord(0, "k", 5)], [TensorRecord(0, 10, TensorKind.INTERMEDIATE, (3,))])
    with pytest.raises(Exception):
        plan_migrations(bad, 100, ChannelRates.symmetric(10))
    # duplicate ids pass straight to the device (no host validation): the
    # library must refuse them (reference trace.py:136-141 invariant)
    dup = Trace([KernelRecord(i, f"k{i}", 5) for i in range(3)],
                [TensorRecord(4, 10, TensorKind.INTERMEDIATE, (0, 2)),
                 TensorRecord(4, 10, TensorKind.INTERMEDIATE, (0, 2))])
    with pytest.raises(_native.TioError, match="duplicate"):
        plan_migrations(dup, 15, ChannelRates.symmetric(10))


def test_native_library_is_the_code_that_ran():
    import os
    info = _native.device_info()
    assert "sm_100a" in info
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert _native.lib_path() in maps


def test_c3_full_plan_bit_exact_vs_oracle():
    """Config C3 (Llama-3-70B shape, E=9,935,960), the north star's 10M-event
    trace: the whole plan (1,347 commits) against the oracle's fingerprint
    (tests/golden/c3.json.gz, tests/golden/make_c2.py c3: 493 s on 8 cores)."""
    from paper_2506_06472_b200 import LLAMA3_70B, gen_llama_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    rec = load_golden("c3")
    tr = gen_llama_trace(LLAMA3_70B)
    assert tr.arrays().num_events == rec["num_events"]
    cap = llama_peak_bytes(tr) // 2
    assert cap == rec["capacity"]
    raw = plan_device(tr, cap, ChannelRates.symmetric(16_000), 0)
    assert hashlib.sha256(raw["plan_bytes"]).hexdigest() == rec["plan_sha256"]
    assert int(raw["info"].num_commits) == rec["num_commits"]
    assert hashlib.sha256(raw["residual"].tobytes()).hexdigest() == rec["residual_sha256"]


def test_c3_lifetime_and_plan_prefix_vs_oracle():
    """Config C3 (Llama-3-70B shape, E=9,935,960): lifetime bit-exact against
    the oracle; the planner's first 24 commits (max_rounds) against the
    oracle's first 24 — a prefix of the same greedy sequence."""
    from paper_2506_06472_b200 import LLAMA3_70B, gen_llama_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    tr = gen_llama_trace(LLAMA3_70B)
    a = tr.arrays()
    assert a.num_events == 9_935_960
    per, tl, act = O.lifetime(a)
    la = lifetime_arrays(tr)
    assert np.array_equal(la.timeline, tl) and np.array_equal(la.active, act)
    assert np.array_equal(la.period_tensor, per["tensor"]) and np.array_equal(la.period_start, per["start"])
    assert np.array_equal(la.period_end, per["end"])
    cap = llama_peak_bytes(tr) // 2
    R = 24
    o = O.plan(a, cap, 16000.0, 16000.0, lifetime_out=(per, tl, act), max_rounds=R)
    g = plan_device(tr, cap, ChannelRates.symmetric(16_000), 0, max_rounds=R)
    assert int(g["info"].num_commits) == len(o["committed"]) == R
    assert g["plan_bytes"] == o["plan_bytes"]
    assert np.array_equal(g["residual"], o["residual"])


def test_criterion_6_characterization_regime():
    """Reference test_acceptance.py:181-188: the default transformer trace at
    half its peak is a capacity problem, not an active-bytes one."""
    from paper_2506_06472_b200 import TransformerGenConfig, gen_transformer_trace
    from paper_2506_06472_b200.analysis import characterize
    tr = gen_transformer_trace(TransformerGenConfig())
    demand = compute_memory_timeline(tr).peak()
    report = characterize(tr, demand // 2)
    assert report.max_active_fraction < 0.15


def test_characterization_known_answers(ex1):
    """Reference test_analysis.py:37-41 (wrap interior) and :72-101
    (characterize, CSV shapes) over the device lifetime columns."""
    from paper_2506_06472_b200.analysis import (characterize, fractions_csv, histogram_csv,
                                                period_interior_duration)
    wrap = mk_trace([10] * 5, [(0, 7, "global", [1, 2])])
    assert period_interior_duration(compute_inactive_periods(wrap)[0], wrap) == 30   # k3, k4, k0
    rep = characterize(ex1, capacity=150_000_000, size_buckets=(10_000_000, 1_000_000_000),
                       duration_buckets=(1_000, 100_000))
    third = 100_000_000 / 150_000_000
    assert rep.active_fraction == [third, 0.0, third, 0.0, third]
    assert rep.histogram == {("[10000000,1000000000)", "[1000,100000)"): 1}
    assert rep.total_periods == 1 and rep.max_active_fraction == pytest.approx(third)
    empty = characterize(mk_trace([], []), capacity=100)
    assert empty.active_bytes == [] and empty.histogram == {} and empty.mean_active_fraction == 0.0
    with pytest.raises(ValueError):
        characterize(ex1, capacity=0)
    rep = characterize(ex1, capacity=150_000_000)
    assert fractions_csv(rep).splitlines()[0] == "kernel,active_bytes,active_fraction"
    assert len(fractions_csv(rep).splitlines()) == 6
    assert histogram_csv(rep).splitlines()[0] == "size_class_bytes,duration_class_us,count"


def test_period_interior_durations_on_device():
    """period_interior_duration (reference analysis.py:86-94) of every period
    from the device kernel (tio_period_interior) equals the one-period host
    restatement on wrap edge cases (last access in the last kernel, first in
    kernel 0, single-access globals), random traces and the C1 trace."""
    import numpy as np
    from paper_2506_06472_b200 import TransformerGenConfig, gen_random_trace, gen_transformer_trace
    from paper_2506_06472_b200.analysis import period_interior_duration, period_interior_durations
    cases = [mk_trace([10, 20, 30, 40, 50], [(0, 7, "global", [1, 2])]),
             mk_trace([10, 20, 30, 40, 50], [(0, 7, "global", [0, 4]), (1, 5, "global", [4]),
                                             (2, 6, "global", [0]), (3, 9, "intermediate", [0, 3])]),
             gen_transformer_trace(TransformerGenConfig(num_layers=2))]
    cases += [gen_random_trace(s, 20 + s, 15 + s % 9) for s in range(20)]
    n = 0
    for tr in cases:
        dev = period_interior_durations(tr)
        per = compute_inactive_periods(tr)
        assert dev.tolist() == [period_interior_duration(p, tr) for p in per]
        n += len(per)
    assert n > 500


@pytest.mark.parametrize("config", ["c2", "c3"])
def test_lifetime_vs_reference_itself_at_scale(config):
    """C2 (1.0M events) and C3 (9.9M events) lifetime products against the
    REFERENCE's own outputs (tests/golden/make_ref_lifetime.py ran
    compute_inactive_periods / compute_memory_timeline / per_kernel_active_bytes
    of /root/reference on the same trace: 237 s at C3), as sha256 of the
    int64 rows (tensor_id, size, start, end, wraps), timeline and active bytes."""
    import json
    import os
    from paper_2506_06472_b200 import LLAMA3_8B, LLAMA3_70B, gen_llama_trace
    path = os.path.join(os.path.dirname(__file__), "golden", f"{config}_lifetime_ref.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    with open(path) as f:
        rec = json.load(f)
    tr = gen_llama_trace({"c2": LLAMA3_8B, "c3": LLAMA3_70B}[config])
    a = tr.arrays()
    assert a.num_events == rec["num_events"]
    la = lifetime_arrays(tr)
    rows = np.stack([a.tensor_id[la.period_tensor], a.size_bytes[la.period_tensor], la.period_start.astype(np.int64),
                     la.period_end.astype(np.int64), la.period_wraps.astype(np.int64)], axis=1)
    h = lambda x: hashlib.sha256(np.ascontiguousarray(x, dtype="<i8").tobytes()).hexdigest()  # noqa: E731
    assert rows.shape[0] == rec["num_periods"]
    assert h(rows) == rec["periods_sha256"]
    assert h(la.timeline) == rec["timeline_sha256"]
    assert h(la.active) == rec["active_sha256"]


def test_c2_host_tier_plan_prefix_vs_oracle():
    """Config C2 with the host tier of SURVEY §8(d) (host 50,000 B/us both
    ways, host_cap 256e9): the first 700 commits of the device plan against
    the oracle's first 700 — a prefix of the same greedy sequence; from commit
    576 on the SSD channels are saturated and candidates fall back to the host
    with the host-cap occupancy test live (124 host commits here; the oracle's
    host-tier rounds cost ~0.4 s each, so its full 32k-round plan is out of
    reach)."""
    from paper_2506_06472_b200 import LLAMA3_8B, gen_llama_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    tr = gen_llama_trace(LLAMA3_8B)
    a = tr.arrays()
    cap = llama_peak_bytes(tr) // 2
    R = 700
    o = O.plan(a, cap, 16000.0, 16000.0, 50000.0, 50000.0, 256 * 10**9, max_rounds=R)
    g = plan_device(tr, cap, ChannelRates.symmetric(16_000, host=50_000), 256 * 10**9, max_rounds=R)
    assert int(g["info"].num_commits) == len(o["committed"]) == R
    assert sum(1 for c in o["committed"] if c[4] == "CPU") >= 100       # the host tier is exercised
    assert g["plan_bytes"] == o["plan_bytes"]
    assert np.array_equal(g["residual"], o["residual"])


def test_c2_host_tier_full_plan_vs_oracle_fingerprint():
    """Config C2 with the host tier of SURVEY §8(d) (host 50,000 B/us both
    ways, host_cap 256e9), the WHOLE plan (18,756 commits, 11,843 of them to
    the host under the live host-cap test): plan bytes, residual timeline and
    planned host bytes against the oracle's fingerprint
    (tests/golden/c2host.json.gz, tests/golden/make_c2.py c2host: 374 s on 8
    cores)."""
    import gzip
    import json
    import os
    from conftest import ROOT
    from paper_2506_06472_b200 import LLAMA3_8B, gen_llama_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    path = os.path.join(ROOT, "tests", "golden", "c2host.json.gz")
    if not os.path.exists(path):
        pytest.skip("c2host fingerprint not generated")
    with gzip.open(path, "rt") as f:
        rec = json.load(f)
    tr = gen_llama_trace(LLAMA3_8B)
    cap = llama_peak_bytes(tr) // 2
    assert cap == rec["capacity"]
    g = plan_device(tr, cap, ChannelRates.symmetric(16_000, host=50_000), rec["host_cap"])
    assert int(g["info"].num_commits) == rec["num_commits"]
    assert hashlib.sha256(g["plan_bytes"]).hexdigest() == rec["plan_sha256"]
    assert hashlib.sha256(g["residual"].astype("<i8").tobytes()).hexdigest() == rec["residual_sha256"]
    assert int(g["info"].planned_host_bytes) == rec["planned_host_bytes"]


def test_c3_host_tier_plan_prefix_vs_oracle_fingerprint():
    """Config C3 (9.9M events) with the host tier of SURVEY §8(d) (host 50,000
    B/us both ways, host_cap 256e9): the first 1,700 commits of the device plan
    against the oracle's (tests/golden/c3host_prefix1700.json.gz,
    tests/golden/make_c2.py c3host 1700: 718 s on 8 cores) — plan bytes,
    residual timeline and planned host bytes.  669 of the 1,700 commits go to
    the host under the live host-cap test, at the 10M-event scale (the whole
    C3 host-tier plan, ~52k rounds, is out of the oracle's reach)."""
    import gzip
    import json
    import os
    from conftest import ROOT
    from paper_2506_06472_b200 import LLAMA3_70B, gen_llama_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    with gzip.open(os.path.join(ROOT, "tests", "golden", "c3host_prefix1700.json.gz"), "rt") as f:
        rec = json.load(f)
    tr = gen_llama_trace(LLAMA3_70B)
    cap = llama_peak_bytes(tr) // 2
    assert cap == rec["capacity"]
    R = rec["max_rounds"]
    g = plan_device(tr, cap, ChannelRates.symmetric(16_000, host=50_000), rec["host_cap"], max_rounds=R)
    assert int(g["info"].num_commits) == rec["num_commits"] == R
    assert rec["host_commits"] >= 600                                   # the host tier is exercised
    assert hashlib.sha256(g["plan_bytes"]).hexdigest() == rec["plan_sha256"]
    assert hashlib.sha256(g["residual"].astype("<i8").tobytes()).hexdigest() == rec["residual_sha256"]
    assert int(g["info"].planned_host_bytes) == rec["planned_host_bytes"]


def test_c3_host_tier_full_plan_vs_oracle_fingerprint():
    """Config C3 (9.9M events) with the host tier of SURVEY §8(d): the whole
    plan against the oracle's fingerprint (tests/golden/c3host.json.gz,
    tests/golden/make_c2.py c3host)."""
    import gzip
    import json
    import os
    from conftest import ROOT
    from paper_2506_06472_b200 import LLAMA3_70B, gen_llama_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    path = os.path.join(ROOT, "tests", "golden", "c3host.json.gz")
    if not os.path.exists(path):
        pytest.skip("c3host fingerprint not generated")
    with gzip.open(path, "rt") as f:
        rec = json.load(f)
    tr = gen_llama_trace(LLAMA3_70B)
    cap = llama_peak_bytes(tr) // 2
    assert cap == rec["capacity"]
    g = plan_device(tr, cap, ChannelRates.symmetric(16_000, host=50_000), rec["host_cap"])
    assert int(g["info"].num_commits) == rec["num_commits"]
    assert hashlib.sha256(g["plan_bytes"]).hexdigest() == rec["plan_sha256"]
    assert hashlib.sha256(g["residual"].astype("<i8").tobytes()).hexdigest() == rec["residual_sha256"]
    assert int(g["info"].planned_host_bytes) == rec["planned_host_bytes"]
