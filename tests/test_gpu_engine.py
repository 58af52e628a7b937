"""GPU: the migration engine executor (csrc/engine.cu) and its TMA copy
kernels.  Offloaded tensors must come back byte-identical; the executor's
decisions must be the reference engine's (model totals == the reference
simulate() golden values)."""

from __future__ import annotations

import pytest

from conftest import load_golden, mk_trace, regen, rates_of
from paper_2506_06472_b200 import ChannelRates, PlanEntry, simulate
from paper_2506_06472_b200 import engine
from paper_2506_06472_b200.planner import parse_plan

pytestmark = pytest.mark.gpu

MB100 = 100_000_000


def test_pack_unpack_round_trip_byte_identical():
    import torch
    g = torch.Generator(device="cuda").manual_seed(0)
    sizes = [1, 15, 16, 17, 4095, 4096, 4097, 32 * 1024, 32 * 1024 + 3, 3 * 32 * 1024 - 5, 10_000_019, 64 << 20]
    base = torch.randint(0, 256, (sum(sizes) + 64 * len(sizes),), dtype=torch.uint8, device="cuda", generator=g)
    srcs, off = [], 0
    for i, n in enumerate(sizes):
        off += i % 3            # deliberately misaligned views for some segments
        srcs.append(base[off:off + n])
        off += n
    staging = torch.zeros(sum((n + 4095) // 4096 * 4096 for n in sizes), dtype=torch.uint8, device="cuda")
    offs = engine.pack(srcs, staging)
    assert all(o % 4096 == 0 for o in offs)
    outs = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes]
    engine.unpack(staging, offs, outs)
    torch.cuda.synchronize()
    for s, o, b in zip(srcs, outs, offs):
        assert torch.equal(s, o)
        assert torch.equal(staging[b:b + s.numel()], s)


def test_replay_ex1_round_trip_and_model(ex1, rates20k):
    plan = [PlanEntry(0, "offload", 10_000, 15_000, "SSD", False),
            PlanEntry(0, "prefetch", 35_000, 40_000, "GPU", True)]
    r = engine.replay(ex1, plan, 150_000_000, rates20k, time_scale=0.05)
    assert r.model_total_us == 50_000 and r.model_stall_us == 0
    assert r.n_offloads == 1 and r.n_prefetches == 1
    assert r.offload_bytes == MB100 and r.prefetch_bytes == MB100
    assert r.verified_bytes == MB100 and r.verify_mismatches == 0
    assert r.replay_ms > 0 and r.ideal_ms > 0


def test_replay_on_demand_emergency_round_trip(ex1, rates20k):
    r = engine.replay(ex1, [], 150_000_000, rates20k, time_scale=0.05)
    assert r.emergency_offloads == 1
    assert r.model_total_us == 60_000
    assert r.verify_mismatches == 0 and r.verified_bytes == MB100


def test_replay_wrap_plan_folded_state():
    tr = mk_trace([10_000] * 5, [(0, MB100, "global", [1]), (1, MB100, "intermediate", [3])])
    plan = [PlanEntry(0, "offload", 20_000, 25_000, "SSD", False),
            PlanEntry(0, "prefetch", 55_000, 60_000, "GPU", True)]
    r = engine.replay(tr, plan, 150_000_000, ChannelRates.symmetric(20_000), time_scale=0.05)
    assert r.model_total_us == 50_000 and r.verify_mismatches == 0


def test_replay_matches_reference_engine_on_corpus():
    sims = [r for r in load_golden("sim") if r["corpus"] == "crit2"]   # real bytes move: no PB tensors
    plans = {r["trace_sha256"]: r for r in load_golden("crit2")}
    done = 0
    for rec in sims[:60]:
        base = plans[rec["trace_sha256"]]
        if "plan" not in base or "error" in rec["plan"]:
            continue
        tr = regen(rec)
        entries = parse_plan(base["plan"])[1]
        r = engine.replay(tr, entries, base["capacity"], rates_of(base), time_scale=0.002)
        assert r.model_total_us == rec["plan"]["total_time"]
        assert r.model_stall_us == rec["plan"]["stall_time_total"]
        assert r.emergency_offloads == rec["plan"]["emergency_offloads"]
        assert r.verify_mismatches == 0
        assert r.verified_bytes == r.prefetch_bytes
        done += 1
    assert done >= 30
