"""The engine program (the scheduler's output the GPU executor runs) is
consistent: replayed in the engine's processing order, every offload finds
its tensor resident, every prefetch finds it off the GPU, every kernel finds
its tensors resident or allocates a fresh intermediate, on the criterion-2
corpus with the reference's plans.  Host-only (no GPU)."""

from __future__ import annotations

import numpy as np

from conftest import load_golden, rates_of, regen
from paper_2506_06472_b200.planner import parse_plan
from paper_2506_06472_b200.simulator import schedule


def _check(tr, xs, starts, kseq, loc):
    a = tr.arrays()
    N, T = a.num_kernels, a.num_tensors
    acc = [a.accesses[a.access_ptr[t]:a.access_ptr[t + 1]].tolist() for t in range(T)]
    act = [[] for _ in range(N)]
    for t in range(T):
        for k in acc[t]:
            act[k].append(t)
    ops = sorted([(int(x["seq"]), 0, j) for j, x in enumerate(xs)] + [(int(kseq[k]), 1, k) for k in range(N)])
    assert len({o[0] for o in ops}) == len(ops), "processing positions are unique"
    res = (loc == 1).copy()
    moved = np.zeros(T, bool)
    for _, kind, j in ops:
        if kind == 0:
            t = int(xs[j]["tensor_pos"])
            if xs[j]["action"] == 0:
                assert res[t], f"offload of non-resident tensor {t}"
                res[t] = False
            else:
                assert not res[t], f"prefetch of resident tensor {t}"
                res[t] = True
            moved[t] = True
        else:
            for t in act[j]:
                if not res[t]:
                    assert a.kind[t] != 1 and not moved[t], f"kernel {j} needs tensor {t} off the GPU"
                    res[t] = True
            for t in act[j]:
                if a.kind[t] != 1 and acc[t][-1] == j:
                    res[t] = False


def test_engine_program_consistent_on_corpus():
    sims = load_golden("sim")
    plans = {r["trace_sha256"]: r for r in load_golden("crit2") + load_golden("extreme")}
    n = 0
    for rec in sims:
        base = plans[rec["trace_sha256"]]
        tr = regen(rec)
        for entries in ((parse_plan(base["plan"])[1] if "plan" in base else None), []):
            if entries is None:
                continue
            key = "plan" if entries else "on_demand"
            if "error" in rec[key]:
                continue
            xs, starts, kseq, loc = schedule(tr, entries, base["capacity"], rates_of(base))
            _check(tr, xs, starts, kseq, loc)
            n += 1
    assert n >= 1500


def test_online_engine_program_holds_over_consecutive_steps():
    """The online engine (csrc/engine_online.cu) walked for 3 consecutive
    steps without a device (tio_engine_check_program): steady-state folding,
    boundary-straddling transfers handed from one step to the next, emergency
    evictions — every offload finds its tensor resident, every prefetch finds
    it gone, every kernel finds its tensors on the GPU."""
    from paper_2506_06472_b200.engine import check_program
    sims = load_golden("sim")
    plans = {r["trace_sha256"]: r for r in load_golden("crit2") + load_golden("extreme")}
    n = 0
    for rec in sims:
        base = plans[rec["trace_sha256"]]
        tr = regen(rec)
        for entries in ((parse_plan(base["plan"])[1] if "plan" in base else None), []):
            if entries is None:
                continue
            key = "plan" if entries else "on_demand"
            if "error" in rec[key]:
                continue
            check_program(tr, entries, base["capacity"], rates_of(base), steps=3)
            n += 1
    assert n >= 1500


def test_online_engine_program_on_llama_traces_with_oracle_plans():
    """Appendix-C Llama-3-8B traces (1 and 4 microbatches) planned by the
    oracle at tight capacities: the plans have wrap periods of globals, folded
    prefetches and straddling transfers; 3 steps of the online program."""
    from oracle import oracle as O
    from paper_2506_06472_b200 import ChannelRates, PlanEntry
    from paper_2506_06472_b200 import tracegen as G
    from paper_2506_06472_b200.engine import check_program
    for mb, frac, rate in ((1, 0.5, 16_000.0), (1, 0.7, 50_000.0), (4, 0.5, 50_000.0), (4, 0.8, 50_000.0)):
        tr = G.gen_llama_trace(G.LlamaTraceConfig(microbatches=mb))
        a = tr.arrays()
        cap = int(G.llama_peak_bytes(tr) * frac)
        p = O.plan(a, cap, rate, rate)
        entries = [PlanEntry(tid, act, trig, dl, tgt, urg) for tid, act, trig, dl, tgt, urg in p["entries"]]
        info = check_program(tr, entries, cap, ChannelRates.symmetric(rate), steps=3)
        assert info["num_transfers"] > 0
