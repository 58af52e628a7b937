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
