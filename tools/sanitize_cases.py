"""Small workloads for compute-sanitizer: every libtio kernel
family on inputs small enough for memcheck / racecheck / synccheck.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py lifetime_plan
    cases: lifetime_plan | virtual | replay | online

lifetime_plan  lifetime kernels + the persistent planner (SSD and host tier)
               on random traces and C1, checked against the oracle
virtual        the sharded planner, 2 virtual ranks exchanging through device
               mailboxes (the grid-wide winner publication + mailbox flags)
replay         the migration executor (tio_engine_replay) on a small trace
online         the online engine under a tiny Llama step (OffloadMode)
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lifetime_plan():
    import numpy as np
    from oracle import oracle as O
    from paper_2506_06472_b200 import ChannelRates, gen_random_trace, lifetime_arrays, plan_device
    n = 0
    for seed in (3, 17):
        tr = gen_random_trace(seed, 30, 28, size_range=(1_000_000, 50_000_000), duration_range=(100, 3_000))
        a = tr.arrays()
        per, tl, act = O.lifetime(a)
        la = lifetime_arrays(tr)
        assert np.array_equal(la.timeline, tl) and np.array_equal(la.active, act)
        cap = max(int(act.max()), int(tl.max() * 0.6))
        for rates, hc in ((ChannelRates.symmetric(8_000), 0), (ChannelRates.symmetric(2_000, host=6_000), 10**9)):
            o = O.plan(a, cap, rates.ssd_offload, rates.ssd_prefetch, rates.host_offload, rates.host_prefetch, hc,
                       lifetime_out=(per, tl, act))
            g = plan_device(tr, cap, rates, hc)
            assert g["plan_bytes"] == o["plan_bytes"]
            n += 1
    print("lifetime_plan ok", n)


def virtual():
    from paper_2506_06472_b200 import ChannelRates, compute_memory_timeline, gen_random_trace, plan_device
    from paper_2506_06472_b200.planner import plan_device_virtual
    tr = gen_random_trace(5, 30, 28, size_range=(1_000_000, 50_000_000), duration_range=(100, 3_000))
    cap = int(compute_memory_timeline(tr).peak() * 0.6)
    rates = ChannelRates.symmetric(4_000)
    one = plan_device(tr, cap, rates, 0)
    outs = plan_device_virtual(tr, cap, rates, 0, 2)
    assert all(o["plan_bytes"] == one["plan_bytes"] for o in outs)
    print("virtual ok")


def replay():
    from paper_2506_06472_b200 import ChannelRates, compute_memory_timeline, gen_random_trace, plan_migrations
    from paper_2506_06472_b200 import engine
    tr = gen_random_trace(11, 24, 20, size_range=(1 << 20, 16 << 20), duration_range=(200, 2_000))
    cap = int(compute_memory_timeline(tr).peak() * 0.6)
    rates = ChannelRates.symmetric(20_000)
    plan = plan_migrations(tr, cap, rates)
    r = engine.replay(tr, plan, cap, rates, verify=True)
    assert r.verify_mismatches == 0
    print("replay ok", r.n_offloads, r.n_prefetches)


def online():
    import torch
    from paper_2506_06472_b200 import ChannelRates, compute_memory_timeline, plan_migrations
    from paper_2506_06472_b200.engine import OffloadMode
    from paper_2506_06472_b200.llama_step import LlamaConfig, Step
    from paper_2506_06472_b200.profiler import profile_step
    cfg = LlamaConfig(vocab=512, dim=128, layers=1, heads=4, kv_heads=2, ffn=256, seq=64)
    s = Step(cfg, seed=0)
    s()
    tr = profile_step(s, globals_=s.globals_of())
    cap = int(compute_memory_timeline(tr).peak() * 0.7)
    rates = ChannelRates.symmetric(20_000.0)
    mode = OffloadMode(tr, plan_migrations(tr, cap, rates), cap, rates, s.globals_of(), verify=True)
    for _ in range(2):
        with mode.step():
            s()
    torch.cuda.synchronize()
    st = mode.stats()
    mode.close()
    assert st["verify_mismatches"] == 0
    print("online ok", st["offload_bytes"], st["prefetch_bytes"])


if __name__ == "__main__":
    {"lifetime_plan": lifetime_plan, "virtual": virtual, "replay": replay, "online": online}[sys.argv[1]]()
