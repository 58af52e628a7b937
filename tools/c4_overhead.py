"""Cost of the online engine's per-operator hook on the C4 step, with NO
transfers (plan at capacity 10x the peak: zero entries): step time vs the
plain step, with and without the per-operator divergence check, plus the
host time per step.  python tools/c4_overhead.py [8b|tiny]"""
import dataclasses
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")


def main():
    import torch
    from paper_2506_06472_b200 import ChannelRates, compute_memory_timeline, engine, plan_migrations
    from paper_2506_06472_b200.llama_step import LLAMA3_8B_MODEL, TINY, Step
    from paper_2506_06472_b200.profiler import profile_step
    cfg = dataclasses.replace(LLAMA3_8B_MODEL if "8b" in sys.argv else TINY, deterministic=False)
    s = Step(cfg, seed=0)
    for _ in range(2):
        s()
    stream = torch.cuda.current_stream()

    def timed(n, mode=None):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0 = time.perf_counter()
        e0.record(stream)
        for _ in range(n):
            if mode is None:
                s()
            else:
                with mode.step():
                    s()
        e1.record(stream)
        c1 = time.perf_counter()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n, (c1 - c0) * 1e3 / n

    ideal = timed(3)
    tr = profile_step(s, globals_=s.globals_of())
    cap = compute_memory_timeline(tr).peak() * 10
    rates = ChannelRates.symmetric(50_000.0)
    plan = plan_migrations(tr, cap, rates)
    out = {"kernels": tr.arrays().num_kernels, "plan_entries": len(plan.entries),
           "plain": {"step_ms": ideal[0], "host_ms": ideal[1]}}
    for check in (True, False):
        mode = engine.OffloadMode(tr, plan, cap, rates, s.globals_of(), check=check)
        with mode.step():
            s()
        r = timed(3, mode)
        mode.close()
        out[f"hook_check_{check}"] = {"step_ms": r[0], "host_ms": r[1], "vs_plain": r[0] / ideal[0]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
