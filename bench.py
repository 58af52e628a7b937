"""Benchmark of the lifetime + plan hot path (BASELINE.json metric 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c2|c1|llama1] [--secondary c2|...|""]

One step = one pass of the hot path over the trace: the lifetime stage
(reference analysis.py:58-117) and the Algorithm-1 planner with entry sort
and mark_urgent (planner.py:267-397) on a device-resident trace.

Workloads: the headline line is config C3 (BASELINE.json configs[2]: the
north star's 10M-event Llama-3-70B-shaped trace, which fits one B200); the
same measurement on C2 (configs[1], 1M events) is reported under the "c2"
key.  Both plans are bit-exact with the oracle fingerprints in tests/golden.

  value  = trace events / s = E / (device time of lifetime + plan), CUDA
           events on the libtio stream, L2 flushed (256 MiB write) before every
           step outside the timed region; summed over K steps.
  e2e    = the same metric through the C-ABI one-shot call tio_plan_host with
           pinned HOST trace columns in and host plan entries out (H2D + D2H
           inside the timed region).
  roofline        the lifetime kernel (HBM-bound, SURVEY §8d B_L bytes).
  planner         the round-loop kernel: latency-bound, reported as us/round.
  cpu_baseline    the CPU oracle port (oracle/tio_oracle.c, OpenMP) on this
                  host: full lifetime stage + the first R planner rounds over
                  the same trace, extrapolated linearly to all rounds.

--impl reference times that CPU path (the reference's algorithm; the Python
reference itself cannot run here: ~8 h per planner round at C2)
over one FULL lifetime + plan of the trace (measured, with its plan sha256)
and prints its own JSON line.

Multi-GPU (torchrun, one process per GPU): strong scaling of the SAME trace —
every rank runs the lifetime stage and the sharded planner
(distributed.PlanGroup: candidate tiles split over the ranks, replicated
planner state, each round's local bests exchanged through CUDA-IPC mailboxes
over NVLink), so value = E / (max over ranks of the device time), and the
line reports whether every rank's plan sha256 is the same.  The C4 leg runs
at N = 1 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0


def _peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def _trace(config: str):
    from paper_2506_06472_b200 import tracegen as G
    from paper_2506_06472_b200 import ChannelRates, TransformerGenConfig
    if config == "c2":
        tr = G.gen_llama_trace(G.LLAMA3_8B)
        cap = G.llama_peak_bytes(tr) // 2
        return tr, cap, ChannelRates.symmetric(16_000), 0, "C2 Llama-3-8B-shaped trace (Appendix C, 292 microbatches)"
    if config in ("c2host", "c3host"):
        tr = G.gen_llama_trace(G.LLAMA3_8B if config == "c2host" else G.LLAMA3_70B)
        cap = G.llama_peak_bytes(tr) // 2
        return tr, cap, ChannelRates.symmetric(16_000, host=50_000), 256 * 10**9, \
            f"{config[:2].upper()} trace with the host tier (SURVEY 8d: host 50,000 B/us, host_cap 256e9)"
    if config == "c3":
        tr = G.gen_llama_trace(G.LLAMA3_70B)
        cap = G.llama_peak_bytes(tr) // 2
        return tr, cap, ChannelRates.symmetric(16_000), 0, "C3 Llama-3-70B-shaped trace (Appendix C, 1160 microbatches)"
    if config == "llama1":
        tr = G.gen_llama_trace(G.LlamaTraceConfig(microbatches=1))
        cap = G.llama_peak_bytes(tr) // 2
        return tr, cap, ChannelRates.symmetric(16_000), 0, "Llama-3-8B-shaped trace, 1 microbatch"
    if config == "c1":
        tr = G.gen_transformer_trace(TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8,
                                                          seq_len=1024, bytes_per_element=4,
                                                          compute_rate=1_000_000_000, seed=0))
        cap = G.llama_peak_bytes(tr) // 2
        return tr, cap, ChannelRates.symmetric(16_000), 0, "C1 GPT-2 small transformer trace"
    raise SystemExit(f"unknown config {config}")


def _lifetime_bytes(N: int, T: int, E: int, P: int) -> int:
    """SURVEY §8d algorithmic bytes B_L = 8E + 16T + 8N + 24P + 24N."""
    return 8 * E + 16 * T + 8 * N + 24 * P + 24 * N


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"tio_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = max(mx, float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        except FileNotFoundError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(config: str, rounds_total: int | None, sample_rounds: int = 40, threads: int | None = None):
    """Oracle port on this host's cores: lifetime + the first R plan rounds,
    extrapolated to the full plan (rounds_total, from the GPU run)."""
    from oracle import oracle as O
    tr, cap, rates, hc, _ = _trace(config)
    a = tr.arrays()
    # every host thread this process may use (torchrun exports OMP_NUM_THREADS=1;
    # the oracle's libgomp reads the variable when the library is first loaded)
    os.environ["OMP_NUM_THREADS"] = str(threads or len(os.sched_getaffinity(0)))
    L = O.lib()
    t0 = time.perf_counter()
    lo = O.lifetime(a)
    t1 = time.perf_counter()
    p = O.plan(a, cap, rates.ssd_offload, rates.ssd_prefetch, rates.host_offload, rates.host_prefetch, hc,
               lifetime_out=lo, max_rounds=sample_rounds)
    t2 = time.perf_counter()
    done = max(1, int(p["rounds"]))
    total = rounds_total if rounds_total else done
    t_plan = (t2 - t1) * (total / done)
    ev = a.num_events / ((t1 - t0) + t_plan)
    return {"value": ev, "unit": "events/s", "cores": int(L.tio_oracle_threads()), "kind": "port",
            "sample": (f"oracle/tio_oracle.c on {config}: full lifetime ({t1 - t0:.3f} s) + first {done} of "
                       f"{total} planner rounds ({t2 - t1:.2f} s), plan time extrapolated linearly by rounds")}


def run_reference(args, rank: int, world: int):
    """The reference arm: the reference's algorithm on this host's cores — the
    oracle port (oracle/tio_oracle.c, OpenMP over candidates; the Python
    reference itself needs ~716 h per planner round at C3).

    Each timed step is one FULL lifetime + plan of the config's trace (C3:
    ~150 s on 16 threads), so the value is measured, not extrapolated, and the
    arm prints the plan's sha256 (equal to the GPU arm's and to
    tests/golden/<config>.json.gz).  At most --ref-full-steps of the requested
    K steps are run (a full C3 plan per step); warm-up steps run the lifetime
    stage only (page-in, thread pool start).  The old 12-round extrapolation is
    kept under "sampled_extrapolation" as a labelled secondary."""
    if rank != 0:
        return
    import hashlib
    from oracle import oracle as O
    tr, cap, rates, hc, desc = _trace(args.config)
    a = tr.arrays()
    E = a.num_events
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    L = O.lib()
    for _ in range(args.warmup):
        O.lifetime(a)
    steps = max(1, min(args.steps, args.ref_full_steps))
    t_life, t_plan, shas, rounds = [], [], set(), 0
    wall0 = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        lo = O.lifetime(a)
        t1 = time.perf_counter()
        p = O.plan(a, cap, rates.ssd_offload, rates.ssd_prefetch, rates.host_offload, rates.host_prefetch, hc,
                   lifetime_out=lo)
        t2 = time.perf_counter()
        t_life.append(t1 - t0)
        t_plan.append(t2 - t1)
        shas.add(hashlib.sha256(p["plan_bytes"]).hexdigest())
        rounds = int(p["rounds"])
    wall = time.perf_counter() - wall0
    sec = sum(t_life) + sum(t_plan)
    v = E * steps / sec
    sample = (f"oracle/tio_oracle.c on {args.config}: {steps} full lifetime + plan pass(es) "
              f"(lifetime {statistics.mean(t_life):.2f} s, plan {statistics.mean(t_plan):.1f} s, "
              f"{rounds} rounds), measured")
    line = {"metric": "trace events/s (lifetime+plan)", "value": v, "unit": "events/s", "n_gpus": world,
            "steps": steps, "steps_requested": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic", "impl": "reference",
            "config": {"workload": desc, "events": E, "capacity": cap, "rates": "ssd 16000 B/us symmetric",
                       "host_cap": hc, "plan_sha256": sorted(shas)[0] if len(shas) == 1 else sorted(shas)},
            "cpu_baseline": {"value": v, "unit": "events/s", "cores": int(L.tio_oracle_threads()), "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "breakdown_s": {"lifetime": statistics.mean(t_life), "plan": statistics.mean(t_plan)},
            "rounds": rounds, "wall_s": wall}
    if args.ref_sampled:
        line["sampled_extrapolation"] = cpu_baseline(args.config, rounds, sample_rounds=args.ref_rounds_c3
                                                     if args.config == "c3" else args.ref_rounds)
    print(json.dumps(line), flush=True)


def measure(config: str, steps: int, warmup: int, dev, rank: int, world: int) -> dict:
    """Device-timed lifetime + plan on one config (see module docstring)."""
    import torch
    from paper_2506_06472_b200 import _native
    from paper_2506_06472_b200.planner import _rates_struct

    tr, cap, rates, hc, desc = _trace(config)
    a = tr.arrays()
    N, T, E = a.num_kernels, a.num_tensors, a.num_events
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream
    lib = _native.load()
    dt = _native.DeviceTrace(a, stream=sh)
    r = _rates_struct(rates)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    group = None
    if world > 1:
        # strong scaling: ONE trace planned by all ranks, candidate tiles
        # sharded, per-round winner exchange over NVLink (distributed.PlanGroup)
        from paper_2506_06472_b200.distributed import PlanGroup
        group = PlanGroup(rank, world)

    def plan_call():
        return group.plan(dt, cap, r, hc) if group is not None else dt.plan(cap, r, hc)

    def step(evs=None):
        if evs:
            evs[0].record(stream)
        _native.check(lib.tio_lifetime(dt.handle, ctypes.c_void_p(sh)))
        if evs:
            evs[1].record(stream)
        p = plan_call()
        if evs:
            evs[2].record(stream)
        return p

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            step().close()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        launches0 = _native.kernel_launches()
        tot_ms, life_ms, plan_ms, loop_ms = 0.0, 0.0, 0.0, 0.0
        info = None
        plan_bytes = b""
        with Clocks(dev.index) as clk:
            for i in range(steps):
                flush.fill_(1)          # L2 flush, outside the timed region
                torch.cuda.synchronize()
                if world > 1:
                    torch.distributed.barrier()
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                p = step(evs)
                torch.cuda.synchronize()
                life_ms += evs[0].elapsed_time(evs[1])
                plan_ms += evs[1].elapsed_time(evs[2])
                tot_ms += evs[0].elapsed_time(evs[2])
                info = p.info
                loop_ms += info.loop_ns / 1e6
                if i == 0:
                    plan_bytes = p.write()
                p.close()
        launches = _native.kernel_launches() - launches0
        torch.cuda.synchronize()
    t = torch.tensor([tot_ms, loop_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    tot_ms_max = float(t[0].item())
    loop_ms = float(t[1].item())
    agree = group.plans_agree(plan_bytes) if group is not None else True

    # ---- e2e: C-ABI one-shot call, pinned host columns, host entries out
    cols = _native.HostColumns(a)
    pinned = {}
    for name in ("dur", "tid", "size", "kind", "ptr", "acc"):
        src = getattr(cols, name)
        pt = torch.empty(src.shape, dtype=getattr(torch, str(src.dtype)), pin_memory=True)
        pt.numpy()[...] = src
        pinned[name] = pt
    desc_c = _native.TraceDesc(N, pinned["dur"].data_ptr(), T, pinned["tid"].data_ptr(), pinned["size"].data_ptr(),
                               pinned["kind"].data_ptr(), pinned["ptr"].data_ptr(), E, pinned["acc"].data_ptr())
    ne = int(info.num_entries)
    ent = torch.empty(max(1, ne) * _native.ENTRY_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
    pinfo = _native.PlanInfo()
    h2d = sum(int(v.numel() * v.element_size()) for v in pinned.values())
    d2h = ne * _native.ENTRY_DTYPE.itemsize

    def one_shot():
        if group is None:
            _native.check(lib.tio_plan_host(ctypes.byref(desc_c), ctypes.c_int64(cap), ctypes.byref(r),
                                            ctypes.c_int64(hc), ctypes.c_void_p(sh), ctypes.byref(pinfo),
                                            ctypes.c_void_p(ent.data_ptr()), ctypes.c_int64(ne)))
            return
        # N > 1: the same C-ABI calls composed — trace upload from the pinned
        # host columns, lifetime, sharded plan, entries back to pinned host
        th = ctypes.c_void_p()
        _native.check(lib.tio_trace_create(ctypes.byref(desc_c), _native.TIO_MEM_HOST, ctypes.c_void_p(sh),
                                           ctypes.byref(th)))
        pdt = _native.DeviceTrace.__new__(_native.DeviceTrace)      # owns th from here on
        pdt._lib, pdt.handle, pdt.stream = lib, th, ctypes.c_void_p(sh)
        pdt.num_kernels, pdt.num_tensors = N, T
        try:
            p = group.plan(pdt, cap, r, hc)
            _native.check(lib.tio_plan_copy_out(p.handle, ctypes.c_void_p(sh), None,
                                                ctypes.c_void_p(ent.data_ptr()), None, None))
            p.close()
        finally:
            pdt.close()
    for _ in range(2):
        one_shot()
    e2e_ms = 0.0
    for _ in range(steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_shot()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = float(t.item())

    import hashlib
    K = steps
    P = int(info.num_candidates)
    B_L = _lifetime_bytes(N, T, E, P)
    life_s = life_ms / K / 1e3
    peak, peak_kind = _peaks()
    achieved = B_L / life_s / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "lifetime_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get(config)
        except Exception:
            traffic = None
    rounds = int(info.rounds)
    ptraffic = None
    pp = os.path.join(ROOT, "profiles", "planner_traffic.json")
    if os.path.exists(pp):
        try:
            with open(pp) as f:
                ptraffic = json.load(f).get(config)
        except Exception:
            ptraffic = None
    loop_s = loop_ms / K / 1e3
    if group is not None:
        group.close()
    return {
        "value": E * K / (tot_ms_max / 1e3), "ms_per_step": tot_ms_max / K,
        "config": {"workload": desc, "events": E, "kernels": N, "tensors": T, "periods": P,
                   "capacity": cap, "rates": ("ssd 16000 B/us symmetric" + (", host 50000 B/us" if hc else "")),
                   "host_cap": hc,
                   "parallelism": (f"sharded{world}: one trace, candidate tiles split over ranks, per-round "
                                   f"winner exchange through CUDA-IPC mailboxes over NVLink") if world > 1
                   else "single",
                   "l2": "flushed (256 MiB write) before every step, outside the timed region",
                   "plan_sha256": hashlib.sha256(plan_bytes).hexdigest(),
                   "plan_sha256_equal_on_all_ranks": bool(agree)},
        "breakdown_ms": {"lifetime": life_ms / K, "plan": plan_ms / K, "plan_round_loop": loop_ms / K,
                         "plan_setup_epilogue_host": (plan_ms - loop_ms) / K},
        "roofline": {"kernel": "lifetime (k_tile_owners + k_events + k_kernels)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes": B_L,
                     "share_of_step": life_ms / tot_ms,
                     "note": "the step's dominant kernel is plan_loop_kernel (see 'planner'): sequential greedy "
                             "rounds, latency-bound, no byte/flop roofline (SURVEY 8d); this is the HBM "
                             "roofline of the lifetime kernels"},
        "planner": {"kernel": "plan_loop_kernel (the step's dominant kernel)",
                    "bound": "latency (2 grid barriers + dependent L2 loads per round)",
                    "rounds": rounds, "commits": int(info.num_commits),
                    "us_per_round": (loop_ms / K) * 1e3 / max(1, rounds),
                    "share_of_step": loop_ms / tot_ms,
                    # ncu DRAM bytes of one launch over the measured loop time:
                    # the dominant kernel is latency-bound, not HBM-bound
                    "traffic": ptraffic,
                    "dram_gbs": (ptraffic / loop_s / 1e9) if ptraffic and loop_s > 0 else None,
                    "frac_of_hbm_peak": (ptraffic / loop_s / 1e9 / peak) if ptraffic and loop_s > 0 else None,
                    **({"debug_build": {
                        "phase_us_per_round_block0": dict(zip(
                            ["prologue", "evaluate", "block_reduce", "barrier1", "argmax", "channel_merge",
                             "residual", "commit_barrier2"],
                            [round(info.dbg[q] / 1e3 / max(1, rounds), 3) for q in range(8)])),
                        "dirty_tiles_per_round": info.dbg[8] / max(1, rounds),
                        "refits_per_round": info.dbg[9] / max(1, rounds),
                        "max_block_phase_E_us_per_round": info.dbg[10] / 1e3 / max(1, rounds),
                        "max_block_dirty_tiles_per_round": info.dbg[13] / max(1, rounds)}}
                       if any(info.dbg[q] for q in range(12)) else {})},
        "e2e": {"value": E * K / (e2e_ms / 1e3), "unit": "events/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "tio_plan_host (C ABI), pinned host buffers" if world == 1 else
                       "tio_trace_create (pinned host) + tio_lifetime + sharded tio_plan_create2 + "
                       "tio_plan_copy_out (C ABI), per rank"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "rounds": rounds,
    }


def sharded_lifetime_leg(config: str, dev, rank: int, world: int) -> dict:
    """the lifetime stage sharded by tensor id over the ranks
    (libtio kernels per shard, NCCL all_reduce of timeline/active bytes and
    all_gather of the period lists; paper_2506_06472_b200/distributed.py),
    checked against the whole-trace lifetime computed locally.  Wall time,
    max over ranks, host conversions included."""
    import hashlib
    import torch
    import torch.distributed as dist
    from paper_2506_06472_b200 import _native
    from paper_2506_06472_b200.distributed import sharded_lifetime
    try:
        tr, cap, rates, hc, desc = _trace(config)
        a = tr.arrays()
        full = _native.DeviceTrace(a)
        ref = full.lifetime()
        full.close()
        sharded_lifetime(a, rank, world, device=dev)          # warm-up
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = sharded_lifetime(a, rank, world, device=dev)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        same = all(np.array_equal(out[k].cpu().numpy() if hasattr(out[k], "cpu") else np.asarray(out[k]),
                                  np.asarray(ref[k]))
                   for k in ("timeline", "active", "period_tensor", "period_start", "period_end", "period_wraps"))
        ok = torch.tensor([1 if same else 0], dtype=torch.int64, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        return {"workload": desc, "ranks": world, "ms_wall_max_over_ranks": float(t.item()) * 1e3,
                "bit_exact_vs_unsharded": bool(ok.item()), "shard_events": int(a.access_ptr[out["shard"][1]] -
                                                                               a.access_ptr[out["shard"][0]]),
                "collectives": f"{dist.get_backend()} all_reduce(int64[2N]) + all_gather(counts, padded period "
                               f"columns), device-resident"}
    except Exception as exc:  # reported, not fatal: the headline line must still print
        return {"error": f"{type(exc).__name__}: {exc}"}


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    warm = max(args.warmup, 3) if args.warmup >= 3 else args.warmup
    m = measure(args.config, args.steps, warm, dev, rank, world)
    m_sh = sharded_lifetime_leg(args.config, dev, rank, world) if world > 1 else None
    extra = None
    if args.secondary and args.secondary != args.config:
        extra = measure(args.secondary, args.steps, warm, dev, rank, world)
    host_m = measure(args.host_leg, args.steps, warm, dev, rank, world) if args.host_leg else None
    c5 = c5_leg(args, rank, world) if args.c5 and world > 1 else None
    if rank != 0:
        return
    rounds = m.pop("rounds")
    line = {
        "metric": "trace events/s (lifetime+plan)", "value": m.pop("value"), "unit": "events/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": m.pop("ms_per_step"), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        **m,
    }
    if extra is not None:
        extra.pop("clocks", None)
        rx = extra.pop("rounds")
        if not args.no_cpu_baseline and world == 1:
            extra["cpu_baseline"] = cpu_baseline(args.secondary, rx, sample_rounds=args.ref_rounds)
        line[args.secondary] = extra
    if not args.no_cpu_baseline and world == 1:     # rank 0 at N = 1 only (the reference arm covers N > 1)
        line["cpu_baseline"] = cpu_baseline(args.config, rounds, sample_rounds=args.ref_rounds_c3
                                            if args.config == "c3" else args.ref_rounds)
    if world > 1 and m_sh is not None:
        line["sharded_lifetime"] = m_sh
    if c5 is not None:
        line["migration_dp"] = c5
    if host_m is not None:
        host_m.pop("clocks", None)
        host_m.pop("rounds", None)
        line[args.host_leg] = host_m
    if not args.no_migration and world == 1:
        # C4 on one GPU; at N > 1 the per-rank pinned host extents (24-78 GB
        # each) would exceed the box's host memory, so the leg runs at N = 1 only
        from paper_2506_06472_b200 import engine
        link = engine.measure_link()
        line["migration"] = real_step_bench(link=link, model=args.offload_model, rate_scale=args.c4_rate_scale,
                                            fracs=tuple(args.c4_fracs),
                                            identity_frac=0 if args.no_identity else 0.8)
        if args.replay_leg:
            # the synthetic Appendix-C replay against placeholder kernels (round 1's leg)
            line["migration_replay"] = [migration_bench(mb, link=link, cap_frac=f)
                                        for mb, f in ((4, 0.5), (8, 0.8), (8, 0.9))]
    print(json.dumps(line), flush=True)


def c5_leg(args, rank: int, world: int) -> dict:
    """Configs C5 (BASELINE.json configs[4]): data-parallel Llama-3-8B, one
    rank per GPU, every rank profiling its own step (gradients all-reduced
    between backward and the optimizer — the collective is a trace kernel
    touching the gradients, so they stay resident across it), planning it
    and running its own online engine over its own link, all at once.
    Reported: per capacity, the slowest rank's offloaded step vs the slowest
    rank's no-offload step, and every rank's link rates and byte checks."""
    import torch.distributed as dist
    from paper_2506_06472_b200 import engine
    own_link = engine.measure_link()
    box = [own_link]
    dist.broadcast_object_list(box, src=0)      # every rank plans with rank 0's link rate: identical plans
    r = real_step_bench(fracs=tuple(args.c5_fracs), link=box[0], model=args.offload_model, identity_frac=0,
                        dp=True)
    r["own_link"] = own_link
    allr = [None] * world
    dist.all_gather_object(allr, r)
    if rank != 0:
        return None
    out = {"workload": allr[0]["workload"] + f"; data parallel over {world} ranks (gradient all-reduce)",
           "ranks": world, "ideal_step_ms_max": max(x["ideal"]["step_ms"] for x in allr),
           "plans_identical": len({json.dumps([run["plan"]["sha256"] for run in x["runs"]]) for x in allr}) == 1,
           "links_gbs": [{"h2d": x["own_link"]["h2d_gbs"], "d2h": x["own_link"]["d2h_gbs"]} for x in allr],
           "plan_link": "rank 0's measured bidirectional rate (broadcast), rank 0's profiled durations", "runs": []}
    for i, frac in enumerate(args.c5_fracs):
        runs = [x["runs"][i] for x in allr]
        out["runs"].append({
            "capacity_frac_of_trace_peak": frac,
            "step_ms_max": max(q["step_ms"] for q in runs),
            "step_vs_ideal": max(q["step_ms"] for q in runs) / out["ideal_step_ms_max"],
            "model_step_vs_ideal": max(q["model_step_vs_ideal"] for q in runs),
            "offload_gbs_min": min(q["offload_gbs"] for q in runs),
            "prefetch_gbs_min": min(q["prefetch_gbs"] for q in runs),
            "verify_mismatches": sum(q["verify"]["mismatches"] for q in runs),
            "allocator_peak_vs_capacity_max": max(q["allocator_peak_vs_capacity"] for q in runs)})
    return out


def migration_bench(microbatches: int = 8, verify: bool = True, link: dict | None = None,
                    cap_frac: float = 0.5) -> dict:
    """Configs C4 (BASELINE.json): the migration engine executing a
    Llama-3-8B plan on 1 B200 (Appendix-C trace with `microbatches`
    microbatches of 8,192 tokens, real tensor sizes, capacity = peak // 2,
    the plan's channel rates = the measured pinned link, both directions at
    once).  Device time of the iteration with every transfer executed vs the
    same kernels with no migration; link GB/s vs the measured link."""
    from paper_2506_06472_b200 import engine, plan_migrations, ChannelRates
    from paper_2506_06472_b200 import tracegen as G
    link = link or engine.measure_link()
    rate = float(int(link["bidir_gbs_each"] * 1e3))        # bytes/us, integral
    tr = G.gen_llama_trace(G.LlamaTraceConfig(microbatches=microbatches))
    peak = G.llama_peak_bytes(tr)
    cap = peak // 2 if cap_frac == 0.5 else int(peak * cap_frac)
    rates = ChannelRates.symmetric(rate)
    t0 = time.perf_counter()
    plan = plan_migrations(tr, cap, rates)
    t_plan = time.perf_counter() - t0
    r = engine.replay(tr, plan, cap, rates, time_scale=1.0, verify=verify)
    link_each = link["bidir_gbs_each"]
    return {
        "workload": f"Llama-3-8B Appendix-C trace, {microbatches} microbatches x 8192 tokens, "
                    f"E={tr.arrays().num_events}, peak={peak}, capacity={cap_frac}*peak={cap}",
        "plan": {"entries": len(plan.entries), "warning": plan.warning, "over_capacity_kernels":
                 len(plan.over_capacity_kernels), "seconds": t_plan},
        "step_ms": r.replay_ms, "ideal_ms": r.ideal_ms, "step_vs_ideal": r.step_vs_ideal,
        "model_step_vs_ideal": r.model_total_us / r.model_ideal_us,
        "offload_gbs": r.offload_gbs, "prefetch_gbs": r.prefetch_gbs,
        "link": link, "offload_frac_of_link": r.offload_gbs / link_each if link_each else None,
        "prefetch_frac_of_link": r.prefetch_gbs / link_each if link_each else None,
        "bytes": {"offload": r.offload_bytes, "prefetch": r.prefetch_bytes, "host_extents": r.host_bytes},
        "transfers": {"offloads": r.n_offloads, "prefetches": r.n_prefetches, "emergency": r.emergency_offloads},
        "peak_device_bytes": r.peak_device_bytes, "capacity": cap,
        "verify": {"bytes": r.verified_bytes, "mismatches": r.verify_mismatches},
        "tier": "pinned host (no GDS: nvidia-fs absent); plan rates = measured bidirectional pinned link",
    }


def real_step_bench(fracs=(0.5, 0.8, 0.9), steps: int = 3, link: dict | None = None, model: str = "8b",
                    identity_frac: float = 0.8, identity_steps: int = 2, dp: bool = False,
                    rate_scale: float = 1.0) -> dict:
    """Configs C4 (BASELINE.json configs[3]): the migration engine executing
    the plan of a REAL Llama-3-8B training step on 1 B200 (random init bf16
    weights, fp32 AdamW moments, synthetic 8,192-token batch;
    paper_2506_06472_b200/llama_step.py).

    ideal   the same step, no engine, capacity unconstrained;
    profile one step under TraceProfiler -> trace (every aten operator a
            kernel, CUDA-event durations) -> device plan at capacity =
            frac x the trace's memory-timeline peak, channel rates = the
            measured pinned link (both directions busy);
    run     fresh model, same step sequence, OffloadMode (libtio online
            engine: storages freed / restored on side streams, event gated).

    Timing runs use the model's fast attention (cuDNN / flash SDPA, whose
    backward is not run-to-run deterministic).  Each timed step (K back to
    back, CUDA events on the compute stream, the last step fenced on every
    transfer) includes the batch H2D from pinned host and the loss D2H.  One
    verification step (checksum of every tensor at offload and after its
    prefetch) precedes the timed steps.

    identity: the same sequence on the deterministic model
    (FlashAttention-2 deterministic backward; run-to-run bit-identical) at
    capacity identity_frac x peak: losses and the checksum of every weight /
    AdamW moment after the offloaded steps must EQUAL the no-offload run's."""
    import dataclasses
    import gc
    import torch
    import hashlib
    from paper_2506_06472_b200 import ChannelRates, compute_memory_timeline, engine, plan_migrations, write_plan
    from paper_2506_06472_b200.llama_step import LLAMA3_8B_MODEL, TINY, Step
    from paper_2506_06472_b200.profiler import profile_step
    cfg_det = LLAMA3_8B_MODEL if model == "8b" else TINY
    cfg = dataclasses.replace(cfg_det, deterministic=False)
    dev = torch.device("cuda", torch.cuda.current_device())
    group = None
    if dp:                                     # configs C5: every rank runs this leg at once
        import torch.distributed as dist
        group = dist.group.WORLD

        def Step(c, seed=0, _S=Step):          # noqa: N802 - the DP form of the step
            return _S(c, seed=seed, dp_group=group)

    def sync():
        if group is not None:
            import torch.distributed as dist
            dist.barrier()

    def common_trace(tr):
        """DP: the ranks' traces have the same operators and tensors; their
        profiled durations differ by timing noise.  Every rank takes rank 0's
        durations (one int64[N] broadcast), so every rank plans the same trace
        and holds the same plan (identical per-rank plans)."""
        if group is None:
            return tr
        import dataclasses as dc
        import numpy as np
        import torch.distributed as dist
        from paper_2506_06472_b200.trace import Trace
        a = tr.arrays()
        d = torch.from_numpy(np.ascontiguousarray(a.duration_us, dtype=np.int64))
        d = d.to(dev) if dist.get_backend(group) == "nccl" else d
        dist.broadcast(d, src=0, group=group)
        return Trace.from_arrays(dc.replace(a, duration_us=d.cpu().numpy().astype(np.int64)), dict(tr.meta))
    link = link or engine.measure_link()
    # the plan's channel rate: the measured link with both directions busy,
    # optionally scaled (rate_scale < 1 plans with headroom for the copies'
    # achieved per-transfer rate)
    rate = float(int(link["bidir_gbs_each"] * 1e3 * rate_scale))   # bytes/us, integral
    rates = ChannelRates.symmetric(rate)
    stream = torch.cuda.current_stream()
    loss_host = torch.empty((), dtype=torch.float32, pin_memory=True)

    def run(s, n, mode=None):
        losses = []
        torch.cuda.synchronize()
        sync()                                 # DP: every rank starts the timed steps together
        torch.cuda.reset_peak_memory_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(n):
            batch = s.host_batch.to(dev, non_blocking=True)
            if mode is None:
                loss = s(batch)
            else:
                with mode.step(done_stream=stream if i == n - 1 else None):
                    loss = s(batch)
            loss_host.copy_(loss, non_blocking=True)
            losses.append(loss)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n, [float(x.item()) for x in losses], torch.cuda.max_memory_allocated()

    def digest(s):
        names = sorted(s.globals_of())
        g = s.globals_of()
        return engine.checksums([g[n] for n in names])

    def free():
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    def log(msg):
        print(f"[c4] {msg}  (allocated {torch.cuda.memory_allocated() / 1e9:.1f} GB)", file=sys.stderr, flush=True)

    def ideal_run(c, n):
        s = Step(c, seed=0)
        for _ in range(3):
            s()
        ms, losses, peak = run(s, n)
        dg = digest(s)
        return ms, losses, peak, dg

    def offloaded(c, tr, frac, n, peak):
        """steps 1 (plain) + 2 (profiled, done by the caller or here) + 3
        (verification) + n timed: the same step count as ideal_run."""
        cap = int(peak * frac)
        t0 = time.perf_counter()
        plan = plan_migrations(tr, cap, rates)
        t_plan = time.perf_counter() - t0
        s = Step(c, seed=0)
        for _ in range(2):
            s()
        mode = engine.OffloadMode(tr, plan, cap, rates, s.globals_of(), verify=True)
        with mode.step():                      # step 3: sets up the steady state, checksums every round trip
            s()
        torch.cuda.synchronize()
        vst = mode.stats()
        mode.set_verify(False)
        ms, losses, apeak = run(s, n, mode)
        st = mode.stats()
        mode.restore()                         # globals offloaded at the step boundary come back
        dg = digest(s)
        info = mode.info
        mode.close()
        return cap, plan, t_plan, vst, ms, losses, apeak, st, dg, info

    # ---- ideal: plain PyTorch, capacity unconstrained (+ the model's own spread)
    log("ideal run")
    ideal_ms, ideal_losses, ideal_peak, ideal_digest = ideal_run(cfg, steps)
    free()
    _, rerun_losses, _, rerun_digest = ideal_run(cfg, steps)
    free()

    # ---- profile (step 2 of a fresh model) -> trace
    log(f"ideal {ideal_ms:.1f} ms/step, peak {ideal_peak / 1e9:.1f} GB; profiling")
    s = Step(cfg, seed=0)
    s()
    t0 = time.perf_counter()
    tr = common_trace(profile_step(s, globals_=s.globals_of(), meta={"generator": "TraceProfiler",
                                                                       "model": f"llama3-{model}"}))
    t_prof = time.perf_counter() - t0
    s = None
    free()
    a = tr.arrays()
    peak = compute_memory_timeline(tr).peak()
    out = {"workload": f"Llama-3-{model.upper()} real training step (random init bf16 weights, fp32 AdamW, "
                       f"1 x {cfg.seq} synthetic tokens); trace of the profiled step: {a.num_kernels} kernels "
                       f"(aten operators), {a.num_tensors} tensors, {a.num_events} events, peak {peak} B",
           "link": link, "plan_rates_bytes_per_us": rate, "plan_rate_scale": rate_scale,
           "ideal": {"step_ms": ideal_ms, "allocator_peak_bytes": ideal_peak, "losses": ideal_losses,
                     "rerun_losses": rerun_losses, "rerun_state_checksums_equal": rerun_digest == ideal_digest,
                     "deterministic": rerun_losses == ideal_losses and rerun_digest == ideal_digest,
                     "attention": "SDPA (cuDNN / flash; backward not run-to-run deterministic)"},
           "profile_s": t_prof, "runs": []}
    log(f"trace: {a.num_kernels} kernels, {a.num_tensors} tensors, peak {peak / 1e9:.1f} GB ({t_prof:.1f} s)")
    for frac in fracs:
        log(f"capacity {frac} x peak")
        cap, plan, t_plan, vst, ms, losses, apeak, st, dg, info = offloaded(cfg, tr, frac, steps, peak)
        free()
        off_gbs = st["last_offload_bytes"] / (st["last_offload_busy_ms"] * 1e6) if st["last_offload_busy_ms"] else 0.0
        pre_gbs = st["last_prefetch_bytes"] / (st["last_prefetch_busy_ms"] * 1e6) if st["last_prefetch_busy_ms"] else 0.0
        per_step_off = st["offload_bytes"] / max(1, st["steps"])
        per_step_pre = st["prefetch_bytes"] / max(1, st["steps"])
        lb_ms = max(per_step_off / (link["d2h_gbs"] * 1e6), per_step_pre / (link["h2d_gbs"] * 1e6))
        out["runs"].append({
            "capacity_frac_of_trace_peak": frac, "capacity": cap,
            "plan": {"entries": len(plan.entries), "warning": plan.warning,
                     "over_capacity_kernels": len(plan.over_capacity_kernels), "seconds": t_plan,
                     "sha256": hashlib.sha256(write_plan(plan)).hexdigest()},
            "step_ms": ms, "step_vs_ideal": ms / ideal_ms,
            "model_step_vs_ideal": info["model_total_us"] / max(1, info["model_ideal_us"]),
            "link_lower_bound_ms": lb_ms, "link_lower_bound_vs_ideal": max(1.0, lb_ms / ideal_ms),
            "allocator_peak_bytes": apeak, "allocator_peak_vs_capacity": apeak / cap,
            "model_peak_resident": info["model_peak_resident"],
            "offload_gbs": off_gbs, "prefetch_gbs": pre_gbs,
            "offload_frac_of_link_d2h": off_gbs / link["d2h_gbs"] if link["d2h_gbs"] else None,
            "prefetch_frac_of_link_h2d": pre_gbs / link["h2d_gbs"] if link["h2d_gbs"] else None,
            "bytes_per_step": {"offload": per_step_off, "prefetch": per_step_pre, "host_extents": info["host_bytes"]},
            "transfers_per_step": {"offloads": info["model_offloads"], "prefetches": info["model_prefetches"],
                                   "emergency": info["emergency_offloads"]},
            "verify": {"round_trips_checked": vst["n_prefetches"], "mismatches": vst["verify_mismatches"]},
            "losses": losses, "max_loss_dev_vs_ideal": max(abs(x - y) for x, y in zip(losses, ideal_losses)),
            "ideal_rerun_max_loss_dev": max(abs(x - y) for x, y in zip(rerun_losses, ideal_losses)),
        })
        log(f"capacity {frac}: {ms:.1f} ms/step ({ms / ideal_ms:.2f}x ideal), allocator peak {apeak / 1e9:.1f} GB")

    # ---- byte identity on the deterministic model
    if identity_frac:
        log(f"identity leg: deterministic model, capacity {identity_frac} x peak")
        d_ms, d_losses, _, d_digest = ideal_run(cfg_det, identity_steps)
        free()
        s = Step(cfg_det, seed=0)
        s()
        trd = profile_step(s, globals_=s.globals_of(), meta={"generator": "TraceProfiler",
                                                              "model": f"llama3-{model}-deterministic"})
        s = None
        free()
        peak_d = compute_memory_timeline(trd).peak()
        cap, plan, _, vst, ms, losses, apeak, st, dg, info = offloaded(cfg_det, trd, identity_frac, identity_steps,
                                                                       peak_d)
        free()
        out["identity"] = {
            "model": "deterministic attention (FlashAttention-2, deterministic backward)",
            "capacity_frac_of_trace_peak": identity_frac, "capacity": cap, "steps_compared": identity_steps,
            "ideal_step_ms": d_ms, "offloaded_step_ms": ms, "step_vs_ideal": ms / d_ms,
            "offloaded_bytes_per_step": st["offload_bytes"] / max(1, st["steps"]),
            "verify_mismatches": vst["verify_mismatches"],
            "losses_ideal": d_losses, "losses_offloaded": losses, "losses_equal": losses == d_losses,
            "state_checksums_equal": dg == d_digest, "tensors_compared": len(dg)}
        log(f"identity: losses equal {losses == d_losses}, state equal {dg == d_digest}")
    out["tier"] = "pinned host extents (4 KB aligned) via cudaMemcpyAsync on per-channel side streams " \
                  "(cuFile: cuFileDriverOpen blocks on the GPU boxes, profiles/r09/cufile_probe.txt)"
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "llama1"],
                    help="headline workload (default C3: the north star's 10M-event trace)")
    ap.add_argument("--secondary", default="c2", choices=["", "c1", "c2", "c3", "llama1"],
                    help="second workload reported under its own key (default C2, BASELINE configs[1])")
    ap.add_argument("--host-leg", default="c2host", choices=["", "c2host", "c3host"],
                    help="also plan a trace with the host tier (reported under its own key)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-migration", action="store_true", help="skip the C4 offloaded-step leg")
    ap.add_argument("--offload-model", default="8b", choices=["8b", "tiny"],
                    help="model of the C4 leg (8b = Llama-3-8B; tiny for quick checks)")
    ap.add_argument("--c4-rate-scale", type=float, default=1.0,
                    help="C4: plan with this fraction of the measured bidirectional link rate")
    ap.add_argument("--c4-fracs", type=float, nargs="+", default=[0.5, 0.8, 0.9],
                    help="C4: capacities (x trace peak)")
    ap.add_argument("--no-identity", action="store_true", help="C4: skip the byte-identity sub-leg")
    ap.add_argument("--c5", action="store_true",
                    help="N > 1: also run the data-parallel offloaded step on every rank (configs C5)")
    ap.add_argument("--c5-fracs", type=float, nargs="+", default=[0.9],
                    help="capacities (x trace peak) of the C5 leg")
    ap.add_argument("--replay-leg", action="store_true",
                    help="also run the Appendix-C replay against placeholder kernels")
    ap.add_argument("--ref-rounds", type=int, default=40, help="planner rounds in the CPU sample (C2)")
    ap.add_argument("--ref-rounds-c3", type=int, default=12, help="planner rounds in the CPU sample (C3)")
    ap.add_argument("--ref-rounds-total", type=int, default=None,
                    help="total rounds of the full plan (for the sampled extrapolation)")
    ap.add_argument("--ref-full-steps", type=int, default=1,
                    help="reference arm: full lifetime+plan passes actually timed (each ~150 s at C3)")
    ap.add_argument("--ref-sampled", action="store_true",
                    help="reference arm: also report the old sampled-round extrapolation")
    args = ap.parse_args(argv)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # testing the multi-process path on ONE GPU: TIO_BENCH_ONE_GPU=1 puts every
    # rank on cuda:0 and uses gloo (NCCL refuses two ranks on one device)
    one_gpu = os.environ.get("TIO_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local_rank = 0
    if args.impl == "reference":
        if args.ref_rounds_total is None:
            args.ref_rounds_total = _known_rounds(args.config)
        run_reference(args, rank, world)
        return
    # the C4 leg's real training step: expandable segments keep the caching
    # allocator's fragmentation out of the offloaded step's peak (must be set
    # before the first CUDA allocation of the process)
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def _known_rounds(config: str):
    """Total planner rounds of the config (recorded from the GPU path in
    tests/golden; the reference arm needs it to extrapolate its sample)."""
    try:
        import gzip
        with gzip.open(os.path.join(ROOT, "tests", "golden", f"{config}.json.gz"), "rt") as f:
            rec = json.load(f)
        if isinstance(rec, dict):
            return int(rec.get("rounds") or rec.get("num_commits"))
    except Exception:
        pass
    return None


if __name__ == "__main__":
    main()
