"""Generate the golden fixtures of the parity tests from the REFERENCE itself.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # fuzz corpora + C1 (~1 min)
    python tests/golden/make_golden.py --llama1   # + the 1-microbatch Llama plan (~5 min)

It imports the reference package `offloader` read-only from
/root/reference/pkg/src and records, for every case, the reference's own
outputs: compute_inactive_periods (analysis.py:58-83), compute_memory_timeline
(:97-108), per_kernel_active_bytes (:111-117), plan_migrations
(planner.py:267-370) committed rounds and write_plan bytes (:402-420).
The traces themselves are NOT stored: each case records the generator
arguments plus the sha256 of the reference's write_trace bytes, and the tests
regenerate the trace with this repo's generator and check that hash first.

Corpora (the reference's own acceptance generators, test_acceptance.py):
  crit2   criterion 2 (:64-101), random.Random(2024), 1000 traces
  crit3   criterion 3 (:104-131), random.Random(7), eligible instances of the
          first 5000 attempts
  extreme edge magnitudes (benefits past 2^64, fractional rates), all-equal
          sizes/durations (ties everywhere), 1-3 kernel traces; 300 cases
  layers  simulate_layer_granularity on transformer traces (+ layer maps) and
          layer-less random traces
  roofline roofline_curve + saturation_bandwidth on random traces and C1
  c1      config C1: GPT-2 small transformer trace, 4 rate setups
  llama1  Appendix-C Llama-3-8B trace with 1 microbatch (E=4,579; slow)

Output: tests/golden/*.json.gz (small; committed).  Nothing on the GPU box
reads /root/reference: only these fixtures travel.
"""

from __future__ import annotations

import argparse
import gzip
import hashlib
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import offloader  # noqa: E402  (the reference, read-only)
    return offloader


def _record(ref, trace, capacity, rates, host_cap, with_plan=True):
    periods = ref.compute_inactive_periods(trace)
    out = {
        "trace_sha256": hashlib.sha256(ref.write_trace(trace)).hexdigest(),
        "periods": [[p.tensor_id, p.size_bytes, p.start_kernel, p.end_kernel, int(p.wraps)]
                    for p in periods],
        "timeline": ref.compute_memory_timeline(trace).per_kernel_bytes,
        "active": ref.per_kernel_active_bytes(trace),
        "capacity": capacity,
        "rates": [rates.ssd_offload, rates.ssd_prefetch, rates.host_offload, rates.host_prefetch],
        "host_cap": host_cap,
    }
    if with_plan:
        try:
            plan = ref.plan_migrations(trace, capacity, rates, host_cap=host_cap)
        except ref.UnsatisfiableTraceError as exc:
            out["unsat_kernel"] = exc.kernel_index
            return out
        out["plan"] = ref.write_plan(plan).decode()
        out["committed"] = [[c.tensor_id, c.start_kernel, c.end_kernel, int(c.wraps), c.destination,
                             list(c.offload_interval), list(c.prefetch_interval), str(c.benefit),
                             c.cost, list(c.relieved_kernels)] for c in plan.committed]
        out["residual"] = plan.residual_timeline.per_kernel_bytes
    return out


def crit2(ref):
    """test_acceptance.py:64-101, same RNG call sequence."""
    rng = random.Random(2024)
    cases = []
    for _ in range(1000):
        nk = rng.randint(4, 64)
        nt = rng.randint(2, 32)
        seed = rng.randint(0, 10**9)
        gen = {"seed": seed, "num_kernels": nk, "num_tensors": nt,
               "size_range": [500_000, 60_000_000], "duration_range": [200, 5_000]}
        trace = ref.gen_random_trace(seed, nk, nt, size_range=(500_000, 60_000_000),
                                     duration_range=(200, 5_000))
        peak = ref.compute_memory_timeline(trace).peak()
        floor = max(ref.per_kernel_active_bytes(trace), default=0)
        capacity = max(floor, int(peak * rng.choice((0.55, 0.7, 0.85))))
        ssd = rng.choice((2_000, 10_000, 40_000))
        if rng.random() < 0.3:
            rates = ref.ChannelRates.symmetric(ssd, host=2 * ssd)
            host_cap = rng.choice((0, 200_000_000))
        else:
            rates = ref.ChannelRates.symmetric(ssd)
            host_cap = 0
        rec = _record(ref, trace, capacity, rates, host_cap)
        rec["gen"] = gen
        cases.append(rec)
    return cases


def crit3(ref):
    """test_acceptance.py:104-131 generator (all eligible instances of the
    first 5000 attempts; the reference test starves at 500 with commits)."""
    rng = random.Random(7)
    cases = []
    for _ in range(5000):
        seed = rng.randint(0, 10**9)
        nk = rng.randint(3, 8)
        nt = rng.randint(1, 4)
        trace = ref.gen_random_trace(seed, nk, nt, size_range=(1_000, 900_000),
                                     duration_range=(10, 400))
        periods = ref.compute_inactive_periods(trace)
        if not periods or len(periods) > 6:
            continue
        peak = ref.compute_memory_timeline(trace).peak()
        floor = max(ref.per_kernel_active_bytes(trace), default=0)
        capacity = max(floor, int(peak * 0.6))
        if rng.random() < 0.4:
            rates = ref.ChannelRates.symmetric(rng.choice((50, 500)), host=1_000)
            host_cap = rng.choice((0, 2_000_000))
        else:
            rates = ref.ChannelRates.symmetric(rng.choice((50, 500)))
            host_cap = 0
        rec = _record(ref, trace, capacity, rates, host_cap)
        rec["gen"] = {"seed": seed, "num_kernels": nk, "num_tensors": nt,
                      "size_range": [1_000, 900_000], "duration_range": [10, 400]}
        cases.append(rec)
    return cases


def extreme(ref):
    """Edge magnitudes and ties (not in the reference's own corpora):
    sizes 2^40-2^50 B with kernel durations up to 1e9 us (benefits past
    2^64, fractional rates -> exact Fraction transfer durations), all-equal
    sizes and durations (every ratio ties: the lowest candidate index must
    win), and 1-3 kernel traces (no gaps, only wraps)."""
    rng = random.Random(4242)
    cases = []
    for i in range(300):
        kind = i % 3
        if kind == 0:
            nk, nt = rng.randint(4, 48), rng.randint(2, 24)
            sr, dr = (1 << 40, 1 << 50), (1_000_000, 1_000_000_000)
            ssd = rng.choice((1_100_000, 33_000_000, 1_234_567.5, 987_654.321))
        elif kind == 1:
            nk, nt = rng.randint(4, 64), rng.randint(2, 32)
            s, d = rng.choice((50_000_000, 1 << 30)), rng.choice((1_000, 7))
            sr, dr = (s, s), (d, d)
            ssd = s / (d * rng.choice((0.25, 0.5, 1.5)))
        else:
            nk, nt = rng.randint(1, 3), rng.randint(1, 6)
            sr, dr = (1_000, 900_000), (10, 400)
            ssd = rng.choice((50_000, 5_000_000, 123_456.75))
        seed = rng.randint(0, 10**9)
        gf = rng.choice((0.0, 0.3, 0.8))
        trace = ref.gen_random_trace(seed, nk, nt, size_range=sr, duration_range=dr, global_fraction=gf)
        peak = ref.compute_memory_timeline(trace).peak()
        floor = max(ref.per_kernel_active_bytes(trace), default=0)
        capacity = max(floor, int(peak * rng.choice((0.5, 0.7, 0.9))))
        if rng.random() < 0.3:
            rates = ref.ChannelRates.symmetric(ssd, host=ssd * 2)
            host_cap = rng.choice((0, int(peak // 3)))
        else:
            rates = ref.ChannelRates.symmetric(ssd)
            host_cap = 0
        rec = _record(ref, trace, capacity, rates, host_cap)
        rec["gen"] = {"seed": seed, "num_kernels": nk, "num_tensors": nt, "size_range": list(sr),
                      "duration_range": list(dr), "global_fraction": gf}
        cases.append(rec)
    return cases


LAYER_FIELDS = ("total_time", "ideal_time", "per_kernel_start", "stall_per_kernel", "per_kernel_resident",
                "stall_time_total", "peak_resident_bytes", "channel_utilization", "emergency_offloads",
                "throughput_vs_ideal")


def _layer_record(ref, trace, capacity, rates, layer_map=None):
    try:
        r = ref.simulate_layer_granularity(trace, capacity, rates, layer_map=layer_map)
    except (ref.SimulationError, ref.ConfigurationError) as exc:
        return {"error": f"{type(exc).__name__}: {exc}"}
    return {f: getattr(r, f) for f in LAYER_FIELDS}


def layers(ref):
    """simulate_layer_granularity (simulator.py:549-560, policy :95-177) on
    transformer traces (C1 and random small shapes) across capacities and
    rates, with tensor layer maps, plus layer-less random traces (the
    ConfigurationError path when the policy engages)."""
    rng = random.Random(555)
    cases = []
    gens = [dict(num_layers=12, hidden_dim=768, num_heads=12, batch=8, seq_len=1024, bytes_per_element=4,
                 compute_rate=cr, seed=0) for cr in (1_000_000_000, 10_000_000)]
    for _ in range(40):
        gens.append(dict(num_layers=rng.randint(1, 6), hidden_dim=rng.choice((64, 128, 256)), num_heads=4,
                         batch=rng.randint(1, 4), seq_len=rng.choice((64, 128, 512)), bytes_per_element=rng.choice((2, 4)),
                         compute_rate=rng.choice((1_000, 100_000, 10_000_000)), seed=rng.randint(0, 999)))
    for g in gens:
        trace = ref.gen_transformer_trace(ref.TransformerGenConfig(**g))
        peak = ref.compute_memory_timeline(trace).peak()
        floor = max(ref.per_kernel_active_bytes(trace), default=0)
        for _ in range(3):
            capacity = max(floor, int(peak * rng.choice((0.3, 0.5, 0.7, 0.9, 1.0))))
            ssd = rng.choice((1_000, 16_000, 64_000, 2_500.5))
            rates = ref.ChannelRates.symmetric(ssd, host=ssd * 2) if rng.random() < 0.3 else \
                ref.ChannelRates.symmetric(ssd)
            lmap = None
            if rng.random() < 0.3:
                ids = [t.id for t in trace.tensors]
                lmap = {i: rng.randint(0, g["num_layers"] - 1) for i in rng.sample(ids, max(1, len(ids) // 4))}
            rec = _layer_record(ref, trace, capacity, rates, lmap)
            rec.update({"gen": {"transformer": g}, "trace_sha256": hashlib.sha256(ref.write_trace(trace)).hexdigest(),
                        "capacity": capacity, "rates": [rates.ssd_offload, rates.ssd_prefetch, rates.host_offload,
                                                        rates.host_prefetch],
                        "layer_map": sorted(lmap.items()) if lmap else None})
            cases.append(rec)
    for _ in range(20):   # no layer ids: ConfigurationError once the policy engages, a plain run otherwise
        seed = rng.randint(0, 10**9)
        gen = {"seed": seed, "num_kernels": rng.randint(3, 30), "num_tensors": rng.randint(2, 12),
               "size_range": [500_000, 60_000_000], "duration_range": [200, 5_000]}
        trace = ref.gen_random_trace(seed, gen["num_kernels"], gen["num_tensors"], size_range=(500_000, 60_000_000),
                                     duration_range=(200, 5_000))
        peak = ref.compute_memory_timeline(trace).peak()
        floor = max(ref.per_kernel_active_bytes(trace), default=0)
        capacity = max(floor, int(peak * rng.choice((0.6, 1.0))))
        rates = ref.ChannelRates.symmetric(10_000)
        rec = _layer_record(ref, trace, capacity, rates)
        rec.update({"gen": gen, "trace_sha256": hashlib.sha256(ref.write_trace(trace)).hexdigest(),
                    "capacity": capacity, "rates": [rates.ssd_offload, rates.ssd_prefetch, rates.host_offload,
                                                    rates.host_prefetch], "layer_map": None})
        cases.append(rec)
    return cases


def roofline(ref):
    """roofline_curve / saturation_bandwidth (roofline.py:39-125) on random
    traces (the reference's test_roofline generator and wider ones, globals
    included) and on C1, over integer and fractional bandwidth grids."""
    rng = random.Random(777)
    cases = []
    for i in range(120):
        seed = rng.randint(0, 10**9)
        nk, nt = (10, 8) if i < 30 else (rng.randint(2, 60), rng.randint(1, 30))
        sr, dr = ((1_000, 80_000), (50, 500)) if i < 30 else ((500_000, 60_000_000), (200, 5_000))
        gf = 0.3 if i < 30 else rng.choice((0.0, 0.3, 0.9))
        trace = ref.gen_random_trace(seed, nk, nt, size_range=sr, duration_range=dr, global_fraction=gf)
        if i < 30:
            capacity = max(1, sum(t.size_bytes for t in trace.tensors) // 2)
            grid = [10, 30, 100, 300, 1_000, 10_000]
        else:
            capacity = max(1, int(ref.compute_memory_timeline(trace).peak() * rng.choice((0.3, 0.6, 0.9, 1.1))))
            grid = sorted(rng.sample([7.5, 100, 1_000, 2_500.25, 10_000, 16_000, 40_000, 123_456.5, 1e6], 5))
        pts = ref.roofline_curve(trace, capacity, grid)
        cases.append({"gen": {"seed": seed, "num_kernels": nk, "num_tensors": nt, "size_range": list(sr),
                              "duration_range": list(dr), "global_fraction": gf},
                      "trace_sha256": hashlib.sha256(ref.write_trace(trace)).hexdigest(),
                      "capacity": capacity, "grid": grid,
                      "points": [p.normalized_throughput for p in pts],
                      "saturation": ref.saturation_bandwidth(trace)})
    cfg = ref.TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8, seq_len=1024,
                                   bytes_per_element=4, compute_rate=1_000_000_000, seed=0)
    trace = ref.gen_transformer_trace(cfg)
    grid = [1_000, 4_000, 16_000, 64_000, 256_000, 1_000_000]
    capacity = ref.compute_memory_timeline(trace).peak() // 2
    cases.append({"gen": {"c1": True}, "trace_sha256": hashlib.sha256(ref.write_trace(trace)).hexdigest(),
                  "capacity": capacity, "grid": grid,
                  "points": [p.normalized_throughput for p in ref.roofline_curve(trace, capacity, grid)],
                  "saturation": ref.saturation_bandwidth(trace)})
    return cases


C1_SETUPS = [  # (compute_rate, ssd, host, host_cap) — SURVEY §8d
    (1_000_000_000, 16_000, None, 0),
    (1_000_000_000, 64_000, None, 0),
    (1_000_000_000, 16_000, 32_000, 8_000_000_000),
    (10_000_000, 16_000, None, 0),
]


def c1(ref):
    cases = []
    for cr, ssd, host, host_cap in C1_SETUPS:
        cfg = ref.TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8,
                                       seq_len=1024, bytes_per_element=4, compute_rate=cr, seed=0)
        trace = ref.gen_transformer_trace(cfg)
        capacity = ref.compute_memory_timeline(trace).peak() // 2
        rates = ref.ChannelRates.symmetric(ssd, host=host)
        rec = _record(ref, trace, capacity, rates, host_cap)
        rec["gen"] = {"compute_rate": cr}
        rec["plan_sha256"] = hashlib.sha256(rec["plan"].encode()).hexdigest()
        cases.append(rec)
    return cases


def llama1(ref):
    """Appendix-C trace with 1 microbatch, converted to a reference Trace
    through the JSONL format (reference parse_trace, trace.py:217-275)."""
    sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
    from paper_2506_06472_b200 import tracegen, trace as T
    ours = tracegen.gen_llama_trace(tracegen.LlamaTraceConfig(microbatches=1))
    trace = ref.parse_trace(T.write_trace(ours))
    capacity = ref.compute_memory_timeline(trace).peak() // 2
    rates = ref.ChannelRates.symmetric(16_000)
    t0 = time.time()
    rec = _record(ref, trace, capacity, rates, 0)
    rec["gen"] = {"microbatches": 1}
    rec["ref_seconds"] = round(time.time() - t0, 1)
    rec["plan_sha256"] = hashlib.sha256(rec["plan"].encode()).hexdigest()
    return [rec]


def _sim_record(ref, trace, plan_text, capacity, rates):
    """Reference simulate() (simulator.py:539-542) under the plan and with no
    plan (simulate_on_demand, :545-547); SimulationError recorded as text."""
    out = {}
    for key, entries in (("plan", ref.parse_plan(plan_text)[1] if plan_text else None), ("on_demand", None)):
        try:
            r = ref.simulate(trace, entries, capacity, rates) if entries is not None else \
                ref.simulate_on_demand(trace, capacity, rates)
        except ref.SimulationError as exc:
            out[key] = {"error": str(exc)}
            continue
        out[key] = {"total_time": r.total_time, "ideal_time": r.ideal_time,
                    "per_kernel_start": r.per_kernel_start, "stall_per_kernel": r.stall_per_kernel,
                    "per_kernel_resident": r.per_kernel_resident, "stall_time_total": r.stall_time_total,
                    "peak_resident_bytes": r.peak_resident_bytes, "channel_utilization": r.channel_utilization,
                    "emergency_offloads": r.emergency_offloads, "throughput_vs_ideal": r.throughput_vs_ideal}
    return out


def sim(ref):
    """simulate / simulate_on_demand on the criterion-2 and extreme corpora
    (every case, with its reference plan)."""
    cases = []
    for corpus in ("crit2", "extreme"):
        for rec in json.load(gzip.open(os.path.join(HERE, f"{corpus}.json.gz"), "rt")):
            if "unsat_kernel" in rec:
                continue
            g = rec["gen"]
            trace = ref.gen_random_trace(g["seed"], g["num_kernels"], g["num_tensors"],
                                         size_range=tuple(g["size_range"]),
                                         duration_range=tuple(g["duration_range"]),
                                         global_fraction=g.get("global_fraction", 0.3))
            so, sp, ho, hp = rec["rates"]
            rates = ref.ChannelRates(so, sp, ho, hp)
            out = _sim_record(ref, trace, rec.get("plan"), rec["capacity"], rates)
            out.update({"corpus": corpus, "gen": g, "trace_sha256": rec["trace_sha256"]})
            cases.append(out)
    return cases


def _dump(name, cases):
    path = os.path.join(HERE, f"{name}.json.gz")
    with gzip.open(path, "wt", encoding="utf-8", compresslevel=9) as f:
        json.dump(cases, f, separators=(",", ":"))
    print(f"{name}: {len(cases)} cases -> {path} ({os.path.getsize(path)} B)")


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--llama1", action="store_true", help="also the slow 1-microbatch Llama plan")
    ap.add_argument("--only", default=None)
    args = ap.parse_args(argv)
    ref = _ref()
    todo = {"crit2": crit2, "crit3": crit3, "extreme": extreme, "c1": c1, "sim": sim, "layers": layers, "roofline": roofline}
    if args.llama1:
        todo["llama1"] = llama1
    for name, fn in todo.items():
        if args.only and name != args.only:
            continue
        t0 = time.time()
        cases = fn(ref)
        _dump(name, cases)
        print(f"  {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
