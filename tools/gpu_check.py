"""Ad-hoc GPU bring-up check: device planner vs the CPU oracle."""
import hashlib, random, sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2506_06472_b200 import _native, tracegen as G
from paper_2506_06472_b200 import plan_device, ChannelRates
from oracle import oracle as O

print(_native.device_info(), flush=True)

def cmp_case(tr, cap, rates, hc, tag):
    a = tr.arrays()
    o = O.plan(a, cap, rates.ssd_offload, rates.ssd_prefetch,
               rates.host_offload if rates.has_host else None,
               rates.host_prefetch if rates.has_host else None, hc)
    g = plan_device(tr, cap, rates, hc)
    ok = g["plan_bytes"] == o["plan_bytes"] and np.array_equal(g["residual"], o["residual"])
    if not ok:
        print("MISMATCH", tag, len(g["commits"]), len(o["committed"]))
        for j, (x, y) in enumerate(zip(g["commits"], o["committed"])):
            if (int(x["tensor_id"]), int(x["start_kernel"]), (int(x["off_start"]), int(x["off_end"])), (int(x["pre_start"]), int(x["pre_end"]))) != (y[0], y[1], y[5], y[6]):
                print(" first diff at", j, x, y); break
    return ok

rng = random.Random(2024)
bad = 0
t0 = time.time()
for case in range(300):
    nk = rng.randint(4, 64); nt = rng.randint(2, 32)
    tr = G.gen_random_trace(rng.randint(0, 10**9), nk, nt, size_range=(500_000, 60_000_000), duration_range=(200, 5_000))
    a = tr.arrays()
    lo = O.lifetime(a)
    peak = int(lo[1].max()); floor = int(lo[2].max())
    cap = max(floor, int(peak * rng.choice((0.55, 0.7, 0.85))))
    ssd = rng.choice((2000, 10000, 40000))
    if rng.random() < 0.3:
        rates = ChannelRates.symmetric(ssd, host=2 * ssd); hc = rng.choice((0, 200_000_000))
    else:
        rates = ChannelRates.symmetric(ssd); hc = 0
    if not cmp_case(tr, cap, rates, hc, f"fuzz{case}"):
        bad += 1
        if bad > 3: break
print("fuzz mismatches", bad, "in", time.time() - t0, "s", flush=True)

for cr, rates, hc, exp in [(1_000_000_000, ChannelRates.symmetric(16000), 0, "ed841d86"),
                           (1_000_000_000, ChannelRates.symmetric(64000), 0, "b5a35595"),
                           (1_000_000_000, ChannelRates.symmetric(16000, host=32000), 8_000_000_000, "4d1ff45f"),
                           (10_000_000, ChannelRates.symmetric(16000), 0, "27c8b0f8")]:
    tr = G.gen_transformer_trace(G.TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8, seq_len=1024, bytes_per_element=4, compute_rate=cr, seed=0))
    cap = G.llama_peak_bytes(tr) // 2
    g = plan_device(tr, cap, rates, hc)
    print("C1", hashlib.sha256(g["plan_bytes"]).hexdigest()[:8], exp, flush=True)

tr = G.gen_llama_trace(G.LLAMA3_8B)
a = tr.arrays()
cap = G.llama_peak_bytes(tr) // 2
dt = _native.DeviceTrace(a)
t0 = time.time(); lt = dt.lifetime(); t1 = time.time()
per, tl, act = O.lifetime(a)
print("C2 lifetime", t1 - t0, np.array_equal(lt["timeline"], tl), np.array_equal(lt["active"], act),
      np.array_equal(lt["period_tensor"], per["tensor"]), np.array_equal(lt["period_start"], per["start"]), flush=True)
for rep in range(2):
    t0 = time.time()
    p = dt.plan(cap, _native.Rates(16000.0, 16000.0, 0, 0.0, 0.0), 0)
    t1 = time.time()
    b = p.write()
    print("C2 plan", t1 - t0, "s rounds", p.info.rounds, "commits", p.info.num_commits,
          hashlib.sha256(b).hexdigest(), flush=True)
    p.close()
print("expect 3c54a7c3e2cd90e4b49bf4eb162f8223c7ccc6d64e0e81acbc945492fab3348f")
