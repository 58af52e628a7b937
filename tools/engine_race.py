"""Debug: replay the first corpus cases that fail byte verification under variants."""
import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import load_golden, regen, rates_of
from paper_2506_06472_b200 import engine
from paper_2506_06472_b200.planner import parse_plan
sims = load_golden("sim"); plans = {r["trace_sha256"]: r for r in load_golden("crit2")}
bad = []
for i, rec in enumerate(sims[:200]):
    base = plans[rec["trace_sha256"]]
    if "plan" not in base or "error" in rec["plan"]:
        continue
    tr = regen(rec); entries = parse_plan(base["plan"])[1]
    r = engine.replay(tr, entries, base["capacity"], rates_of(base), time_scale=float(os.environ.get("TS", "0.002")))
    if r.verify_mismatches:
        bad.append((i, r.verify_mismatches, r.emergency_offloads, r.n_offloads, r.n_prefetches, base["rates"]))
print("variant", os.environ.get("TIO_POOL_STRICT"), os.environ.get("TS"), "bad cases:", len(bad), bad[:8])
