"""Fingerprints of the C2 / C3 plans computed by the CPU oracle (slow: tens
of minutes on 8 cores each; run once in the build container).

    python tests/golden/make_c2.py [c2|c3|c2host|c3host]

`*host` adds the host tier of SURVEY §8(d): host 50,000 B/us both ways,
host_cap 256e9 (output: tests/golden/<config>.json.gz).

The reference planner cannot run at C2 (~8 h per round), so the
C2/C3 checker is the oracle (oracle/tio_oracle.c), whose bit-exactness against
the reference is pinned by tests/test_oracle_golden.py on the fuzz corpora,
C1 and the 1-microbatch Llama trace.  Output: tests/golden/<config>.json.gz.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)


def main(config: str = "c2", max_rounds: int = 0):
    from oracle import oracle as O
    from paper_2506_06472_b200 import LLAMA3_8B, LLAMA3_70B, gen_llama_trace, write_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    host = config.endswith("host")
    tr = gen_llama_trace({"c2": LLAMA3_8B, "c3": LLAMA3_70B}[config[:2]])
    a = tr.arrays()
    cap = llama_peak_bytes(tr) // 2
    rates = [16000, 16000, 50000, 50000] if host else [16000, 16000, None, None]
    host_cap = 256 * 10**9 if host else 0
    t0 = time.time()
    if host:
        p = O.plan(a, cap, 16000.0, 16000.0, 50000.0, 50000.0, host_cap, verbose=True, max_rounds=max_rounds)
    else:
        p = O.plan(a, cap, 16000.0, 16000.0, verbose=True, max_rounds=max_rounds)
    rec = {
        "trace_sha256": hashlib.sha256(write_trace(tr)).hexdigest(),
        "num_events": a.num_events, "capacity": cap, "rates": rates, "host_cap": host_cap,
        "rounds": int(p["rounds"]), "num_commits": len(p["committed"]),
        "plan_sha256": hashlib.sha256(p["plan_bytes"]).hexdigest(),
        "residual_sha256": hashlib.sha256(p["residual"].astype("<i8").tobytes()).hexdigest(),
        "over_capacity_kernels": len(p["over_capacity_kernels"]),
        "host_commits": int(sum(1 for c in p["committed"] if c[4] == "CPU")),
        "planned_host_bytes": int(p["planned_host_bytes"]),
        "oracle_seconds": round(time.time() - t0, 1), "oracle_threads": int(O.lib().tio_oracle_threads()),
    }
    out_dir = os.environ.get("TIO_GOLDEN_OUT", HERE)       # e.g. gpurun_out/ when run on the GPU box's host
    os.makedirs(out_dir, exist_ok=True)
    if max_rounds:
        rec["max_rounds"] = max_rounds          # a prefix of the greedy sequence (planner.py:293-351)
    name = f"{config}_prefix{max_rounds}" if max_rounds else config
    with gzip.open(os.path.join(out_dir, f"{name}.json.gz"), "wt") as f:
        json.dump(rec, f)
    print(rec)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c2", int(sys.argv[2]) if len(sys.argv) > 2 else 0)
