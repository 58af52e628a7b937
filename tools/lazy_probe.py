"""Run tools/lazy_probe.c (lazy greedy) in place of the oracle planner and
compare plan bytes with the oracle / golden fingerprints.  Experiment only.

    python tools/lazy_probe.py [c1|llama1|crit2|c2|c3]
"""
import ctypes
import gzip
import hashlib
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = "/tmp/lazy_probe.so"
subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wno-unused-function", "-o", SO,
                os.path.join(ROOT, "tools", "lazy_probe.c")], check=True)
from oracle import oracle as O  # noqa: E402

lazy = ctypes.CDLL(SO)
lazy.tio_lazy_stats.restype = ctypes.POINTER(ctypes.c_int64)


class Shim:
    def __init__(self, real):
        self.real = real

    def __getattr__(self, k):
        if k == "tio_oracle_plan":
            return lazy.tio_lazy_plan
        return getattr(self.real, k)


def run(a, cap, r, host=None, hc=0):
    real = O.lib()
    O._lib = Shim(real)
    try:
        t0 = time.time()
        p = O.plan(a, cap, r, r, host, host, hc)
        dt = time.time() - t0
    finally:
        O._lib = real
    st = lazy.tio_lazy_stats()
    return p, dt, (st[0], st[1], st[2])


def main(cfg):
    from paper_2506_06472_b200 import tracegen as G
    if cfg in ("c2", "c3"):
        tr = G.gen_llama_trace(G.LLAMA3_8B if cfg == "c2" else G.LLAMA3_70B)
        a = tr.arrays()
        cap = G.llama_peak_bytes(tr) // 2
        p, dt, st = run(a, cap, 16000.0)
        gold = os.path.join(ROOT, "tests", "golden", f"{cfg}.json.gz")
        want = json.load(gzip.open(gold, "rt"))["plan_sha256"] if os.path.exists(gold) else None
        got = hashlib.sha256(p["plan_bytes"]).hexdigest()
        print(cfg, "commits", len(p["committed"]), "pops", st[0], "evals", st[1], "host evals", st[2],
              f"{dt:.1f}s", "sha match" if got == want else f"sha {got[:12]} want {str(want)[:12]}")
        return
    if cfg == "llama1":
        tr = G.gen_llama_trace(G.LlamaTraceConfig(microbatches=1))
        a = tr.arrays()
        cap = G.llama_peak_bytes(tr) // 2
        for host in (None, 32000.0):
            p, dt, st = run(a, cap, 16000.0, host, 8 * 10**9 if host else 0)
            o = O.plan(a, cap, 16000.0, 16000.0, host, host, 8 * 10**9 if host else 0)
            print(cfg, host, "commits", len(p["committed"]), "pops", st[0], "evals", st[1],
                  "match" if p["plan_bytes"] == o["plan_bytes"] else "MISMATCH")
        return


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "llama1")
