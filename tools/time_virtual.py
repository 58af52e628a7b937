"""Time the sharded planner's virtual ranks on one GPU (tio_plan_create_virtual):
python tools/time_virtual.py c3|c2 [nranks ...]  — wall time of the call,
rounds, us/round and whether every rank's plan equals the golden sha256."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2506_06472_b200.planner import plan_device_virtual, plan_device
    cfg = sys.argv[1]
    ranks = [int(x) for x in sys.argv[2:]] or [1, 2, 4]
    tr, cap, rates, hc, desc = bench._trace(cfg)
    for R in ranks:
        for rep in range(2):
            t0 = time.perf_counter()
            outs = [plan_device(tr, cap, rates, hc)] if R == 1 else plan_device_virtual(tr, cap, rates, hc, R)
            dt = time.perf_counter() - t0
        shas = {hashlib.sha256(o["plan_bytes"]).hexdigest()[:16] for o in outs}
        info = outs[0]["info"]
        print(json.dumps({"config": cfg, "nranks": R, "wall_s": dt, "rounds": int(info.rounds),
                          "loop_ms_rank0": info.loop_ns / 1e6, "us_per_round": info.loop_ns / 1e3 / max(1, info.rounds),
                          "plan_sha16": sorted(shas)}), flush=True)


if __name__ == "__main__":
    main()
