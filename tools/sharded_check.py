"""Two ranks on one GPU (gloo; NCCL needs one GPU per rank) running bench.py's
sharded-lifetime leg: libtio per shard + all_reduce/all_gather merge, checked
against the whole-trace lifetime.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/sharded_check.py [c2|c3]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    r = bench.sharded_lifetime_leg(sys.argv[1] if len(sys.argv) > 1 else "c2", torch.device("cuda", 0), rank, world)
    if rank == 0:
        print(json.dumps(r))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
