"""Multi-process (gloo, world size 2 and 3, CPU) test of the tensor-id
sharded lifetime stage (paper_2506_06472_b200/distributed.py): the merged
timeline, active bytes and period list equal the unsharded result.  The
per-shard compute here is the CPU oracle (the GPU path runs the libtio
kernel per shard; the host-side sharding, the all_reduce and the all_gather
merge are what this test covers)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_local(sub):
    from oracle import oracle as O
    per, tl, act = O.lifetime(sub)
    return {"timeline": tl, "active": act, "period_tensor": per["tensor"], "period_start": per["start"],
            "period_end": per["end"], "period_wraps": per["wraps"].astype(np.int8)}


def _worker(rank, world, port, cases, q, device_kernels=False):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    from paper_2506_06472_b200 import gen_random_trace, LlamaTraceConfig, gen_llama_trace
    from paper_2506_06472_b200.distributed import sharded_lifetime
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for kind, arg in cases:
            tr = gen_llama_trace(LlamaTraceConfig(microbatches=arg)) if kind == "llama" else \
                gen_random_trace(arg, 3 + arg % 50, 1 + arg % 37)
            if device_kernels:      # libtio lifetime kernels per shard on cuda:0
                import torch
                torch.cuda.set_device(0)
                r = sharded_lifetime(tr.arrays(), rank, world, device=torch.device("cuda", 0))
            else:
                r = sharded_lifetime(tr.arrays(), rank, world, local_fn=_oracle_local)
            if device_kernels:      # device-resident columns (never left HBM during the exchange)
                assert all(r[k].is_cuda for k in ("timeline", "active", "period_tensor"))
            out.append({k: (v.tolist() if isinstance(v, np.ndarray) else
                            v.cpu().tolist() if hasattr(v, "cpu") else v) for k, v in r.items()})
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_lifetime_equals_unsharded(world):
    from oracle import oracle as O
    from paper_2506_06472_b200 import gen_random_trace, LlamaTraceConfig, gen_llama_trace
    cases = [("random", s) for s in (1, 7, 42, 99, 123)] + [("llama", 1), ("llama", 2)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (kind, arg) in enumerate(cases):
        tr = gen_llama_trace(LlamaTraceConfig(microbatches=arg)) if kind == "llama" else \
            gen_random_trace(arg, 3 + arg % 50, 1 + arg % 37)
        per, tl, act = O.lifetime(tr.arrays())
        for r in range(world):
            got = results[r][ci]
            assert got["timeline"] == tl.tolist()
            assert got["active"] == act.tolist()
            assert got["period_tensor"] == per["tensor"].tolist()
            assert got["period_start"] == per["start"].tolist()
            assert got["period_end"] == per["end"].tolist()
            assert got["period_wraps"] == per["wraps"].astype(int).tolist()


@pytest.mark.gpu
def test_sharded_lifetime_device_kernels_equals_oracle():
    """The same exchange with the libtio kernels computing each shard on the
    GPU (two ranks sharing cuda:0 over gloo; one GPU per rank would use NCCL)."""
    from oracle import oracle as O
    from paper_2506_06472_b200 import gen_random_trace, LlamaTraceConfig, gen_llama_trace
    world = 2
    cases = [("random", s) for s in (3, 11)] + [("llama", 2)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q, True)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (kind, arg) in enumerate(cases):
        tr = gen_llama_trace(LlamaTraceConfig(microbatches=arg)) if kind == "llama" else \
            gen_random_trace(arg, 3 + arg % 50, 1 + arg % 37)
        per, tl, act = O.lifetime(tr.arrays())
        for r in range(world):
            got = results[r][ci]
            assert got["timeline"] == tl.tolist() and got["active"] == act.tolist()
            assert got["period_tensor"] == per["tensor"].tolist()
            assert got["period_start"] == per["start"].tolist() and got["period_end"] == per["end"].tolist()


def test_shard_bounds_balanced_and_contiguous():
    from paper_2506_06472_b200.distributed import shard_bounds
    ptr = np.cumsum([0] + [3, 1, 4, 1, 5, 9, 2, 6, 5, 3])
    for world in (1, 2, 3, 4, 8, 16):
        b = shard_bounds(ptr, world)
        assert b[0][0] == 0 and b[-1][1] == 10
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))


# ---------------------------------------------------------------- planner exchange
def _kbetter(x, y):
    """The device key order (csrc/planner.cuh kbetter; planner.py:309 and
    App. A-12): larger benefit/cost ratio wins (exact cross products), ties go
    to the lower candidate index; a zero benefit never wins."""
    (bx, cx, ix), (by, cy, iy) = x, y
    if bx == 0:
        return False
    if by == 0:
        return True
    if bx * cy != by * cx:
        return bx * cy > by * cx
    return ix < iy


def _exchange_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import random
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = 0
        for seed in range(300):
            rng = random.Random(seed)
            P = rng.randrange(1, 200)
            # candidates with many exact ratio ties and benefits past 2^64
            keys = [(rng.choice([0, 3, 6, 2**70, 3 * 2**66]) * rng.randrange(1, 4), rng.choice([2, 4, 8]), i)
                    for i in range(P)]
            tiles = [list(range(t, min(t + 32, P))) for t in range(0, P, 32)]
            local = (0, 1, -1)
            for t, members in enumerate(tiles):
                if t % world != rank:          # tile t belongs to rank t mod R
                    continue
                for c in members:
                    if _kbetter(keys[c], local):
                        local = keys[c]
            # the round message: every rank's local best, gathered (the device
            # version writes it into every peer's mailbox)
            enc = torch.tensor([local[0] >> 64, local[0] & (2**63 - 1), (local[0] >> 63) & 1, local[1], local[2]],
                               dtype=torch.int64)
            allm = [torch.zeros_like(enc) for _ in range(world)]
            dist.all_gather(allm, enc)
            best = (0, 1, -1)
            for m in allm:
                hi, lo, b63, c, i = (int(v) for v in m.tolist())
                k = ((hi << 64) | (b63 << 63) | lo, c, i)
                if _kbetter(k, best):
                    best = k
            brute = (0, 1, -1)
            for k in keys:
                if _kbetter(k, brute):
                    brute = k
            assert best == brute, (seed, best, brute)
            ok += 1
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_round_winner_exchange_picks_the_global_argmax(world):
    """The sharded planner's per-round protocol on gloo: ranks own the
    candidate tiles t mod R, exchange their local best and take the best of
    the R messages — the result is the reference's global argmax
    (planner.py:295-310, strict > in candidate order) on 300 random rounds
    with exact-ratio ties and 2^64+ benefits."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(v == 300 for v in res.values())
