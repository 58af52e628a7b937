"""GPU: the sharded planner (north star: "the trace shards by
tensor id across the GPUs ... allgather for the merged plan").

Candidate tiles are split over ranks (tile t belongs to rank t % R); every
rank keeps the whole replicated planner state, evaluates only its own tiles,
publishes its round's best (key + window) into every rank's mailbox, takes
the best of the R messages (ratio, then lowest candidate index) and applies
the same commit — so every rank ends with the whole plan.  On one B200 the R
ranks run as R concurrent planner instances (own state, own stream, own
cooperative grid of SMs / R blocks) exchanging through device memory: the
same kernel and protocol as the multi-GPU run, where the mailboxes are
CUDA-IPC mappings of the peers' memory.  Bar: every rank's plan bytes and
residual timeline are bit-identical to the single-rank plan and to the
reference / oracle fingerprints."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import load_golden, rates_of, regen
from paper_2506_06472_b200 import ChannelRates, gen_random_trace, plan_device
from paper_2506_06472_b200.planner import plan_device_virtual

pytestmark = pytest.mark.gpu


def _same(outs, ref_bytes, ref_resid):
    for r, o in enumerate(outs):
        assert o["plan_bytes"] == ref_bytes, f"rank {r} plan differs"
        assert np.array_equal(o["residual"], ref_resid), f"rank {r} residual differs"


def _golden_traces():
    from paper_2506_06472_b200 import LlamaTraceConfig, TransformerGenConfig, gen_llama_trace, gen_transformer_trace
    for rec in load_golden("c1"):
        cfg = TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8, seq_len=1024,
                                   bytes_per_element=4, compute_rate=rec["gen"]["compute_rate"], seed=0)
        yield gen_transformer_trace(cfg), rec
    rec = load_golden("llama1")[0]
    yield gen_llama_trace(LlamaTraceConfig(microbatches=1)), rec


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_virtual_ranks_match_reference_goldens(nranks):
    """C1 (4 rate setups) and the 1-microbatch Llama trace (625 commits):
    plan bytes made by the reference itself (tests/golden)."""
    n = 0
    for tr, rec in _golden_traces():
        outs = plan_device_virtual(tr, rec["capacity"], rates_of(rec), rec["host_cap"], nranks)
        for o in outs:
            assert hashlib.sha256(o["plan_bytes"]).hexdigest() == rec["plan_sha256"]
            assert o["residual"].tolist() == rec["residual"]
        n += 1
    assert n == 5


def test_virtual_ranks_on_the_crit2_corpus():
    """The reference's criterion-2 corpus (tests/golden/crit2, plans made by
    the reference) at 2 and 3 ranks."""
    n = 0
    for i, rec in enumerate(load_golden("crit2")):
        if "plan" not in rec or i % 10:
            continue
        tr = regen(rec)
        for nranks in (2, 3):
            for o in plan_device_virtual(tr, rec["capacity"], rates_of(rec), rec.get("host_cap", 0), nranks):
                assert o["plan_bytes"].decode() == rec["plan"]
        n += 1
    assert n >= 50


@pytest.mark.parametrize("nranks", [2, 4])
def test_virtual_ranks_on_random_traces_with_host_tier(nranks):
    for seed in range(12):
        tr = gen_random_trace(9000 + seed, 40 + 5 * seed, 60, size_range=(1_000_000, 80_000_000),
                              duration_range=(50, 4_000))
        from paper_2506_06472_b200 import compute_memory_timeline
        cap = int(compute_memory_timeline(tr).peak() * 0.55)
        rates = ChannelRates.symmetric(3_000, host=9_000) if seed % 2 else ChannelRates.symmetric(5_000)
        hc = 2 * 10**9 if seed % 2 else 0
        try:
            one = plan_device(tr, cap, rates, hc)
        except Exception:
            continue
        outs = plan_device_virtual(tr, cap, rates, hc, nranks)
        _same(outs, one["plan_bytes"], one["residual"])


@pytest.mark.parametrize("nranks", [2, 4])
def test_virtual_ranks_c2_full_plan(nranks):
    """Config C2 (1.0M events, 32,879 commits): every rank's plan equals the
    oracle's fingerprint."""
    from paper_2506_06472_b200 import LLAMA3_8B, gen_llama_trace
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    rec = load_golden("c2")
    tr = gen_llama_trace(LLAMA3_8B)
    cap = llama_peak_bytes(tr) // 2
    outs = plan_device_virtual(tr, cap, ChannelRates.symmetric(16_000), 0, nranks)
    for o in outs:
        assert hashlib.sha256(o["plan_bytes"]).hexdigest() == rec["plan_sha256"]
        assert hashlib.sha256(o["residual"].tobytes()).hexdigest() == rec["residual_sha256"]


# ---------------------------------------------------------------- processes
def _proc_worker(rank, world, port, q):
    """One rank in its own process: gloo for the IPC-handle exchange (two
    ranks cannot share a GPU under NCCL), mailboxes mapped over CUDA IPC,
    libtio's sharded planner on cuda:0 (the ranks time-share the device)."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_2506_06472_b200 import _native
    from paper_2506_06472_b200.distributed import PlanGroup
    from paper_2506_06472_b200.planner import _rates_struct
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = PlanGroup(rank, world)
        out = []
        for tr, rec in _golden_traces():
            dt = _native.DeviceTrace(tr.arrays())
            # two consecutive calls over the same mailboxes (epochs advance)
            for _ in range(2):
                p = g.plan(dt, rec["capacity"], _rates_struct(rates_of(rec)), rec["host_cap"])
                b = p.write()
                resid = p.copy_out()["residual"]
                out.append((hashlib.sha256(b).hexdigest(), resid.tolist(), g.plans_agree(b)))
                p.close()
            dt.close()
        dist.barrier()
        g.close()
        q.put((rank, out, None))
    except Exception as exc:  # reported to the parent
        q.put((rank, None, f"{type(exc).__name__}: {exc}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_processes_ipc_mailboxes_match_reference_goldens():
    """The multi-process path of the sharded planner (PlanGroup: device
    mailboxes exchanged as CUDA IPC handles, one process per rank) on one
    B200: both ranks' plans equal the reference goldens, twice in a row."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, out, err = q.get(timeout=540)
        assert err is None, f"rank {r}: {err}"
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    recs = [rec for _, rec in _golden_traces() for _ in range(2)]
    for r in (0, 1):
        assert len(res[r]) == len(recs)
        for (sha, resid, agree), rec in zip(res[r], recs):
            assert sha == rec["plan_sha256"]
            assert resid == rec["residual"]
            assert agree
