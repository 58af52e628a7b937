"""Multi-GPU lifetime stage: the trace sharded by tensor id.

Periods are per-tensor, and the memory timeline and active bytes are sums
over tensors, so the lifetime stage (reference analysis.py:58-117) shards
exactly: rank r owns a contiguous range of tensors (balanced by access
events), runs the libtio lifetime kernel on its shard (all kernel durations
replicated), then

  * all_reduce(SUM, int64[N]) of its partial timeline and active bytes
    (exact integer sums; each global counts once, in its owner's shard);
  * all_gather of its period list (counts first, then padded columns);
    concatenated in rank order this is the reference order (tensor order,
    gaps ascending, wrap last) because the shards are contiguous in trace
    order.

The planner's commits are a single sequential greedy over all candidates
(planner.py:293-351); every rank plans on the merged lifetime products and
the plans are identical (checked with an all_gather of the plan hash).

Collectives go through torch.distributed: NCCL over NVLink on the GPU box,
gloo on CPU for the tests.  `local_fn` computes one shard's lifetime; the
default is the libtio kernel.
"""

from __future__ import annotations

import numpy as np

from .trace import TraceArrays


def shard_bounds(access_ptr: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous tensor ranges [t0, t1) with about E / world events each."""
    T = access_ptr.shape[0] - 1
    E = int(access_ptr[-1])
    cuts = [0]
    for r in range(1, world):
        target = E * r // world
        cuts.append(int(np.searchsorted(access_ptr, target, side="left")))
    cuts.append(T)
    cuts = [min(max(c, 0), T) for c in cuts]
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def shard_arrays(a: TraceArrays, t0: int, t1: int) -> TraceArrays:
    """Every kernel, tensors [t0, t1) only."""
    e0, e1 = int(a.access_ptr[t0]), int(a.access_ptr[t1])
    return TraceArrays(
        duration_us=a.duration_us, kernel_index=a.kernel_index, kernel_name_code=a.kernel_name_code,
        name_table=a.name_table, kernel_stage=a.kernel_stage, kernel_layer=a.kernel_layer,
        tensor_id=a.tensor_id[t0:t1], size_bytes=a.size_bytes[t0:t1], kind=a.kind[t0:t1],
        tensor_layer=a.tensor_layer[t0:t1], access_ptr=a.access_ptr[t0:t1 + 1] - e0,
        accesses=a.accesses[e0:e1])


def _device_lifetime(sub: TraceArrays) -> dict:
    from . import _native
    dt = _native.DeviceTrace(sub)
    try:
        return dt.lifetime()
    finally:
        dt.close()


def sharded_lifetime(a: TraceArrays, rank: int, world: int, group=None, local_fn=None, device=None) -> dict:
    """The lifetime products of the whole trace, computed shard-wise.

    Returns numpy columns: timeline, active (int64[N]) and the periods in
    reference order (tensor position, start, end, wraps), plus `shard`.
    """
    import torch
    import torch.distributed as dist

    local_fn = local_fn or _device_lifetime
    t0, t1 = shard_bounds(a.access_ptr, world)[rank]
    loc = local_fn(shard_arrays(a, t0, t1))
    N = a.num_kernels
    dev = device if device is not None else torch.device("cpu")
    # one exchange step: partial sums of the timeline and active bytes
    sums = torch.from_numpy(np.concatenate([np.asarray(loc["timeline"], np.int64),
                                            np.asarray(loc["active"], np.int64)])).to(dev)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    sums = sums.cpu().numpy()
    # periods: counts, then padded columns (tensor position is made global)
    p = np.asarray(loc["period_tensor"], np.int64) + t0
    cols = np.stack([p, np.asarray(loc["period_start"], np.int64), np.asarray(loc["period_end"], np.int64),
                     np.asarray(loc["period_wraps"], np.int64)]) if p.size else np.zeros((4, 0), np.int64)
    cnt = torch.tensor([cols.shape[1]], dtype=torch.int64, device=dev)
    cnts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    counts = [int(c.item()) for c in cnts]
    width = max(counts) if counts else 0
    pad = np.zeros((4, width), np.int64)
    pad[:, :cols.shape[1]] = cols
    mine = torch.from_numpy(pad).to(dev)
    outs = [torch.zeros((4, width), dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(outs, mine, group=group)
    merged = np.concatenate([o.cpu().numpy()[:, :c] for o, c in zip(outs, counts)], axis=1) \
        if width else np.zeros((4, 0), np.int64)
    return {"timeline": sums[:N], "active": sums[N:], "period_tensor": merged[0],
            "period_start": merged[1].astype(np.int32), "period_end": merged[2].astype(np.int32),
            "period_wraps": merged[3].astype(np.int8), "shard": (t0, t1), "counts": counts}
