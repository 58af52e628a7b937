"""Multi-GPU lifetime + plan: one process per GPU.

Lifetime stage, sharded by tensor id.  Periods are per-tensor, and the
memory timeline and active bytes are sums over tensors, so the lifetime
stage (reference analysis.py:58-117) shards exactly: rank r owns a
contiguous range of tensors (balanced by access events), runs the libtio
lifetime kernels on its shard (all kernel durations replicated), then

  * all_reduce(SUM, int64[2N]) of its partial timeline and active bytes
    (exact integer sums; each global counts once, in its owner's shard);
  * all_gather of its period list (counts first, then padded columns);
    concatenated in rank order this is the reference order (tensor order,
    gaps ascending, wrap last) because the shards are contiguous in trace
    order.

On CUDA devices the whole exchange stays in HBM (the shard's lifetime
products are read through the handle's device views, the collectives run on
device tensors); on CPU (gloo, the tests) the columns are numpy.

Planner, sharded by candidate tile (`PlanGroup`).  Algorithm 1's commits are
one sequential greedy (planner.py:293-351), but the per-round candidate scan
(:295-310) shards: every rank holds the replicated planner state (channel
bookings, residual, critical-duration prefix) and evaluates only its own
candidate tiles (tile t belongs to rank t mod R).  Each round the
last-arriving block of every rank's persistent kernel puts its local best
(the 192-bit key + the winner's window, 112 B) into every rank's mailbox
over NVLink (CUDA IPC mappings of each rank's device mailbox, release/acquire
at system scope) and takes the best of the R messages — the same winner on
every rank, ties to the lowest candidate index (App. A-12) — then every rank
applies the same commit.  Every rank therefore ends with the whole plan; the
plans are checked equal with an all_gather of their sha256.

Collectives go through torch.distributed: NCCL over NVLink on the GPU box,
gloo on CPU for the tests.  `local_fn` computes one shard's lifetime; the
default is the libtio kernel.
"""

from __future__ import annotations

import hashlib

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


class _DevCol:
    """__cuda_array_interface__ over a libtio device view column."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def _device_lifetime_torch(sub: TraceArrays, device) -> dict:
    """One shard's lifetime products as device tensors (cloned out of the
    handle's views: no host round trip)."""
    import ctypes
    import torch
    from . import _native
    lib = _native.load()
    stream = torch.cuda.current_stream(device)
    dt = _native.DeviceTrace(sub, stream=stream.cuda_stream)
    try:
        _native.check(lib.tio_lifetime(dt.handle, ctypes.c_void_p(stream.cuda_stream)))
        v = _native.LifetimeView()
        _native.check(lib.tio_lifetime_view_get(dt.handle, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(v)))
        n, p = int(v.num_kernels), int(v.num_periods)

        def col(ptr, m, ts):
            if m == 0 or not ptr:
                return torch.zeros(m, dtype={"<i8": torch.int64, "<i4": torch.int32, "|i1": torch.int8}[ts],
                                   device=device)
            return torch.as_tensor(_DevCol(int(ptr), m, ts), device=device).clone()
        out = {"timeline": col(v.timeline, n, "<i8"), "active": col(v.active, n, "<i8"),
               "period_tensor": col(v.period_tensor, p, "<i8"), "period_start": col(v.period_start, p, "<i4"),
               "period_end": col(v.period_end, p, "<i4"), "period_wraps": col(v.period_wraps, p, "|i1")}
        torch.cuda.current_stream(device).synchronize()
        return out
    finally:
        dt.close()


def sharded_lifetime(a: TraceArrays, rank: int, world: int, group=None, local_fn=None, device=None) -> dict:
    """The lifetime products of the whole trace, computed shard-wise.

    Returns timeline, active (int64[N]) and the periods in reference order
    (tensor position, start, end, wraps), plus `shard` and `counts`.  With a
    CUDA `device` and the default kernel the columns are device tensors and
    never leave HBM; otherwise numpy columns.
    """
    import torch
    import torch.distributed as dist

    dev = device if device is not None else torch.device("cpu")
    on_device = local_fn is None and dev.type == "cuda"
    t0, t1 = shard_bounds(a.access_ptr, world)[rank]
    sub = shard_arrays(a, t0, t1)
    N = a.num_kernels
    if on_device:
        loc = _device_lifetime_torch(sub, dev)
        sums = torch.cat([loc["timeline"], loc["active"]])
        cols = torch.stack([loc["period_tensor"] + t0, loc["period_start"].long(), loc["period_end"].long(),
                            loc["period_wraps"].long()]) if loc["period_tensor"].numel() else \
            torch.zeros((4, 0), dtype=torch.int64, device=dev)
    else:
        loc = (local_fn or _device_lifetime)(sub)
        sums = torch.from_numpy(np.concatenate([np.asarray(loc["timeline"], np.int64),
                                                np.asarray(loc["active"], np.int64)])).to(dev)
        p = np.asarray(loc["period_tensor"], np.int64) + t0
        cols = torch.from_numpy(np.stack([p, np.asarray(loc["period_start"], np.int64),
                                          np.asarray(loc["period_end"], np.int64),
                                          np.asarray(loc["period_wraps"], np.int64)])
                                if p.size else np.zeros((4, 0), np.int64)).to(dev)
    # one exchange step: partial sums of the timeline and active bytes
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    # periods: counts, then padded columns (tensor position is made global)
    cnt = torch.tensor([cols.shape[1]], dtype=torch.int64, device=dev)
    cnts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    counts = [int(c.item()) for c in cnts]
    width = max(counts) if counts else 0
    pad = torch.zeros((4, width), dtype=torch.int64, device=dev)
    pad[:, :cols.shape[1]] = cols
    outs = [torch.zeros((4, width), dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    merged = torch.cat([o[:, :c] for o, c in zip(outs, counts)], dim=1) if width else \
        torch.zeros((4, 0), dtype=torch.int64, device=dev)
    res = {"timeline": sums[:N], "active": sums[N:], "period_tensor": merged[0],
           "period_start": merged[1].to(torch.int32), "period_end": merged[2].to(torch.int32),
           "period_wraps": merged[3].to(torch.int8)}
    if not on_device:
        res = {k: v.cpu().numpy() for k, v in res.items()}
    res["shard"] = (t0, t1)
    res["counts"] = counts
    return res


class PlanGroup:
    """Sharded planning over the ranks of a torch.distributed group (one
    process per GPU).  Creates this rank's device mailbox, exchanges the CUDA
    IPC handles (all_gather) and maps every peer's mailbox once; `plan` then
    runs libtio's sharded planner on a DeviceTrace of the whole trace.

    Every rank must call `plan` with the same trace and arguments, in the
    same order (the calls are matched by their epochs)."""

    def __init__(self, rank: int, world: int, group=None):
        import torch
        import torch.distributed as dist
        from . import _native
        self.rank, self.world, self.group = rank, world, group
        self.mailbox = _native.Mailbox()
        mine = torch.frombuffer(bytearray(self.mailbox.handle), dtype=torch.uint8)
        dev = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(group) == "nccl" else torch.device("cpu")
        mine = mine.to(dev)
        allh = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allh, mine, group=group)
        self.peers: list[int] = []
        self._mapped: list[int] = []
        for r, h in enumerate(allh):
            if r == rank:
                self.peers.append(int(self.mailbox.ptr.value))
            else:
                ptr = _native.mailbox_open(bytes(h.cpu().numpy().tobytes()))
                self._mapped.append(ptr)
                self.peers.append(ptr)
        self.epoch = 0
        dist.barrier(group=group)

    def plan(self, dt, capacity: int, rates, host_cap: int = 0, max_rounds: int = 0):
        """This rank's DevicePlan of the whole trace (every rank's is the
        same plan).  `rates` is a _native.Rates struct."""
        p = dt.plan(capacity, rates, host_cap, max_rounds,
                    shard=(self.rank, self.world, int(self.mailbox.ptr.value), self.peers, self.epoch))
        self.epoch += int(p.info.rounds) + 2
        return p

    def plans_agree(self, plan_bytes: bytes) -> bool:
        """all_gather of the plan sha256: True iff every rank holds the same
        plan bytes."""
        import torch
        import torch.distributed as dist
        h = torch.frombuffer(bytearray(hashlib.sha256(plan_bytes).digest()), dtype=torch.uint8)
        if dist.get_backend(self.group) == "nccl":
            h = h.to(torch.device("cuda", torch.cuda.current_device()))
        allh = [torch.zeros_like(h) for _ in range(self.world)]
        dist.all_gather(allh, h, group=self.group)
        return all(torch.equal(x.cpu(), allh[0].cpu()) for x in allh)

    def close(self) -> None:
        """Unmap the peers' mailboxes and free this rank's.  Collective: every
        rank calls it (a barrier first, so no rank frees a mailbox a peer is
        still writing into)."""
        import torch.distributed as dist
        from . import _native
        if dist.is_initialized():
            dist.barrier(group=self.group)
        for ptr in self._mapped:
            try:
                _native.mailbox_close(ptr)
            except Exception:
                pass
        self._mapped = []
        if self.mailbox is not None:
            self.mailbox.close()
            self.mailbox = None
