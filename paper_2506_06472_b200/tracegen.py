"""Synthetic trace sources.

* `gen_transformer_trace` / `transformer_peak_bytes` / `gen_random_trace`:
  the reference generators (`offloader/tracegen.py:72-186`), restated so the
  same arguments give the same trace (C1 and the fuzz corpora depend on it).
* `gen_llama_trace`: the per-op Llama-shaped iteration of SURVEY.md
  Appendix C (configs C2 = Llama-3-8B shape, ~1M events, and C3 = Llama-3-70B
  shape, ~10M events).  Every microbatch has the same op structure, so one
  microbatch is built as a template and tiled with numpy; the result is a
  column-form `Trace` that never materialises per-event Python objects.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from .trace import (KIND_GLOBAL, KIND_INTERMEDIATE, NONE_I64, KernelRecord, TensorKind,
                    TensorRecord, Trace, TraceArrays, make_trace)

# per-layer sizing constants of the reference generator (tracegen.py:21-32)
ATTN_WEIGHT_ELEMS = 4
MLP_WEIGHT_ELEMS = 8
OPT_STATE_FACTOR = 2
ATTN_ACT_ELEMS = 2
MLP_ACT_ELEMS = 6


@dataclass(frozen=True)
class TransformerGenConfig:
    num_layers: int = 12
    hidden_dim: int = 4096
    num_heads: int = 32
    batch: int = 8
    seq_len: int = 1024
    bytes_per_element: int = 4
    pipeline_stages: int = 1
    compute_rate: int = 1_000_000_000
    optimizer_intensity: int = 25
    seed: int = 0

    def __post_init__(self):
        for name in ("num_layers", "hidden_dim", "num_heads", "batch", "seq_len",
                     "bytes_per_element", "pipeline_stages", "compute_rate",
                     "optimizer_intensity"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def gen_transformer_trace(cfg: TransformerGenConfig) -> Trace:
    """Decoder-block-shaped iteration (reference tracegen.py:72-149):
    L attention+MLP forward kernel pairs, the backward pairs in reverse layer
    order, then one optimizer kernel per layer.  Per layer: 6 global tensors
    (attn/mlp weights, their grads, their two-moment optimizer states) and
    two activations each used by one forward and the matching backward kernel.
    """
    L = cfg.num_layers
    h = cfg.hidden_dim
    tokens = cfg.batch * cfg.seq_len
    attn_flops = 8 * tokens * h * h + 4 * cfg.batch * cfg.seq_len ** 2 * h
    mlp_flops = 16 * tokens * h * h
    layer_params = (ATTN_WEIGHT_ELEMS + MLP_WEIGHT_ELEMS) * h * h

    def dur(flops: int) -> int:
        return max(1, _ceil_div(flops, cfg.compute_rate))

    # kernel index of each op
    fwd_attn = [2 * i for i in range(L)]
    fwd_mlp = [2 * i + 1 for i in range(L)]
    bwd_mlp = [2 * L + 2 * (L - 1 - i) for i in range(L)]
    bwd_attn = [2 * L + 2 * (L - 1 - i) + 1 for i in range(L)]
    opt = [4 * L + i for i in range(L)]

    def stage(i: int) -> int:
        return i * cfg.pipeline_stages // L

    slots: dict[int, KernelRecord] = {}
    for i in range(L):
        slots[fwd_attn[i]] = KernelRecord(fwd_attn[i], f"attn_fwd_{i}", dur(attn_flops), stage(i), i)
        slots[fwd_mlp[i]] = KernelRecord(fwd_mlp[i], f"mlp_fwd_{i}", dur(mlp_flops), stage(i), i)
        slots[bwd_mlp[i]] = KernelRecord(bwd_mlp[i], f"mlp_bwd_{i}", dur(2 * mlp_flops), stage(i), i)
        slots[bwd_attn[i]] = KernelRecord(bwd_attn[i], f"attn_bwd_{i}", dur(2 * attn_flops), stage(i), i)
        slots[opt[i]] = KernelRecord(opt[i], f"opt_step_{i}",
                                     dur(cfg.optimizer_intensity * layer_params), stage(i), i)
    # the reference appends kernels in this order: forward pairs by layer,
    # backward pairs by descending layer, optimizer by layer
    order = ([x for i in range(L) for x in (fwd_attn[i], fwd_mlp[i])]
             + [x for i in reversed(range(L)) for x in (bwd_mlp[i], bwd_attn[i])]
             + opt)
    kernels = [slots[k] for k in order]

    bpe = cfg.bytes_per_element
    attn_w = ATTN_WEIGHT_ELEMS * h * h * bpe
    mlp_w = MLP_WEIGHT_ELEMS * h * h * bpe
    act = tokens * h * bpe
    G, I = TensorKind.GLOBAL, TensorKind.INTERMEDIATE
    tensors: list[TensorRecord] = []
    for i in range(L):
        specs = [
            (attn_w, G, (fwd_attn[i], bwd_attn[i], opt[i])),
            (mlp_w, G, (fwd_mlp[i], bwd_mlp[i], opt[i])),
            (attn_w, G, (bwd_attn[i], opt[i])),
            (mlp_w, G, (bwd_mlp[i], opt[i])),
            (OPT_STATE_FACTOR * attn_w, G, (opt[i],)),
            (OPT_STATE_FACTOR * mlp_w, G, (opt[i],)),
            (ATTN_ACT_ELEMS * act, I, (fwd_attn[i], bwd_attn[i])),
            (MLP_ACT_ELEMS * act, I, (fwd_mlp[i], bwd_mlp[i])),
        ]
        for size, kind, acc in specs:
            tensors.append(TensorRecord(len(tensors), size, kind, acc, i))

    meta = {"generator": "transformer", "num_layers": L, "hidden_dim": h,
            "num_heads": cfg.num_heads, "batch": cfg.batch, "seq_len": cfg.seq_len,
            "bytes_per_element": bpe, "pipeline_stages": cfg.pipeline_stages,
            "compute_rate": cfg.compute_rate, "seed": cfg.seed}
    return make_trace(kernels, tensors, meta)


def transformer_peak_bytes(cfg: TransformerGenConfig) -> int:
    """Closed-form peak of `gen_transformer_trace` (reference :152-162)."""
    bpe = cfg.bytes_per_element
    weights = cfg.num_layers * (ATTN_WEIGHT_ELEMS + MLP_WEIGHT_ELEMS) * cfg.hidden_dim ** 2 * bpe
    acts = (cfg.num_layers * (ATTN_ACT_ELEMS + MLP_ACT_ELEMS)
            * cfg.batch * cfg.seq_len * cfg.hidden_dim * bpe)
    return weights * (2 + OPT_STATE_FACTOR) + acts


def gen_random_trace(seed: int, num_kernels: int, num_tensors: int,
                     size_range: tuple[int, int] = (1_000_000, 200_000_000),
                     duration_range: tuple[int, int] = (100, 10_000),
                     global_fraction: float = 0.3) -> Trace:
    """Random valid trace; the RNG call sequence follows reference
    tracegen.py:165-186 so identical arguments give identical traces."""
    if size_range[0] <= 0 or duration_range[0] <= 0:
        raise ValueError("ranges must be positive")
    rng = random.Random(seed)
    kernels = [KernelRecord(i, f"k{i}", rng.randint(*duration_range))
               for i in range(num_kernels)]
    tensors = []
    for tid in range(num_tensors if num_kernels > 0 else 0):
        count = rng.randint(1, min(4, num_kernels))
        acc = tuple(sorted(rng.sample(range(num_kernels), count)))
        kind = TensorKind.GLOBAL if rng.random() < global_fraction else TensorKind.INTERMEDIATE
        tensors.append(TensorRecord(tid, rng.randint(*size_range), kind, acc))
    return make_trace(kernels, tensors, {"generator": "random", "seed": seed})


# --------------------------------------------------------------------------
# per-op Llama-shaped iteration

@dataclass(frozen=True)
class LlamaTraceConfig:
    num_layers: int = 32
    hidden: int = 4096
    ffn: int = 14336
    kv_dim: int = 1024
    tokens: int = 8192
    microbatches: int = 292
    attn_span: int = 2048          # S in the flash-attention FLOP model
    flops_per_us: int = 1_000_000_000


LLAMA3_8B = LlamaTraceConfig()                                   # C2
LLAMA3_70B = LlamaTraceConfig(num_layers=80, hidden=8192, ffn=28672, kv_dim=1024,
                              tokens=4096, microbatches=1160)     # C3

_WEIGHTS = ("attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w1", "w3", "w2")


class _MicrobatchTemplate:
    """Op list of one microbatch with tensor touches.

    Global tensors are referenced by their global index (0..G-1); new
    intermediates get template-local ids 0..M-1 in creation order.
    """

    def __init__(self, cfg: LlamaTraceConfig):
        self.cfg = cfg
        self.kernels: list[tuple[str, int, int | None]] = []   # (name, flops, layer)
        self.g_touch: list[tuple[int, int]] = []                # (global idx, kernel)
        self.i_touch: list[tuple[int, int]] = []                # (local id, kernel)
        self.i_size: list[int] = []
        self.i_layer: list[int | None] = []
        self._build()

    def _w(self, layer: int, name: str, which: int = 0) -> tuple[str, int]:
        # global index: layer-major, weight-major, then (weight, grad, m, v)
        return ("g", (layer * len(_WEIGHTS) + _WEIGHTS.index(name)) * 4 + which)

    def _op(self, name: str, flops: int, layer, touched, new_sizes=()):
        k = len(self.kernels)
        self.kernels.append((name, flops, layer))
        created = []
        for size in new_sizes:
            lid = len(self.i_size)
            self.i_size.append(size)
            self.i_layer.append(layer)
            created.append(("i", lid))
        for kind, idx in list(touched) + created:
            (self.g_touch if kind == "g" else self.i_touch).append((idx, k))
        return created[0] if len(created) == 1 else created

    def _build(self) -> None:
        c = self.cfg
        tok, h, ffn, kv, S = c.tokens, c.hidden, c.ffn, c.kv_dim, c.attn_span
        th = tok * h * 2
        tkv = tok * kv * 2
        tffn = tok * ffn * 2
        lse_b = tok * 32 * 4
        W = self._w
        x = self._op("embed", tok * h, None, [], [th])
        saved = []
        for l in range(c.num_layers):
            xin = x
            hh = self._op("rmsnorm", 4 * tok * h, l, [x, W(l, "attn_norm")], [th])
            q = self._op("q_proj", 2 * tok * h * h, l, [hh, W(l, "wq")], [th])
            k = self._op("k_proj", 2 * tok * h * kv, l, [hh, W(l, "wk")], [tkv])
            v = self._op("v_proj", 2 * tok * h * kv, l, [hh, W(l, "wv")], [tkv])
            self._op("rope", 8 * tok * h, l, [q, k])
            o, lse = self._op("flash_fwd", 4 * tok * S * h, l, [q, k, v], [th, lse_b])
            a = self._op("o_proj", 2 * tok * h * h, l, [o, W(l, "wo")], [th])
            x2 = self._op("residual", tok * h, l, [x, a], [th])
            h2 = self._op("rmsnorm", 4 * tok * h, l, [x2, W(l, "ffn_norm")], [th])
            g = self._op("w1", 2 * tok * h * ffn, l, [h2, W(l, "w1")], [tffn])
            u = self._op("w3", 2 * tok * h * ffn, l, [h2, W(l, "w3")], [tffn])
            m = self._op("silu_mul", 4 * tok * ffn, l, [g, u], [tffn])
            f = self._op("w2", 2 * tok * h * ffn, l, [m, W(l, "w2")], [th])
            x3 = self._op("residual", tok * h, l, [x2, f], [th])
            saved.append(dict(x=xin, h=hh, q=q, k=k, v=v, o=o, lse=lse, x2=x2, h2=h2,
                              g=g, u=u, m=m))
            x = x3
        dy = self._op("loss", 64 * tok * h, None, [x], [th])
        for l in reversed(range(c.num_layers)):
            s = saved[l]
            dm = self._op("w2_dgrad", 2 * tok * h * ffn, l, [dy, W(l, "w2")], [tffn])
            self._op("w2_wgrad", 2 * tok * h * ffn, l, [dy, s["m"], W(l, "w2", 1)])
            dg, du = self._op("silu_mul_bwd", 8 * tok * ffn, l, [dm, s["g"], s["u"]],
                              [tffn, tffn])
            dh2 = self._op("w1w3_dgrad", 4 * tok * h * ffn, l,
                           [dg, du, W(l, "w1"), W(l, "w3")], [th])
            self._op("w1w3_wgrad", 4 * tok * h * ffn, l,
                     [dg, du, s["h2"], W(l, "w1", 1), W(l, "w3", 1)])
            dx2 = self._op("rmsnorm_bwd", 8 * tok * h, l,
                           [dh2, s["x2"], W(l, "ffn_norm"), W(l, "ffn_norm", 1), dy], [th])
            do = self._op("o_dgrad", 2 * tok * h * h, l, [dx2, W(l, "wo")], [th])
            self._op("o_wgrad", 2 * tok * h * h, l, [dx2, s["o"], W(l, "wo", 1)])
            dq, dk, dv = self._op("flash_bwd", 10 * tok * S * h, l,
                                  [do, s["q"], s["k"], s["v"], s["o"], s["lse"]],
                                  [th, tkv, tkv])
            self._op("rope_bwd", 8 * tok * h, l, [dq, dk])
            dh = self._op("qkv_dgrad", 2 * tok * h * (h + 2 * kv), l,
                          [dq, dk, dv, W(l, "wq"), W(l, "wk"), W(l, "wv")], [th])
            self._op("qkv_wgrad", 2 * tok * h * (h + 2 * kv), l,
                     [dq, dk, dv, s["h"], W(l, "wq", 1), W(l, "wk", 1), W(l, "wv", 1)])
            dx = self._op("rmsnorm_bwd", 8 * tok * h, l,
                          [dh, s["x"], W(l, "attn_norm"), W(l, "attn_norm", 1), dx2], [th])
            dy = dx


def _weight_elems(cfg: LlamaTraceConfig, name: str) -> int:
    h, ffn, kv = cfg.hidden, cfg.ffn, cfg.kv_dim
    return {"attn_norm": h, "wq": h * h, "wk": h * kv, "wv": h * kv, "wo": h * h,
            "ffn_norm": h, "w1": h * ffn, "w3": h * ffn, "w2": ffn * h}[name]


def _dedupe_sorted(pairs: np.ndarray) -> np.ndarray:
    """pairs: (n,2) [tensor, kernel], sorted; drop exact repeats (the
    "unless its last access is already k" rule)."""
    if pairs.shape[0] < 2:
        return pairs
    keep = np.ones(pairs.shape[0], dtype=bool)
    keep[1:] = np.any(pairs[1:] != pairs[:-1], axis=1)
    return pairs[keep]


def gen_llama_trace(cfg: LlamaTraceConfig = LLAMA3_8B) -> Trace:
    """Appendix-C per-op trace, column form.

    Ids: globals first (layer, weight, then weight/grad/m/v), then the
    intermediates of each microbatch in creation order.  Kernel durations
    are max(1, flops // flops_per_us).  Kernel order: per microbatch
    [embed, forward layers, loss, backward layers], then one `adamw` kernel
    per (layer, weight).
    """
    tpl = _MicrobatchTemplate(cfg)
    L, nw = cfg.num_layers, len(_WEIGHTS)
    G = L * nw * 4
    K = len(tpl.kernels)
    M = len(tpl.i_size)
    MB = cfg.microbatches

    # kernels
    names = sorted({n for n, _, _ in tpl.kernels} | {"adamw"})
    code_of = {n: i for i, n in enumerate(names)}
    tpl_code = np.array([code_of[n] for n, _, _ in tpl.kernels], dtype=np.int32)
    tpl_dur = np.array([max(1, f // cfg.flops_per_us) for _, f, _ in tpl.kernels], dtype=np.int64)
    tpl_layer = np.array([NONE_I64 if l is None else l for _, _, l in tpl.kernels], dtype=np.int64)
    adam_sizes = []
    adam_layer = []
    for l in range(L):
        for w in _WEIGHTS:
            adam_sizes.append(_weight_elems(cfg, w) * 2)
            adam_layer.append(l)
    adam_dur = np.array([max(1, 12 * s // cfg.flops_per_us) for s in adam_sizes], dtype=np.int64)
    N = K * MB + G // 4
    duration = np.concatenate([np.tile(tpl_dur, MB), adam_dur])
    name_code = np.concatenate([np.tile(tpl_code, MB),
                                np.full(G // 4, code_of["adamw"], dtype=np.int32)])
    k_layer = np.concatenate([np.tile(tpl_layer, MB), np.array(adam_layer, dtype=np.int64)])

    # globals: per-microbatch touches + the adamw kernel of their weight
    gt = np.array(sorted(set(tpl.g_touch)), dtype=np.int64).reshape(-1, 2)   # (g, k) sorted by g, k
    gt = _dedupe_sorted(gt)
    mb_off = np.arange(MB, dtype=np.int64) * K
    # (MB, len(gt)) kernel indices; reorder so each global's accesses are contiguous & ascending
    g_idx = np.broadcast_to(gt[:, 0], (MB, gt.shape[0]))
    g_ker = gt[:, 1][None, :] + mb_off[:, None]
    adam_k = K * MB + np.arange(G) // 4
    all_g = np.concatenate([g_idx.reshape(-1), np.arange(G, dtype=np.int64)])
    all_k = np.concatenate([g_ker.reshape(-1), adam_k])
    order = np.lexsort((all_k, all_g))
    g_sorted_k = all_k[order]
    g_counts = np.bincount(all_g, minlength=G)

    # intermediates: per-template accesses, tiled
    it = _dedupe_sorted(np.array(sorted(set(tpl.i_touch)), dtype=np.int64).reshape(-1, 2))
    i_counts_tpl = np.bincount(it[:, 0], minlength=M)
    i_acc = (it[:, 1][None, :] + mb_off[:, None]).reshape(-1)
    i_counts = np.tile(i_counts_tpl, MB)

    T = G + M * MB
    counts = np.concatenate([g_counts, i_counts])
    ptr = np.zeros(T + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    accesses = np.concatenate([g_sorted_k, i_acc])

    g_size = np.empty(G, dtype=np.int64)
    g_layer = np.empty(G, dtype=np.int64)
    for l in range(L):
        for wi, w in enumerate(_WEIGHTS):
            e = _weight_elems(cfg, w)
            base = (l * nw + wi) * 4
            g_size[base:base + 4] = (2 * e, 2 * e, 4 * e, 4 * e)
            g_layer[base:base + 4] = l
    i_size = np.tile(np.array(tpl.i_size, dtype=np.int64), MB)
    i_layer = np.tile(np.array([NONE_I64 if l is None else l for l in tpl.i_layer],
                               dtype=np.int64), MB)
    kind = np.concatenate([np.full(G, KIND_GLOBAL, np.int8), np.full(M * MB, KIND_INTERMEDIATE, np.int8)])

    arrays = TraceArrays(
        duration_us=duration,
        kernel_index=np.arange(N, dtype=np.int64),
        kernel_name_code=name_code,
        name_table=names,
        kernel_stage=np.full(N, NONE_I64, dtype=np.int64),
        kernel_layer=k_layer,
        tensor_id=np.arange(T, dtype=np.int64),
        size_bytes=np.concatenate([g_size, i_size]),
        kind=kind,
        tensor_layer=np.concatenate([g_layer, i_layer]),
        access_ptr=ptr,
        accesses=accesses,
    )
    return Trace.from_arrays(arrays, {"generator": "probe-llama", "microbatches": MB})


def llama_peak_bytes(trace: Trace) -> int:
    """Peak of the no-offload memory timeline (host numpy; used to pick the
    peak//2 capacity of configs C2/C3)."""
    a = trace.arrays()
    n = a.num_kernels
    diff = np.zeros(n + 1, dtype=np.int64)
    first = a.accesses[a.access_ptr[:-1]]
    last = a.accesses[a.access_ptr[1:] - 1]
    glob = a.kind == KIND_GLOBAL
    np.add.at(diff, first[~glob], a.size_bytes[~glob])
    np.add.at(diff, last[~glob] + 1, -a.size_bytes[~glob])
    return int(np.cumsum(diff[:-1]).max() + a.size_bytes[glob].sum())
