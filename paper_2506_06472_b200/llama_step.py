"""The C4 / C5 workload (BASELINE.json configs[3-4]): one training
step of a randomly initialised Llama-3-8B on one B200 — the step the
migration engine offloads.

  * model: Llama-3 architecture (RMSNorm, RoPE theta 5e5, GQA attention with
    8 KV heads — FlashAttention-2 with its deterministic backward, so a rerun
    of the same steps is bit-identical; SDPA when flash_attn is absent —
    SwiGLU FFN, untied LM head);
    Llama-3-8B = 32 layers, hidden 4096, FFN 14336, vocab 128,256;
  * weights bf16, `torch.manual_seed(seed)` random init (no checkpoint: no
    network), gradients bf16, AdamW moments fp32 (allocated up front, as in
    the Appendix-C trace: one update per weight, fp32 math);
  * batch: synthetic tokens `torch.randint(0, vocab, (1, seq + 1))` from a
    seeded generator (inputs = [:-1], targets = [1:]), fp32 cross-entropy.

This is plumbing for the measurement (PyTorch + cuBLAS/SDPA library kernels),
not the product: the product is the engine that moves its tensors
(engine.OffloadMode over libtio's tio_engine_*).  `globals_of` names every
tensor that persists across steps (weights, AdamW moments, RoPE tables) so the
profiler and the engine give them the same tensor ids.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F
from torch import nn

try:                                     # FlashAttention-2 (library kernels: plumbing of the workload)
    from flash_attn import flash_attn_func as _flash_attn_func
except Exception:                        # pragma: no cover - absent in some images
    _flash_attn_func = None


@dataclass(frozen=True)
class LlamaConfig:
    vocab: int = 128_256
    dim: int = 4096
    layers: int = 32
    heads: int = 32
    kv_heads: int = 8
    ffn: int = 14_336
    rope_theta: float = 500_000.0
    eps: float = 1e-5
    seq: int = 8192
    deterministic: bool = True     # run-to-run identical kernels (deterministic attention backward)

    @property
    def head_dim(self) -> int:
        return self.dim // self.heads


LLAMA3_8B_MODEL = LlamaConfig()
# a small model of the same architecture for tests and smoke runs
TINY = LlamaConfig(vocab=4096, dim=512, layers=2, heads=8, kv_heads=2, ffn=1536, seq=512)


def _acc(t):
    """accumulation dtype: fp32 for bf16/fp16/fp32 tensors (fp64 stays fp64)"""
    return torch.promote_types(t.dtype, torch.float32)


class _RMSNormFn(torch.autograd.Function):
    """RMSNorm in fp32 that keeps only (x, weight, rstd) for backward — the
    memory profile of a fused norm kernel."""

    @staticmethod
    def forward(ctx, x, w, eps):
        xf = x.to(_acc(x))
        rstd = torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
        ctx.save_for_backward(x, w, rstd)
        return (xf * rstd).to(x.dtype) * w

    @staticmethod
    def backward(ctx, gy):
        x, w, rstd = ctx.saved_tensors
        xhat = x.to(_acc(x)) * rstd
        g = gy.to(_acc(gy))
        gw = (g * xhat).sum(dim=tuple(range(g.dim() - 1))).to(w.dtype)
        gxh = g * w.to(_acc(w))
        gx = rstd * (gxh - xhat * (gxh * xhat).mean(-1, keepdim=True))
        return gx.to(x.dtype), gw, None


class _SwiGLUFn(torch.autograd.Function):
    """silu(g) * u keeping only (g, u) for backward."""

    @staticmethod
    def forward(ctx, g, u):
        ctx.save_for_backward(g, u)
        return F.silu(g) * u

    @staticmethod
    def backward(ctx, gm):
        g, u = ctx.saved_tensors
        gf = g.to(_acc(g))
        sg = torch.sigmoid(gf)
        gmf = gm.to(_acc(gm))
        du = (gmf * gf * sg).to(u.dtype)
        dg = (gmf * u.to(_acc(u)) * sg * (1 + gf * (1 - sg))).to(g.dtype)
        return dg, du


class RMSNorm(nn.Module):
    def __init__(self, dim: int, eps: float):
        super().__init__()
        self.weight = nn.Parameter(torch.ones(dim))
        self.eps = eps

    def forward(self, x):
        return _RMSNormFn.apply(x, self.weight, self.eps)


def _rope(x, cos, sin):
    # x: (B, H, S, D); rotate pairs (even, odd) halves
    x1, x2 = x[..., 0::2], x[..., 1::2]
    c, s = cos.to(x.dtype), sin.to(x.dtype)
    return torch.stack((x1 * c - x2 * s, x1 * s + x2 * c), dim=-1).flatten(-2)


class Block(nn.Module):
    def __init__(self, c: LlamaConfig):
        super().__init__()
        self.c = c
        self.attn_norm = RMSNorm(c.dim, c.eps)
        self.wq = nn.Linear(c.dim, c.dim, bias=False)
        self.wk = nn.Linear(c.dim, c.kv_heads * c.head_dim, bias=False)
        self.wv = nn.Linear(c.dim, c.kv_heads * c.head_dim, bias=False)
        self.wo = nn.Linear(c.dim, c.dim, bias=False)
        self.ffn_norm = RMSNorm(c.dim, c.eps)
        self.w1 = nn.Linear(c.dim, c.ffn, bias=False)
        self.w3 = nn.Linear(c.dim, c.ffn, bias=False)
        self.w2 = nn.Linear(c.ffn, c.dim, bias=False)

    def forward(self, x, cos, sin):
        c = self.c
        B, S, _ = x.shape
        h = self.attn_norm(x)
        q = self.wq(h).view(B, S, c.heads, c.head_dim).transpose(1, 2)
        k = self.wk(h).view(B, S, c.kv_heads, c.head_dim).transpose(1, 2)
        v = self.wv(h).view(B, S, c.kv_heads, c.head_dim).transpose(1, 2)
        q, k = _rope(q, cos, sin), _rope(k, cos, sin)
        if c.deterministic and _flash_attn_func is not None and q.is_cuda:
            # FlashAttention-2 with its deterministic backward (no atomic dq
            # accumulation): the no-offload and offloaded steps are then
            # bit-comparable; layout (B, S, H, D), GQA native
            o = _flash_attn_func(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), causal=True,
                                 deterministic=True)
            x = x + self.wo(o.reshape(B, S, c.dim))
        else:
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
            x = x + self.wo(o.transpose(1, 2).reshape(B, S, c.dim))
        h2 = self.ffn_norm(x)
        return x + self.w2(_SwiGLUFn.apply(self.w1(h2), self.w3(h2)))


class Llama(nn.Module):
    def __init__(self, c: LlamaConfig):
        super().__init__()
        self.c = c
        self.embed = nn.Embedding(c.vocab, c.dim)
        self.blocks = nn.ModuleList([Block(c) for _ in range(c.layers)])
        self.norm = RMSNorm(c.dim, c.eps)
        self.head = nn.Linear(c.dim, c.vocab, bias=False)
        inv = 1.0 / (c.rope_theta ** (torch.arange(0, c.head_dim, 2, dtype=torch.float32) / c.head_dim))
        ang = torch.outer(torch.arange(c.seq, dtype=torch.float32), inv)
        self.register_buffer("cos", ang.cos(), persistent=False)
        self.register_buffer("sin", ang.sin(), persistent=False)

    def forward(self, tokens, targets):
        x = self.embed(tokens)
        for b in self.blocks:
            x = b(x, self.cos, self.sin)
        logits = self.head(self.norm(x))
        return F.cross_entropy(logits.float().view(-1, self.c.vocab), targets.view(-1))


class AdamW:
    """AdamW with fp32 moments for bf16 weights: one fp32 update per weight
    (moments allocated up front so they persist like the Appendix-C trace's
    globals)."""

    def __init__(self, params, lr=1e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1):
        self.params = list(params)
        self.lr, self.b1, self.b2, self.eps, self.wd = lr, betas[0], betas[1], eps, weight_decay
        self.m = [torch.zeros_like(p, dtype=torch.float32) for p in self.params]
        self.v = [torch.zeros_like(p, dtype=torch.float32) for p in self.params]
        self.t = 0

    @torch.no_grad()
    def step(self):
        self.t += 1
        bc1 = 1 - self.b1 ** self.t
        bc2s = math.sqrt(1 - self.b2 ** self.t)
        for p, m, v in zip(self.params, self.m, self.v):
            g = p.grad.float()
            m.mul_(self.b1).add_(g, alpha=1 - self.b1)
            v.mul_(self.b2).addcmul_(g, g, value=1 - self.b2)
            upd = m / v.sqrt().div_(bc2s).add_(self.eps)
            p32 = p.float().mul_(1 - self.lr * self.wd).add_(upd, alpha=-self.lr / bc1)
            p.copy_(p32)
            p.grad = None


class Step:
    """Model + optimizer + batch; `__call__()` runs one training step on the
    current stream and returns the loss tensor (on the device)."""

    def __init__(self, c: LlamaConfig = LLAMA3_8B_MODEL, seed: int = 0, device="cuda", dp_group=None):
        self.c = c
        # data parallel (configs C5): the gradients are all-reduced (mean) over
        # the group between backward and the optimizer step; every rank runs
        # the same seed, hence the same model, batch, trace and plan
        self.dp_group = dp_group
        torch.manual_seed(seed)
        old = torch.get_default_dtype()
        torch.set_default_dtype(torch.bfloat16)
        try:
            with torch.device(device):
                self.model = Llama(c)
        finally:
            torch.set_default_dtype(old)
        self.opt = AdamW(self.model.parameters())
        g = torch.Generator().manual_seed(seed)
        seq = torch.randint(0, c.vocab, (1, c.seq + 1), generator=g)
        self.host_batch = seq.pin_memory() if torch.cuda.is_available() else seq
        self.batch = self.host_batch.to(device)

    def globals_of(self) -> dict:
        """Every tensor that persists across steps, by a stable name."""
        out = {}
        for n, p in self.model.named_parameters():
            out["param:" + n] = p
        for i, (m, v) in enumerate(zip(self.opt.m, self.opt.v)):
            out[f"adam_m:{i}"] = m
            out[f"adam_v:{i}"] = v
        out["rope:cos"] = self.model.cos
        out["rope:sin"] = self.model.sin
        return out

    def __call__(self, batch=None):
        b = self.batch if batch is None else batch
        loss = self.model(b[:, :-1], b[:, 1:])
        loss.backward()
        if self.dp_group is not None:
            import torch.distributed as dist
            world = dist.get_world_size(self.dp_group)
            for p in self.model.parameters():
                dist.all_reduce(p.grad, group=self.dp_group)
                p.grad.div_(world)
        self.opt.step()
        return loss.detach()

    def state_bytes(self) -> dict:
        return {n: t.detach().view(torch.uint8) if t.dtype != torch.uint8 else t for n, t in self.globals_of().items()}
