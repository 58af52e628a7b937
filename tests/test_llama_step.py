"""The C4 workload's model code (paper_2506_06472_b200/llama_step.py) on the
CPU: the lean RMSNorm / SwiGLU autograd functions are exact (gradcheck in
float64) and the tiny model trains one step.  Host-only."""

from __future__ import annotations

import torch

from paper_2506_06472_b200.llama_step import TINY, Llama, _RMSNormFn, _SwiGLUFn


def test_lean_norm_and_swiglu_gradients():
    torch.manual_seed(0)
    x = torch.randn(3, 5, 16, dtype=torch.float64, requires_grad=True)
    w = torch.randn(16, dtype=torch.float64, requires_grad=True)
    assert torch.autograd.gradcheck(lambda a, b: _RMSNormFn.apply(a, b, 1e-5), (x, w))
    g = torch.randn(4, 7, dtype=torch.float64, requires_grad=True)
    u = torch.randn(4, 7, dtype=torch.float64, requires_grad=True)
    assert torch.autograd.gradcheck(lambda a, b: _SwiGLUFn.apply(a, b), (g, u))


def test_tiny_model_forward_backward():
    torch.manual_seed(0)
    m = Llama(TINY)
    tok = torch.randint(0, TINY.vocab, (1, TINY.seq + 1))
    loss = m(tok[:, :-1], tok[:, 1:])
    loss.backward()
    assert 7.0 < loss.item() < 10.0                 # ~ln(4096) at random init
    assert all(p.grad is not None for p in m.parameters())
