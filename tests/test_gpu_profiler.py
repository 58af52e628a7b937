"""GPU: the TorchDispatchMode profiler turns a real training step (a small
Llama, random init, synthetic batch) into a valid trace that the planner,
the engine model and the executor accept."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def _tiny_llama_step():
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM
    torch.manual_seed(0)
    cfg = LlamaConfig(vocab_size=256, hidden_size=128, intermediate_size=352, num_hidden_layers=2,
                      num_attention_heads=4, num_key_value_heads=2, max_position_embeddings=256)
    model = LlamaForCausalLM(cfg).cuda().to(torch.bfloat16)
    opt = torch.optim.AdamW(model.parameters(), lr=1e-3, foreach=False)
    ids = torch.randint(0, 256, (2, 64), device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))

    def step():
        loss = model(input_ids=ids, labels=ids).loss
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=False)

    step()   # materialise grads and optimizer states before profiling

    def globals_():
        ts = list(model.parameters()) + [p.grad for p in model.parameters()]
        for st in opt.state.values():
            ts += [v for v in st.values() if torch.is_tensor(v)]
        return ts
    return step, globals_


def test_profiled_llama_step_is_a_valid_trace_and_plans():
    from paper_2506_06472_b200 import ChannelRates, plan_migrations, simulate, write_trace, parse_trace
    from paper_2506_06472_b200.profiler import profile_step
    step, globals_ = _tiny_llama_step()
    tr = profile_step(step, globals_, {"generator": "TraceProfiler", "model": "tiny-llama"})
    a = tr.arrays()
    assert a.num_kernels > 100 and a.num_tensors > 50
    assert (a.kind == 1).sum() >= 3 * 2 * 9          # params + grads + states of 2 layers
    assert write_trace(parse_trace(write_trace(tr))) == write_trace(tr)
    from paper_2506_06472_b200.tracegen import llama_peak_bytes
    peak = llama_peak_bytes(tr)
    rates = ChannelRates.symmetric(50_000)
    plan = plan_migrations(tr, int(peak * 0.7), rates)
    rep = simulate(tr, plan, int(peak * 0.7), rates)
    assert rep.total_time >= rep.ideal_time > 0
