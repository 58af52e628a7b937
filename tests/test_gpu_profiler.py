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


def test_collective_tensors_are_active_in_the_trace():
    """tensors used by inter-GPU communication must be
    active while the collective runs.  A data-parallel step (NCCL process
    group of one rank) all-reduces its gradients: the profiler records the
    collective as a trace kernel touching the gradient, so the planner never
    offloads a gradient across its all-reduce."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2506_06472_b200.profiler import profile_step
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        torch.manual_seed(0)
        w = torch.randn(256, 256, device="cuda", requires_grad=True)
        x = torch.randn(64, 256, device="cuda")

        def step():
            loss = (x @ w).square().mean()
            loss.backward()
            dist.all_reduce(w.grad)                    # the DP gradient exchange
            with torch.no_grad():
                w.sub_(1e-3 * w.grad)
            w.grad = None

        step()
        tr = profile_step(step, globals_={"w": w})
        a = tr.arrays()
        names = [a.name_table[c] for c in a.kernel_name_code.tolist()]
        ks = [k for k, n in enumerate(names) if "allreduce" in n]
        assert ks, names
        k = ks[0]
        # the collective touches exactly the gradient: an intermediate of the
        # step produced by the backward and consumed by the update
        touched = [t for t in range(a.num_tensors) if k in a.accesses[a.access_ptr[t]:a.access_ptr[t + 1]]]
        assert len(touched) == 1
        t = touched[0]
        assert a.size_bytes[t] == 256 * 256 * 4 and a.kind[t] == 0
        acc = a.accesses[a.access_ptr[t]:a.access_ptr[t + 1]].tolist()
        assert acc[0] < k < acc[-1]                    # produced before, consumed after the collective
    finally:
        dist.destroy_process_group()
