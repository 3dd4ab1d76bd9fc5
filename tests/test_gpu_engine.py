"""Decode engine (one persistent kernel per step) == the per-layer kernel chain, bit for bit,
and == the oracle within the fp16 tolerance."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2505_11076_b200 as P  # noqa: E402
from paper_2505_11076_b200.plan import llama_decode_plan  # noqa: E402
import oracle  # noqa: E402
from conftest import rel_max, rel_norm  # noqa: E402


def _run(plan, x):
    import torch

    plan.buffers[plan.input_buffer].copy_(x)
    plan._eager()
    torch.cuda.synchronize()
    return plan.buffers[plan.output_buffer].clone()


@pytest.mark.parametrize("blocks,grid", [(1, 148), (2, 148), (1, 7), (3, 64)])
def test_engine_equals_layer_chain(blocks, grid):
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(11 + blocks)
    plan = llama_decode_plan("llama2-7b", bpw=2.0, blocks=blocks, generator=g)
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    ref = _run(plan.use_layer_kernels(), x)
    out = _run(plan.use_engine(grid=grid), x)
    assert torch.equal(out, ref)
    # replays reuse LL buffers through the epoch counter
    for _ in range(3):
        assert torch.equal(_run(plan, x), ref)


def test_engine_graph_replay_and_intermediate_parity():
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    plan = llama_decode_plan("llama2-7b", bpw=1.0, blocks=2, generator=g).use_engine()
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    plan.buffers[plan.input_buffer].copy_(x)
    plan.capture()
    outs = []
    for _ in range(3):
        plan.buffers[plan.input_buffer].copy_(x)
        plan.replay()
        torch.cuda.synchronize()
        outs.append(plan.buffers[plan.output_buffer].clone())
    ref = _run(plan.use_layer_kernels(), x)
    for o in outs:
        assert torch.equal(o, ref)


def test_engine_single_layer_vs_oracle():
    import torch
    from paper_2505_11076_b200.plan import DecodePlan, PlanOp

    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    n, k, m = 11008, 5952, 4096
    layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    bufs = [torch.randn((1, m), generator=g, device="cuda").half(), torch.zeros((1, n), device="cuda").half()]
    plan = DecodePlan([layer], [PlanOp(0, 0, 1, "gate")], bufs, input_buffer=0, output_buffer=1).use_engine()
    plan._eager()
    y = bufs[1].float().cpu().numpy()
    ref = oracle.c_forward(bufs[0].double().cpu().numpy(), layer.a.double().cpu().numpy(), layer.A.to_host().bits,
                           layer.mid.double().cpu().numpy(), layer.B.to_host().bits, layer.b.double().cpu().numpy())
    assert rel_max(y, ref) <= 1e-2 and rel_norm(y, ref) <= 1e-2
