"""Token batches of 5-16 (north_star subsystem 2 / BASELINE configs[3]-[4]): every token through the
decode engine (groups of <= 4 tokens per launch), the single-pass batched kernels and the tcgen05
prefill chain, against the float64 oracle on the same bytes (tolerance: max|err|/max|ref| and
||err||/||ref|| <= 1e-2)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2505_11076_b200 as P  # noqa: E402
import oracle  # noqa: E402
from conftest import rel_max, rel_norm  # noqa: E402

TOL = 1e-2


@pytest.mark.parametrize("batch", [5, 8, 16])
@pytest.mark.parametrize("path", ["engine", "prefill", "batched"])
def test_batched_layer_vs_oracle(batch, path):
    import torch
    from paper_2505_11076_b200.plan import DecodePlan, PlanOp

    g = torch.Generator(device="cuda")
    g.manual_seed(batch * 3 + (path == "prefill"))
    n, k, m = 4096, 5952, 11008  # the 7B down shape
    layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    x = torch.randn((batch, m), generator=g, device="cuda").half()
    bufs = [x.clone(), torch.zeros((batch, n), dtype=torch.half, device="cuda")]
    plan = DecodePlan([layer], [PlanOp(0, 0, 1, "down")], bufs, input_buffer=0, output_buffer=1)
    {"engine": plan.use_engine, "prefill": plan.use_prefill, "batched": plan.use_batched}[path]()
    plan._eager()
    torch.cuda.synchronize()
    y = bufs[1].double().cpu().numpy()
    ref = oracle.c_forward(x.double().cpu().numpy(), layer.a.double().cpu().numpy(), layer.A.to_host().bits,
                           layer.mid.double().cpu().numpy(), layer.B.to_host().bits, layer.b.double().cpu().numpy())
    for t in range(batch):
        assert rel_max(y[t], ref[t]) <= TOL and rel_norm(y[t], ref[t]) <= TOL, (t, rel_max(y[t], ref[t]))
    if path == "engine":
        assert plan.engine.kernel_launches_per_step() == -(-batch // 4)


def test_layerwise_k_plan_runs_and_matches_layer_kernels():
    """BASELINE configs[4]: a non-uniform layer-wise k (reference greedy allocation) -- the engine
    chain equals the per-layer kernel chain within tolerance, at batch 1 and 8."""
    import torch
    from paper_2505_11076_b200.plan import layerwise_ks, llama_decode_plan

    ks = layerwise_ks("llama2-13b", target_bpw=1.5, floor_bpw=1.0, cap_bpw=2.3, blocks=2)
    assert len(set(ks)) > 3
    for batch in (1, 8):
        g = torch.Generator(device="cuda")
        g.manual_seed(70 + batch)
        plan = llama_decode_plan("llama2-13b", batch=batch, blocks=2, generator=g, ks=ks)
        x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
        outs = []
        for use in (plan.use_layer_kernels, plan.use_engine):
            use()
            plan.buffers[plan.input_buffer].copy_(x)
            plan._eager()
            torch.cuda.synchronize()
            outs.append(plan.buffers[plan.output_buffer].double().cpu().numpy())
        assert rel_max(outs[1], outs[0]) <= TOL and rel_norm(outs[1], outs[0]) <= TOL
