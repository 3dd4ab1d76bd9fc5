"""The single-pass batched decode (dbf_forward_batched, csrc/batched.cu; north_star subsystem 2,
BASELINE configs[3]-[4] at 2-16 tokens) against the float64 oracle on the same bytes.

Tolerance as for the decode engine whose numerics it shares (13-bit grid per token and 256-column
chunk): max|err|/max|ref| and ||err||/||ref|| <= 1e-2 per token row.  Also: deterministic bits,
ragged shapes, non-finite inputs confined to their own token (NaN + status bit), the fp16-overflow
status, and a decoder chain through DecodePlan.use_batched against the per-layer kernels."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2505_11076_b200 as P  # noqa: E402
import oracle  # noqa: E402
from conftest import rel_max, rel_norm  # noqa: E402

TOL = 1e-2


def _ref(x, layer):
    return oracle.c_forward(x.double().cpu().numpy(), layer.a.double().cpu().numpy(), layer.A.to_host().bits,
                            layer.mid.double().cpu().numpy(), layer.B.to_host().bits, layer.b.double().cpu().numpy())


@pytest.mark.parametrize("batch", [1, 2, 4, 5, 8, 13, 16, 17, 24, 32])
def test_batched_matches_oracle(batch):
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(100 + batch)
    n, k, m = 4096, 5952, 11008  # the 7B down shape
    layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    x = torch.randn((batch, m), generator=g, device="cuda").half()
    y = P.forward_batched(x, layer).double().cpu().numpy()
    ref = _ref(x, layer)
    for t in range(batch):
        assert rel_max(y[t], ref[t]) <= TOL and rel_norm(y[t], ref[t]) <= TOL, (t, rel_max(y[t], ref[t]))


@pytest.mark.parametrize("shape", [(200, 96, 136), (1000, 1100, 1024), (1024, 1792, 8192), (33, 17, 300)])
def test_batched_ragged_shapes(shape):
    import torch

    n, k, m = shape
    g = torch.Generator(device="cuda")
    g.manual_seed(n + k + m)
    layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    for batch in (3, 11, 27):
        x = torch.randn((batch, m), generator=g, device="cuda").half()
        y = P.forward_batched(x, layer).double().cpu().numpy()
        ref = _ref(x, layer)
        for t in range(batch):
            assert rel_max(y[t], ref[t]) <= TOL and rel_norm(y[t], ref[t]) <= TOL, (shape, batch, t)


def test_batched_deterministic_and_strided_io():
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    layer = P.random_device_layer(4096, 2048, 4096, generator=g, keep_words=True)
    big = torch.randn((10, 4096 + 64), generator=g, device="cuda").half()
    x = big[:, 32:32 + 4096]  # row stride 4160
    out = torch.zeros((10, 4096 + 8), dtype=torch.half, device="cuda")
    y1 = P.forward_batched(x, layer, out=out[:, :4096]).clone()
    y2 = P.forward_batched(x.contiguous(), layer)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.count_nonzero(out[:, 4096:]) == 0
    ref = _ref(x, layer)
    assert rel_max(y2.double().cpu().numpy(), ref) <= TOL


def test_batched_nonfinite_confined_and_status():
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(8)
    layer = P.random_device_layer(1024, 1024, 2048, generator=g, keep_words=True)
    x = torch.randn((6, 2048), generator=g, device="cuda").half()
    x[2, 700] = float("inf")
    x[4, 5] = float("nan")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    y = P.forward_batched(x, layer, status=status).double().cpu().numpy()
    assert np.isnan(y[2]).all() and np.isnan(y[4]).all()
    ref = _ref(x[[0, 1, 3, 5]], layer)
    assert rel_max(y[[0, 1, 3, 5]], ref) <= TOL
    assert int(status.item()) & 1


def test_batched_fp16_overflow_status():
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    layer = P.random_device_layer(512, 512, 1024, generator=g)
    layer.a.fill_(60000.0)  # |y| far beyond 65504 for random inputs
    x = torch.randn((5, 1024), generator=g, device="cuda").half()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    y = P.forward_batched(x, layer, status=status)
    torch.cuda.synchronize()
    assert torch.isinf(y).any()
    assert int(status.item()) & 2


def test_batched_rejects_bad_input():
    import torch

    layer = P.random_device_layer(64, 32, 64)
    with pytest.raises(ValueError):
        P.forward_batched(torch.zeros((33, 64), dtype=torch.half, device="cuda"), layer)
    with pytest.raises(ValueError):
        P.forward_batched(torch.zeros((4, 63), dtype=torch.half, device="cuda"), layer)
    with pytest.raises(ValueError):
        P.forward_batched(torch.zeros((64,), dtype=torch.half, device="cuda"), layer)


@pytest.mark.parametrize("batch", [5, 8, 16])
def test_batched_plan_chain_matches_layer_kernels(batch):
    """Two 7B decoder blocks (14 layers in dataflow order) through DecodePlan.use_batched vs the
    exact per-layer kernels (dbf_forward), and the plan's default path at this batch."""
    import torch
    from paper_2505_11076_b200.plan import llama_decode_plan

    g = torch.Generator(device="cuda")
    g.manual_seed(40 + batch)
    plan = llama_decode_plan("llama2-7b", bpw=2.0, batch=batch, blocks=2, generator=g)
    assert plan.default_path() == "batched"
    # four kernels per layer, plus a quantize for each of the first block's q/k/v (their input
    # comes from outside the chain)
    assert plan.use_batched().kernel_launches_per_step() == 4 * 14 + 3
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    outs = []
    for use in (plan.use_layer_kernels, plan.use_batched):
        use()
        plan.buffers[plan.input_buffer].copy_(x)
        plan._eager()
        torch.cuda.synchronize()
        outs.append(plan.buffers[plan.output_buffer].double().cpu().numpy())
    assert rel_max(outs[1], outs[0]) <= TOL and rel_norm(outs[1], outs[0]) <= TOL
    # graph replay of the batched chain reproduces the eager bits; run() checks the status word
    # (capture() runs the chain once as its warm-up, and the plan's input buffer is also its output)
    plan.capture()
    y = plan.run(x.cpu())
    assert np.array_equal(y.double().numpy(), outs[1])


def test_batched_plan_raises_on_overflow():
    import torch
    from paper_2505_11076_b200.plan import DecodePlan, PlanOp

    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    layer = P.random_device_layer(512, 512, 1024, generator=g)
    layer.a.fill_(60000.0)
    bufs = [torch.randn((6, 1024), generator=g, device="cuda").half(), torch.zeros((6, 512), dtype=torch.half,
                                                                                   device="cuda")]
    plan = DecodePlan([layer], [PlanOp(0, 0, 1, "x")], bufs, input_buffer=0, output_buffer=1).use_batched()
    with pytest.raises(P.DbfOverflowError):
        plan.run(bufs[0].cpu())


@pytest.mark.parametrize("xdt,sdt", [("float32", "float32"), ("bfloat16", "float16"), ("float16", "float32")])
def test_batched_dtypes(xdt, sdt):
    """Activations fp16 / bf16 / fp32 and scales fp16 / fp32: the output is in X's dtype and within
    the tolerance of the oracle on the same (rounded) values."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(21)
    layer = P.random_device_layer(1000, 1100, 1024, generator=g, keep_words=True, scale_dtype=getattr(torch, sdt))
    x = torch.randn((7, 1024), generator=g, device="cuda").to(getattr(torch, xdt))
    y = P.forward_batched(x, layer)
    assert y.dtype == x.dtype
    y = y.double().cpu().numpy()
    ref = _ref(x, layer)
    for t in range(7):
        assert rel_max(y[t], ref[t]) <= TOL and rel_norm(y[t], ref[t]) <= TOL, (xdt, sdt, t)


def test_batched_matches_engine_numerics_closely():
    """Same 13-bit chunk grid as the decode engine: at 4 tokens the two paths agree far inside the
    oracle tolerance (the engine rounds t to fp16, the batched path keeps it fp32)."""
    import torch
    from paper_2505_11076_b200.plan import DecodePlan, PlanOp

    g = torch.Generator(device="cuda")
    g.manual_seed(22)
    layer = P.random_device_layer(4096, 2048, 4096, generator=g)
    x = torch.randn((4, 4096), generator=g, device="cuda").half()
    bufs = [x.clone(), torch.zeros((4, 4096), dtype=torch.half, device="cuda")]
    plan = DecodePlan([layer], [PlanOp(0, 0, 1, "q")], bufs, input_buffer=0, output_buffer=1).use_engine()
    plan._eager()
    ye = bufs[1].double().cpu().numpy()
    yb = P.forward_batched(x, layer).double().cpu().numpy()
    assert rel_max(yb, ye) <= 2e-3


def test_batched_chain_bitwise_equals_per_layer_calls():
    """DecodePlan.use_batched chains the layers: each finalize writes the next readers' input
    fragments from its stored output.  That must be bitwise what per-layer forward_batched calls
    (quantizing each stored input on its own) give -- including the 70B dataflow where o reads q
    and h feeds three readers."""
    import torch
    from paper_2505_11076_b200.plan import llama_decode_plan

    for model, batch in (("llama2-7b", 6), ("llama2-70b", 9)):
        g = torch.Generator(device="cuda")
        g.manual_seed(90 + batch)
        plan = llama_decode_plan(model, bpw=2.0, batch=batch, blocks=1, generator=g)
        x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
        plan.use_batched()
        plan.buffers[plan.input_buffer].copy_(x)
        plan._eager()
        torch.cuda.synchronize()
        chained = [b.clone() for b in plan.buffers]
        plan.buffers[plan.input_buffer].copy_(x)
        for op in plan.ops:
            P.forward_batched(plan.buffers[op.src], plan.layers[op.layer], out=plan.buffers[op.dst])
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(zip(chained, plan.buffers)):
            assert torch.equal(a, b), (model, i)


def test_batched_plan_groups_above_32_tokens():
    """40 tokens: two groups (32 + 8) of the batched chain over slices of the same buffers, within
    the tolerance of the exact per-layer kernels; default path batched up to 64 tokens."""
    import torch
    from paper_2505_11076_b200.plan import llama_decode_plan

    g = torch.Generator(device="cuda")
    g.manual_seed(140)
    plan = llama_decode_plan("llama2-7b", bpw=2.0, batch=40, blocks=1, generator=g)
    assert plan.default_path() == "batched"
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    outs = []
    for use in (plan.use_layer_kernels, plan.use_batched):
        use()
        plan.buffers[plan.input_buffer].copy_(x)
        plan._eager()
        torch.cuda.synchronize()
        outs.append(plan.buffers[plan.output_buffer].double().cpu().numpy())
    assert len(plan._bgroups) == 2
    assert rel_max(outs[1], outs[0]) <= TOL and rel_norm(outs[1], outs[0]) <= TOL


def test_batched_plan_fan_out_and_in_place():
    """Dataflow corner cases of the chained batched plan, bitwise against per-layer calls: one
    output read by five later layers (four get their fragments from the writer's finalize, the fifth
    quantizes on its own), and a layer writing its own input buffer."""
    import torch
    from paper_2505_11076_b200.plan import DecodePlan, PlanOp

    g = torch.Generator(device="cuda")
    g.manual_seed(150)
    w = 1024
    layers = [P.random_device_layer(w, 512, w, generator=g) for _ in range(7)]
    bufs = [torch.randn((6, w), generator=g, device="cuda").half()] + [
        torch.zeros((6, w), dtype=torch.half, device="cuda") for _ in range(7)]
    ops = [PlanOp(0, 0, 1, "src")] + [PlanOp(1 + i, 1, 2 + i, f"r{i}") for i in range(5)] + [PlanOp(6, 7, 7, "inplace")]
    plan = DecodePlan(layers, ops, bufs, input_buffer=0, output_buffer=7).use_batched()
    frags, readers, standalone, deps = plan._bchain
    assert len(readers[0]) == 4 and 5 in standalone and 6 in standalone
    x = bufs[0].clone()
    x7 = torch.randn((6, w), generator=g, device="cuda").half()
    bufs[7].copy_(x7)
    plan._eager()
    torch.cuda.synchronize()
    chained = [b.clone() for b in bufs]
    bufs[0].copy_(x)
    for b in bufs[1:7]:
        b.zero_()
    bufs[7].copy_(x7)
    for op in ops:
        P.forward_batched(bufs[op.src], layers[op.layer], out=bufs[op.dst])
    torch.cuda.synchronize()
    for i in range(8):
        assert torch.equal(chained[i], bufs[i]), i
    assert not torch.equal(chained[7], x7)
