"""Decode engine (one persistent kernel per step): parity with the per-layer kernel chain and the
oracle within the fp16 tolerance, and bitwise determinism -- across replays, graph capture and
grid sizes (every unit's sum is exact per chunk and combined in a fixed order, independent of
how units are spread over CTAs)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2505_11076_b200 as P  # noqa: E402
from paper_2505_11076_b200.plan import llama_decode_plan  # noqa: E402
import oracle  # noqa: E402
from conftest import rel_max, rel_norm  # noqa: E402

TOL = 1e-2  # fp16 activations: max|err|/max|ref| and ||err||/||ref||


def _run(plan, x):
    import torch

    plan.buffers[plan.input_buffer].copy_(x)
    plan._eager()
    torch.cuda.synchronize()
    return plan.buffers[plan.output_buffer].clone()


def _close(out, ref):
    o, r = out.double().cpu().numpy(), ref.double().cpu().numpy()
    return rel_max(o, r) <= TOL and rel_norm(o, r) <= TOL, (rel_max(o, r), rel_norm(o, r))


@pytest.mark.parametrize("blocks", [1, 3])
def test_engine_matches_layer_chain_and_is_grid_independent(blocks):
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(11 + blocks)
    plan = llama_decode_plan("llama2-7b", bpw=2.0, blocks=blocks, generator=g)
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    ref = _run(plan.use_layer_kernels(), x)
    out = _run(plan.use_engine(grid=148), x)
    ok, err = _close(out, ref)
    assert ok, err
    for grid in (7, 64):
        assert torch.equal(_run(plan.use_engine(grid=grid), x), out)
    # replays reuse the LL buffers through the epoch counter
    plan.use_engine(grid=148)
    for _ in range(3):
        assert torch.equal(_run(plan, x), out)


def test_engine_graph_replay_is_deterministic():
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    plan = llama_decode_plan("llama2-7b", bpw=1.0, blocks=2, generator=g).use_engine()
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    eager = _run(plan, x)
    plan.capture()
    for _ in range(3):
        plan.buffers[plan.input_buffer].copy_(x)
        plan.replay()
        torch.cuda.synchronize()
        assert torch.equal(plan.buffers[plan.output_buffer], eager)
    ok, err = _close(eager, _run(plan.use_layer_kernels(), x))
    assert ok, err


@pytest.mark.parametrize("n,k,m", [(11008, 5952, 4096), (4096, 5952, 11008), (1000, 300, 777)])
def test_engine_single_layer_vs_oracle(n, k, m):
    import torch
    from paper_2505_11076_b200.plan import DecodePlan, PlanOp

    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    bufs = [torch.randn((1, m), generator=g, device="cuda").half(), torch.zeros((1, n), device="cuda").half()]
    plan = DecodePlan([layer], [PlanOp(0, 0, 1, "gate")], bufs, input_buffer=0, output_buffer=1).use_engine()
    plan._eager()
    y = bufs[1].float().cpu().numpy()
    ref = oracle.c_forward(bufs[0].double().cpu().numpy(), layer.a.double().cpu().numpy(), layer.A.to_host().bits,
                           layer.mid.double().cpu().numpy(), layer.B.to_host().bits, layer.b.double().cpu().numpy())
    assert rel_max(y, ref) <= TOL and rel_norm(y, ref) <= TOL, (rel_max(y, ref), rel_norm(y, ref))


@pytest.mark.parametrize("batch", [2, 3, 4])
def test_batched_engine_matches_layer_chain(batch):
    """1..4 tokens per step share every tensor-core MMA (B columns = 2*token + digit plane); each
    token matches the per-layer chain and is independent of the others and of the grid."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(40 + batch)
    plan = llama_decode_plan("llama2-7b", bpw=2.0, batch=batch, blocks=1, generator=g)
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    ref = _run(plan.use_layer_kernels(), x)
    out = _run(plan.use_engine(grid=148), x)
    for t in range(batch):
        ok, err = _close(out[t:t + 1], ref[t:t + 1])
        assert ok, (t, err)
    assert torch.equal(_run(plan.use_engine(grid=37), x), out)
    # token 0 alone through a batch-1 engine: the same numbers (tokens do not interact)
    g1 = torch.Generator(device="cuda")
    g1.manual_seed(40 + batch)
    plan1 = llama_decode_plan("llama2-7b", bpw=2.0, batch=1, blocks=1, generator=g1).use_engine(grid=148)
    assert torch.equal(_run(plan1, x[:1]), out[:1])


def test_engine_batch_8_runs_in_groups_of_4():
    """8 tokens = two engine launches over token rows 0-3 and 4-7: each group equals a batch-4
    engine over the same rows, and the whole matches the per-layer chain within tolerance."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    plan = llama_decode_plan("llama2-7b", bpw=2.0, batch=8, blocks=1, generator=g)
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    ref = _run(plan.use_layer_kernels(), x)
    out = _run(plan.use_engine(), x)
    assert plan.engine.kernel_launches_per_step() == 2  # one kernel per group of <= 4 tokens
    for t in range(8):
        ok, err = _close(out[t:t + 1], ref[t:t + 1])
        assert ok, (t, err)
    g4 = torch.Generator(device="cuda")
    g4.manual_seed(77)
    plan4 = llama_decode_plan("llama2-7b", bpw=2.0, batch=4, blocks=1, generator=g4).use_engine()
    assert torch.equal(_run(plan4, x[4:]), out[4:])


@pytest.mark.parametrize("batch,n,k,m,act", [(3, 1000, 300, 777, "f32"), (4, 200, 64, 4100, "f16"),
                                              (1, 17, 32, 28500, "f32"), (2, 5000, 2000, 300, "f16"),
                                              (2, 17, 32, 29000, "f32"), (1, 2048, 8192, 28672, "f16")])
def test_engine_ragged_layers_vs_oracle(batch, n, k, m, act):
    """Ragged shapes (rows not a multiple of 16, columns not of 256, inputs wider than 64 chunks, up to
    the batch-1 limit of 112 chunks, with several units per run), fp32 or fp16 activations, 1-4
    tokens; fp32 plain output is the unrounded sum.  Against the
    float64 oracle on the same bytes, and launched again through the per-launch I/O overrides on
    other buffers: bitwise the same."""
    import torch
    from paper_2505_11076_b200.plan import DecodePlan, PlanOp

    dt = torch.float32 if act == "f32" else torch.float16
    g = torch.Generator(device="cuda")
    g.manual_seed(batch * 7 + n)
    layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    x = torch.randn((batch, m), generator=g, device="cuda").to(dt)
    bufs = [x.clone(), torch.zeros((batch, n), dtype=dt, device="cuda")]
    plan = DecodePlan([layer], [PlanOp(0, 0, 1, "l")], bufs, input_buffer=0, output_buffer=1).use_engine()
    plan._eager()
    torch.cuda.synchronize()
    y = bufs[1].double().cpu().numpy()
    ref = oracle.c_forward(x.double().cpu().numpy(), layer.a.double().cpu().numpy(), layer.A.to_host().bits,
                           layer.mid.double().cpu().numpy(), layer.B.to_host().bits, layer.b.double().cpu().numpy())
    assert rel_max(y, ref) <= TOL and rel_norm(y, ref) <= TOL, (rel_max(y, ref), rel_norm(y, ref))
    y2 = torch.empty_like(bufs[1])
    plan.engine.launch_io(x.clone(), y2)
    torch.cuda.synchronize()
    assert torch.equal(y2, bufs[1])


def test_use_fastest_keeps_the_faster_path_and_its_numbers():
    """DecodePlan.use_fastest times the engine (two launches of 4 tokens), the single-pass batched
    kernels and the tcgen05 prefill chain on the plan's buffers and keeps the fastest; the kept
    path gives exactly its own numbers, the paths agree within the fp16 tolerance, and the input
    buffer is restored."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(61)
    plan = llama_decode_plan("llama2-7b", bpw=2.0, batch=8, blocks=1, generator=g, keep_words=True)
    x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
    ref_e = _run(plan.use_engine(), x)
    ref_p = _run(plan.use_prefill(), x)
    ref_b = _run(plan.use_batched(), x)
    for other in (ref_p, ref_b):
        ok, err = _close(ref_e, other)
        assert ok, err
    plan.buffers[plan.input_buffer].copy_(x)
    plan.use_fastest(steps=2)
    assert set(plan.choice_ms) == {"engine", "batched", "prefill"} and plan.choice in plan.choice_ms
    assert torch.equal(plan.buffers[plan.input_buffer], x)
    assert torch.equal(_run(plan, x), {"engine": ref_e, "prefill": ref_p, "batched": ref_b}[plan.choice])
    # the static rule wins unless another path is faster by the margin: a huge margin always
    # keeps it, whatever the timings
    plan.use_fastest(steps=2, margin=1.0)
    assert plan.choice == plan.default_path() == "batched"


@pytest.mark.parametrize("batch,xdt,ydt", [(1, "float16", "float16"), (2, "float16", "float32"),
                                           (4, "float32", "float16"), (3, "float16", "float16")])
def test_forward_engine_vs_oracle(batch, xdt, ydt):
    """forward_engine: the drop-in per-call forward as ONE engine launch (BASELINE configs[0]:
    4096 x 4096, k = 2048), 1-4 token rows, fp16/fp32 in and out; against the float64 oracle on the
    same bytes; repeated calls (the cached program, new buffers through the I/O overrides) are
    bitwise equal; bad shapes / batches are rejected."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(40 + batch)
    n, k, m = 4096, 2048, 4096
    layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)  # words kept for the oracle's bytes
    X = torch.randn((batch, m), generator=g, device="cuda").to(getattr(torch, xdt))
    Y = P.forward_engine(X, layer, out_dtype=getattr(torch, ydt))
    assert Y.dtype == getattr(torch, ydt) and Y.shape == (batch, n)
    ref = oracle.c_forward(X.double().cpu().numpy(), layer.a.double().cpu().numpy(), layer.A.to_host().bits,
                           layer.mid.double().cpu().numpy(), layer.B.to_host().bits, layer.b.double().cpu().numpy())
    y = Y.float().cpu().numpy()
    assert rel_max(y, ref) <= TOL and rel_norm(y, ref) <= TOL, (rel_max(y, ref), rel_norm(y, ref))
    Y2 = torch.empty_like(Y)
    P.forward_engine(X.clone(), layer, out=Y2)
    assert torch.equal(Y, Y2)
    if batch == 1:
        assert torch.equal(P.forward_engine(X[0], layer, out_dtype=getattr(torch, ydt)), Y[0])
    with pytest.raises(ValueError):
        P.forward_engine(torch.zeros((5, m), device="cuda", dtype=torch.float16), layer)
    with pytest.raises(ValueError):
        P.forward_engine(torch.zeros((1, m + 1), device="cuda", dtype=torch.float16), layer)
