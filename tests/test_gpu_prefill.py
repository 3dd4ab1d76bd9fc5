"""GPU parity of the tcgen05 prefill path (dbf_forward_prefill / dbf_sign_gemm).

The prefill path computes in fp16 (north_star): products are exact, sums are fp32 in tensor
memory, the intermediate t is rounded to fp16.  Tolerance (stated here):
max|err| / max|ref| <= 1e-2 and ||err|| / ||ref|| <= 1e-2 against the oracle's float64 forward
(kernel.py:48-62 restated) on the identical packed bytes and fp16-exact inputs.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2505_11076_b200 as P  # noqa: E402
from paper_2505_11076_b200 import _lib  # noqa: E402
from conftest import random_signs, rel_max, rel_norm  # noqa: E402

TOL = 1e-2


def _host_layer(rng, n, k, m):
    A, B = random_signs(rng, n, k), random_signs(rng, k, m)
    a = (rng.uniform(0.5, 1.5, n) / np.sqrt(k)).astype(np.float16).astype(np.float64)
    mid = rng.uniform(0.5, 1.5, k).astype(np.float16).astype(np.float64)
    b = (rng.uniform(0.5, 1.5, m) / np.sqrt(m)).astype(np.float16).astype(np.float64)
    bits_a = np.packbits(A > 0, axis=1, bitorder="little")
    bits_b = np.packbits(B > 0, axis=1, bitorder="little")
    return P.DbfLayer(a=a, A=P.SignMatrix(n, k, bits_a), mid=mid, B=P.SignMatrix(k, m, bits_b), b=b)


@pytest.mark.parametrize(
    "T,n,k,m",
    [
        (64, 128, 64, 64),        # minimum prefill batch, one tile everywhere
        (256, 384, 320, 512),     # exact tiles
        (300, 200, 96, 130),      # ragged tokens / rows / K; m % 8 != 0 exercises the padded copy
        (257, 1000, 160, 1000),   # tails on every dimension
        (1024, 256, 2048, 256),   # long GEMM2 K
        (64, 1024, 2048, 4096),   # small T: MMA N = 64, K split over ~148 CTAs (both GEMMs)
        (100, 512, 1024, 3000),   # small ragged T, ragged split tail
        (200, 2048, 512, 1000),   # GEMM1 split, GEMM2 (K = 512) too short to split
        (64, 256, 128, 28672),    # GEMM1 K = 28672 (70B down): kscale read from global, split K
        (260, 128, 64, 30000),    # wide K without split, ragged K tail through the global kscale
    ],
)
def test_prefill_matches_oracle(rng, T, n, k, m):
    layer = _host_layer(rng, n, k, m)
    X = rng.standard_normal((T, m)).astype(np.float16).astype(np.float64)
    ref = oracle.c_forward(X, layer.a, layer.A.bits, layer.mid, layer.B.bits, layer.b)
    dl = P.DeviceLayer.from_host(layer, scale_dtype=torch.float16)
    Y = P.forward_prefill(torch.from_numpy(X).cuda().half(), dl).float().cpu().numpy()
    assert rel_max(Y, ref) <= TOL, rel_max(Y, ref)
    assert rel_norm(Y, ref) <= TOL, rel_norm(Y, ref)


def test_forward_device_routes_fp16_batches_to_prefill(rng):
    layer = _host_layer(rng, 192, 128, 256)
    dl = P.DeviceLayer.from_host(layer, scale_dtype=torch.float16)
    X = torch.from_numpy(rng.standard_normal((128, 256))).cuda().half()
    assert torch.equal(P.forward_device(X, dl), P.forward_prefill(X, dl))
    # below the threshold the exact-integer GEMV runs; both agree within the fp16 tolerance
    small = P.forward_device(X[:8], dl).float()
    big = P.forward_device(X, dl)[:8].float()
    assert (small - big).abs().max().item() <= TOL * small.abs().max().item()


def test_sign_gemm_matches_torch_reference():
    """One staged sign GEMM at a Llama-2-7B q shape (k = 2048, T = 2048) against the plain
    PyTorch fp32 reference of the same op on the unpacked signs."""
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    T, rows, K = 2048, 2048, 4096
    layer = P.random_device_layer(4096, rows, K, generator=g, keep_words=True)
    X = torch.randn((T, K), generator=g, device="cuda").half()
    out = torch.empty((T, rows), dtype=torch.half, device="cuda")
    S = layer.B.paired
    _lib.check(_lib.lib.dbf_sign_gemm(X.data_ptr(), T, K, K, S.data_ptr(), S.shape[1], rows, layer.b.data_ptr(),
                                      layer.mid.data_ptr(), out.data_ptr(), rows, _lib.stream_ptr()), "gemm")
    ref = layer.mid.float()[None, :] * ((X.float() * layer.b.float()[None, :]) @ layer.B.unpack(torch.float32).t())
    err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err <= TOL


def test_full_size_prefill_is_deterministic_and_finite():
    """Llama-2-7B MLP gate shape at 1 bpw (n=11008, k=2976, m=4096), 2048 tokens: run twice,
    bitwise identical (no atomics, fixed reduction order) and finite; spot-check 16 tokens
    against the float64 oracle on the same bytes."""
    g = torch.Generator(device="cuda")
    g.manual_seed(2)
    n, k, m, T = 11008, 2976, 4096, 2048
    dl = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    X = torch.randn((T, m), generator=g, device="cuda").half()
    Y1 = P.forward_prefill(X, dl)
    Y2 = P.forward_prefill(X, dl)
    assert torch.equal(Y1, Y2)
    assert torch.isfinite(Y1).all()
    rows = torch.arange(0, T, T // 16, device="cuda")
    host = dl.A.to_host(), dl.B.to_host()
    ref = oracle.c_forward(X[rows].double().cpu().numpy(), dl.a.double().cpu().numpy(), host[0].bits,
                           dl.mid.double().cpu().numpy(), host[1].bits, dl.b.double().cpu().numpy())
    out = Y1[rows].double().cpu().numpy()
    assert rel_max(out, ref) <= TOL and rel_norm(out, ref) <= TOL


def test_pair_layout_round_trip(rng):
    """dbf_pair_signs: bit q <-> column 2q, bit 16+q <-> column 2q+1 of every 32-column group."""
    rows, cols = 37, 200
    D = random_signs(rng, rows, cols)
    s = P.DeviceSignMatrix.pack(D)
    paired = s.paired.cpu().numpy().view(np.uint32)
    words = s.words.cpu().numpy().view(np.uint32)
    for j in range(words.shape[1]):
        for q in range(16):
            lo = (paired[:, j] >> q) & 1
            hi = (paired[:, j] >> (16 + q)) & 1
            assert np.array_equal(lo, (words[:, j] >> (2 * q)) & 1)
            assert np.array_equal(hi, (words[:, j] >> (2 * q + 1)) & 1)


def test_small_batch_split_k_is_deterministic():
    """T = 64 at the Llama-2-13B MLP shape (1.5 bpw): the split-K partials are summed in split
    order, so two runs are bitwise identical; a workspace too small for the partials runs the
    unsplit GEMMs, equal within the fp16 tolerance."""
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    n, k, m, T = 13824, 5600, 5120, 64
    dl = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    X = torch.randn((T, m), generator=g, device="cuda").half()
    Y1 = P.forward_prefill(X, dl)
    Y2 = P.forward_prefill(X, dl)
    assert torch.equal(Y1, Y2) and torch.isfinite(Y1).all()
    ws = torch.empty(_lib.lib.dbf_prefill_workspace_bytes(k, T), dtype=torch.uint8, device="cuda")
    Y0 = torch.empty_like(Y1)
    A, B = dl.A.paired, dl.B.paired
    _lib.check(_lib.lib.dbf_forward_prefill(
        A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], dl.a.data_ptr(), dl.mid.data_ptr(), dl.b.data_ptr(),
        n, k, m, X.data_ptr(), T, X.stride(0), Y0.data_ptr(), Y0.stride(0), ws.data_ptr(), ws.numel(),
        _lib.stream_ptr()), "dbf_forward_prefill")
    err = (Y0.float() - Y1.float()).abs().max().item() / Y0.float().abs().max().item()
    assert err <= TOL


def _two_launch(X, dl):
    """The same layer as two per-tile sign GEMM launches (dbf_sign_gemm): t = mid * (X . (B*b)^T),
    Y = a * (t . A^T) -- the path forward_prefill took before the one-launch layer kernel."""
    T, m = X.shape
    n, k = dl.n, dl.k
    ldt = _lib.lib.dbf_prefill_ld(k)
    t = torch.empty((T, ldt), dtype=torch.half, device="cuda")
    Y = torch.empty((T, n), dtype=torch.half, device="cuda")
    A, B = dl.A.paired, dl.B.paired
    _lib.check(_lib.lib.dbf_sign_gemm(X.data_ptr(), T, m, X.stride(0), B.data_ptr(), B.shape[1], k, dl.b.data_ptr(),
                                      dl.mid.data_ptr(), t.data_ptr(), ldt, _lib.stream_ptr()), "gemm1")
    _lib.check(_lib.lib.dbf_sign_gemm(t.data_ptr(), T, k, ldt, A.data_ptr(), A.shape[1], n, None,
                                      dl.a.data_ptr(), Y.data_ptr(), n, _lib.stream_ptr()), "gemm2")
    return Y


@pytest.mark.parametrize(
    "T,n,k,m",
    [
        (2048, 4096, 2048, 4096),    # Llama-2-7B q at 1 bpw (128 GEMM1 + 256 GEMM2 tiles; auto: two launches)
        (2048, 4096, 2976, 11008),   # 7B down: long GEMM1 K, ragged k (last row tile 32 rows)
        (768, 11008, 2976, 4096),    # 7B gate, 3 token blocks
        (300, 200, 96, 130),         # ragged everything, partial second token block
        (1000, 1000, 160, 1000),
        (520, 256, 2048, 28672),     # GEMM1 K = 28672: the kscale from global memory
    ],
)
def test_layer_kernel_bitwise_equals_two_launches(T, n, k, m):
    """T > 256 runs the whole layer as ONE persistent launch (GEMM2 tiles wait on per-token-block
    counters of GEMM1 tiles).  Same K order, same fp32 accumulation, same rounding: bitwise equal to
    the two per-tile launches, on every run (dynamic tile claiming must not change any bit)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(T + n)
    dl = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    # rows padded to 16 bytes (the TMA row pitch), as forward_prefill pads a ragged X
    X = torch.randn((T, (m + 7) // 8 * 8), generator=g, device="cuda").half()[:, :m]
    ref = _two_launch(X, dl)
    assert torch.equal(P.forward_prefill(X, dl, path="two_launches"), ref)
    for _ in range(3):
        Y = P.forward_prefill(X, dl, path="one_launch")
        assert torch.equal(Y, ref)
    assert torch.equal(P.forward_prefill(X, dl), ref)  # whichever path auto picks
    assert torch.isfinite(ref).all()


def test_prefill_auto_path_rule():
    """dbf_prefill_layer_path: one launch where GEMM1's k/128 x T/256 tiles exceed the SM count,
    two launches otherwise and for T <= 256 (measured crossover)."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    f = _lib.lib.dbf_prefill_layer_path
    assert f(4096, 2048, 4096, 2048) == (2 if 16 * 8 > sms else 1)
    assert f(11008, 2976, 4096, 2048) == (2 if 24 * 8 > sms else 1)
    assert f(11008, 2976, 4096, 256) == 1
    X = torch.zeros((300, 64), dtype=torch.half, device="cuda")
    dl = P.random_device_layer(64, 64, 64, keep_words=True)
    with pytest.raises(ValueError):
        P.forward_prefill(X, dl, path="fastest")


def test_one_launch_needs_tma_compatible_output():
    """The one-launch kernel stores Y with TMA (16-byte row pitch).  Asked for explicitly with a
    ragged Y it reports DBF_ERR_UNSUPPORTED; the auto path falls back to two launches, same bits."""
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    n, k, m, T = 100, 2048, 512, 600      # ldy = 100 halves = 200 bytes per row
    dl = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    X = torch.randn((T, m), generator=g, device="cuda").half()
    with pytest.raises(_lib.DbfNativeError):
        P.forward_prefill(X, dl, path="one_launch")
    assert torch.equal(P.forward_prefill(X, dl), _two_launch(X, dl))
