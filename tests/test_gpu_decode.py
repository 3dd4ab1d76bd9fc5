"""GPU decode parity: sign_matvec / forward against the reference (golden.npz) and the oracle.

Tolerances: the reference's own for the float64 drop-in path (1e-5 / 1e-4 norm-relative,
test_kernel.py:26, 80; exact on integer inputs); north_star's for the fp16 path
(max|err| / max|ref| <= 1e-2 and norm-relative <= 1e-2).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2505_11076_b200 as P  # noqa: E402
import oracle  # noqa: E402
from conftest import f32_vector, random_signs, rel_max, rel_norm  # noqa: E402

FP16_TOL = 1e-2


def _layer(golden, i):
    A = golden[f"fw{i}_Abits"]
    B = golden[f"fw{i}_Bbits"]
    k, m = len(golden[f"fw{i}_mid"]), len(golden[f"fw{i}_b"])
    return P.DbfLayer(a=golden[f"fw{i}_a"], A=P.SignMatrix(A.shape[0], k, A.copy()),
                      mid=golden[f"fw{i}_mid"], B=P.SignMatrix(B.shape[0], m, B.copy()), b=golden[f"fw{i}_b"])


# ---- the reference's own kernel tests, verbatim semantics -------------------------------------
def test_all_plus_ones():
    s = P.pack(np.ones((4, 6)))
    assert np.array_equal(P.sign_matvec(s, np.ones(6)), np.full(4, 6.0))


def test_single_row():
    s = P.pack(np.array([[1.0, -1.0, 1.0]]))
    assert P.sign_matvec(s, np.array([1.0, 2.0, 3.0])) == pytest.approx([2.0])


def test_scalar_layer():
    layer = P.DbfLayer(a=np.array([2.0]), A=P.pack(np.array([[1.0]])), mid=np.array([3.0]),
                       B=P.pack(np.array([[-1.0]])), b=np.array([5.0]))
    assert P.forward(np.array([[1.0]]), layer) == pytest.approx(np.array([[-30.0]]))


def test_length_and_column_errors(rng):
    s = P.pack(random_signs(rng, 3, 5))
    with pytest.raises(ValueError, match="length"):
        P.sign_matvec(s, np.ones(6))
    layer = P.DbfLayer(a=np.ones(4), A=P.pack(random_signs(rng, 4, 3)), mid=np.ones(3),
                       B=P.pack(random_signs(rng, 3, 6)), b=np.ones(6))
    with pytest.raises(ValueError, match="columns"):
        P.forward(np.ones((2, 5)), layer)


# ---- golden vectors -------------------------------------------------------------------------
def test_sign_matvec_matches_reference(golden):
    for i in range(int(golden["smv_count"])):
        bits, cols, x, ref = golden[f"smv{i}_bits"], int(golden[f"smv{i}_cols"]), golden[f"smv{i}_x"], golden[f"smv{i}_out"]
        s = P.SignMatrix(bits.shape[0], cols, bits.copy())
        out = P.sign_matvec(s, x)
        assert np.linalg.norm(out - ref) <= 1e-5 * max(np.linalg.norm(ref), 1.0), i


def test_integer_inputs_exact(golden):
    i = int(golden["smv_integer_case"])
    bits, cols = golden[f"smv{i}_bits"], int(golden[f"smv{i}_cols"])
    out = P.sign_matvec(P.SignMatrix(bits.shape[0], cols, bits.copy()), golden[f"smv{i}_x"])
    assert np.array_equal(out, golden[f"smv{i}_out"])  # test_kernel.py:28-33


def test_padding_bits_never_contribute(rng):
    S = random_signs(rng, 6, 13)
    s = P.pack(S)
    x = rng.standard_normal(13)
    base = P.sign_matvec(s, x)
    flipped = s.bits.copy()
    flipped[:, -1] ^= 0b11100000
    assert np.array_equal(P.sign_matvec(P.SignMatrix(6, 13, flipped), x), base)


def test_bitwise_reproducible(rng):
    s = P.pack(random_signs(rng, 500, 3000))
    x = rng.standard_normal(3000)
    first = P.sign_matvec(s, x)
    for _ in range(3):
        assert np.array_equal(P.sign_matvec(s, x), first)


def test_forward_matches_reference(golden):
    for i in range(int(golden["fw_count"])):
        out = P.forward(golden[f"fw{i}_X"], _layer(golden, i))
        ref = golden[f"fw{i}_out"]
        assert np.linalg.norm(out - ref) <= 1e-4 * max(np.linalg.norm(ref), 1e-9), i


def test_forward_identity_probe_equals_reconstruction(golden):
    for i in (1, 2, 3, 50):
        layer = _layer(golden, i)
        out = P.forward(np.eye(layer.m_dim), layer)
        ref = golden[f"fw{i}_recon"].T
        assert np.linalg.norm(out - ref) <= 1e-4 * np.linalg.norm(ref)
        assert np.allclose(P.reconstruct(layer), golden[f"fw{i}_recon"], rtol=1e-12, atol=1e-12)


def test_dbf1_loaded_layer(golden):
    import io

    layer = P.load_dbf(io.BytesIO(golden["dbf1_bytes"].tobytes()))
    out = P.forward(golden["dbf1_X"], layer)
    assert np.linalg.norm(out - golden["dbf1_out"]) <= 1e-5 * np.linalg.norm(golden["dbf1_out"])


# ---- fp16 performance path (north_star tolerance) ---------------------------------------------
def _fp16_device_layer(golden, i):
    import torch

    return P.DeviceLayer.from_host(_layer(golden, i), scale_dtype=torch.float16)


def test_fp16_path_within_tolerance(golden):
    import torch

    i = int(golden["fw_fp16_case"])
    dl = _fp16_device_layer(golden, i)
    X = torch.from_numpy(golden[f"fw{i}_X"]).to("cuda", torch.float16)
    out = P.forward_device(X, dl).float().cpu().numpy()
    ref = golden[f"fw{i}_out"]
    assert rel_max(out, ref) <= FP16_TOL
    assert rel_norm(out, ref) <= FP16_TOL


@pytest.mark.parametrize("batch", [1, 2, 3, 4, 5, 8, 9, 16, 17])
def test_batches_fp32_path(rng, batch):
    import torch

    n, k, m = 300, 416, 520
    A, B = random_signs(rng, n, k), random_signs(rng, k, m)
    a, mid, b = f32_vector(rng, n), f32_vector(rng, k), f32_vector(rng, m)
    X = rng.standard_normal((batch, m))
    ref = oracle.c_forward(X, a, np.packbits(A > 0, axis=1, bitorder="little"), mid,
                           np.packbits(B > 0, axis=1, bitorder="little"), b)
    layer = P.DbfLayer(a=a, A=P.pack(A), mid=mid, B=P.pack(B), b=b)
    out = P.forward(X, layer)
    assert rel_norm(out, ref) <= 1e-6
    dl = P.DeviceLayer.from_host(layer, scale_dtype=torch.float32)
    o32 = P.forward_device(torch.from_numpy(X).float().cuda(), dl).cpu().numpy()
    assert rel_norm(o32, ref) <= 1e-5


# ---- full Llama-2 shapes, fp16 path vs the C oracle ------------------------------------------
LLAMA = {
    "7b_q_2bpw": (4096, 4096, 4096),
    "7b_gate_2bpw": (11008, 5952, 4096),
    "7b_down_2bpw": (4096, 5952, 11008),
    "7b_gate_1bpw": (11008, 2976, 4096),
    "70b_kv_2bpw": (1024, 1792, 8192),
    "70b_down_2bpw": (8192, 12736, 28672),
}


@pytest.mark.parametrize("name", list(LLAMA))
def test_llama_shapes_fp16_vs_oracle(name):
    import torch

    n, k, m = LLAMA[name]
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    dl = P.random_device_layer(n, k, m, generator=g, keep_words=True)  # fp16 scales
    X = torch.randn((1, m), generator=g, device="cuda").half()
    y = P.forward_device(X, dl).float().cpu().numpy()
    # oracle on the identical bytes and fp16-exact values
    A_bytes = dl.A.to_host().bits
    B_bytes = dl.B.to_host().bits
    ref = oracle.c_forward(X.double().cpu().numpy(), dl.a.double().cpu().numpy(), A_bytes,
                           dl.mid.double().cpu().numpy(), B_bytes, dl.b.double().cpu().numpy())
    assert rel_max(y, ref) <= FP16_TOL, rel_max(y, ref)
    assert rel_norm(y, ref) <= FP16_TOL
