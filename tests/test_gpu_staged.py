"""GPU staged-gradient consumers (paper_2505_11076_b200.staged) against the reference's golden
outputs and the reference's own semantic tests (test_budget.py:94-161, test_factorize.py:231-290):
exact zero score for a zero mid channel, equal scores for duplicated channels, finite-difference
gradients, exact targets leave the layer unchanged, monotone loss, perturbation recovery."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2505_11076_b200 as P  # noqa: E402
from conftest import random_signs  # noqa: E402

G = Path(__file__).resolve().parent / "golden" / "golden_staged.npz"


@pytest.fixture(scope="module")
def gs():
    with np.load(G) as z:
        return {k: z[k] for k in z.files}


def _layer_of(gs, i, pre=""):
    p = lambda s: gs[f"c{i}_{s}"]  # noqa: E731
    k, m = len(p("mid")), len(p("b"))
    A, B = p("Abits"), p("Bbits")
    a = p(pre + "a") if pre else p("a")
    mid = p(pre + "mid") if pre else p("mid")
    b = p(pre + "b") if pre else p("b")
    return P.DbfLayer(a=a, A=P.SignMatrix(A.shape[0], k, A.copy()), mid=mid,
                      B=P.SignMatrix(B.shape[0], m, B.copy()), b=b)


def random_layer(rng, n, k, m, positive=True):
    """pkg/tests/conftest.py:17-24"""
    def vec(size):
        v = rng.standard_normal(size).astype(np.float32).astype(np.float64)
        return np.abs(v) + 0.1 if positive else v
    return P.DbfLayer(a=vec(n), A=P.pack(random_signs(rng, n, k)), mid=vec(k), B=P.pack(random_signs(rng, k, m)),
                      b=vec(m))


def test_transposed_signs_are_the_transpose(rng):
    D = random_signs(rng, 37, 70)
    s = P.DeviceSignMatrix.pack(D)
    np.testing.assert_array_equal(s.transposed().unpack().cpu().numpy(), D.T)
    np.testing.assert_array_equal(s.transposed().transposed().words.cpu().numpy(), s.words.cpu().numpy())


def test_channel_scores_and_grads_match_reference(gs):
    for i in range(int(gs["count"])):
        p = lambda s: gs[f"c{i}_{s}"]  # noqa: E731
        layer = _layer_of(gs, i)
        sc = P.channel_scores(layer, [p("X0"), p("X1")], [p("Y0"), p("Y1")]).scores
        np.testing.assert_allclose(sc, p("scores"), rtol=1e-9, atol=1e-12 * np.abs(p("scores")).max())
        loss, ga, gm, gb = P.staged_loss_grads(p("X0"), p("Y0"), layer)
        assert loss == pytest.approx(float(p("loss")), rel=1e-10)
        for got, ref in ((ga, p("ga")), (gm, p("gm")), (gb, p("gb"))):
            np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-10 * np.abs(ref).max())


def test_refine_scales_recovers_like_the_reference(gs):
    for i in range(int(gs["count"])):
        p = lambda s: gs[f"c{i}_{s}"]  # noqa: E731
        pert = _layer_of(gs, i, pre="p")
        out = P.refine_scales(pert, p("Xr"), p("Yr"), steps=20, lr=1e-3)
        ref_out = oracle.c_forward(p("Xr"), out.a, out.A.bits, out.mid, out.B.bits, out.b)  # float64
        loss = float(np.sum((ref_out - p("Yr")) ** 2))
        ploss = float(p("ploss"))
        # same guarded descent on the same data: the same loss trajectory up to float64 noise
        assert loss <= ploss
        assert loss == pytest.approx(float(p("rloss")), rel=1e-6, abs=1e-9 * ploss)
        np.testing.assert_allclose(out.a, p("ra"), rtol=1e-6)
        np.testing.assert_allclose(out.mid, p("rmid"), rtol=1e-6)
        np.testing.assert_allclose(out.b, p("rb"), rtol=1e-6)


def test_zero_mid_gives_zero_score(rng):
    layer = random_layer(rng, 8, 6, 8)
    mid = layer.mid.copy()
    mid[2] = 0.0
    layer = P.DbfLayer(a=layer.a, A=layer.A, mid=mid, B=layer.B, b=layer.b)
    assert P.channel_scores(layer, [rng.standard_normal((5, 8))], [rng.standard_normal((5, 8))]).scores[2] == 0.0


def test_duplicated_channels_score_equally(rng):
    n, k, m = 8, 6, 8
    Ad = random_signs(rng, n, k)
    Ad[:, 3] = Ad[:, 2]
    Bd = random_signs(rng, k, m)
    Bd[3] = Bd[2]
    mid = np.abs(rng.standard_normal(k)) + 0.3
    mid[3] = mid[2]
    layer = P.DbfLayer(a=np.abs(rng.standard_normal(n)) + 0.3, A=P.pack(Ad), mid=mid, B=P.pack(Bd),
                       b=np.abs(rng.standard_normal(m)) + 0.3)
    sc = P.channel_scores(layer, [rng.standard_normal((7, m))], [rng.standard_normal((7, n))]).scores
    assert sc[2] == sc[3]


def test_scores_match_finite_differences(rng):
    layer = random_layer(rng, 8, 6, 8)
    X = [rng.standard_normal((10, 8)) for _ in range(3)]
    Y = [rng.standard_normal((10, 8)) for _ in range(3)]
    got = P.channel_scores(layer, X, Y).scores
    Ad = np.unpackbits(layer.A.bits, axis=1, count=6, bitorder="little") * 2.0 - 1.0
    Bd = np.unpackbits(layer.B.bits, axis=1, count=8, bitorder="little") * 2.0 - 1.0

    def loss(mid, Xb, Yb):
        return np.sum(((Xb * layer.b) @ Bd.T * mid @ Ad.T * layer.a - Yb) ** 2)

    h = 1e-4
    fd = np.zeros(6)
    for i in range(6):
        for Xb, Yb in zip(X, Y):
            up, dn = layer.mid.copy(), layer.mid.copy()
            up[i] += h
            dn[i] -= h
            fd[i] += (((loss(up, Xb, Yb) - loss(dn, Xb, Yb)) / (2 * h)) * layer.mid[i]) ** 2
    assert np.allclose(got, fd, rtol=1e-4)


def test_exact_targets_leave_layer_unchanged(rng):
    layer = random_layer(rng, 6, 4, 5)
    X = rng.standard_normal((12, 5))
    Ad = np.unpackbits(layer.A.bits, axis=1, count=4, bitorder="little") * 2.0 - 1.0
    Bd = np.unpackbits(layer.B.bits, axis=1, count=5, bitorder="little") * 2.0 - 1.0
    Y = (X * layer.b) @ Bd.T * layer.mid @ Ad.T * layer.a  # float64 staged forward
    out = P.refine_scales(layer, X, Y, steps=50, lr=1e-3)
    assert np.allclose(out.a, layer.a, atol=1e-12)
    assert np.allclose(out.mid, layer.mid, atol=1e-12)
    assert np.allclose(out.b, layer.b, atol=1e-12)


def test_loss_monotone_nonincreasing(rng):
    layer = random_layer(rng, 5, 3, 4)
    X = rng.standard_normal((8, 4))
    Y = rng.standard_normal((8, 5))
    prev = P.staged_loss_grads(X, Y, layer)[0]
    current = layer
    for _ in range(10):
        current = P.refine_scales(current, X, Y, steps=1, lr=1e-2)
        now = P.staged_loss_grads(X, Y, current)[0]
        assert now <= prev + 1e-9 * prev
        prev = now


def test_rejects_bad_batches(rng):
    layer = random_layer(rng, 8, 6, 8)
    with pytest.raises(ValueError, match="batch"):
        P.channel_scores(layer, [], [])
    with pytest.raises(ValueError):
        P.channel_scores(layer, [np.ones((4, 5))], [np.ones((4, 8))])


def test_factorization_sign_packing_matches_reference(gs):
    """svid sign projection (svid.py:99-103) and the packed transpose of _assemble
    (factorize.py:193-195): bit-exact against the reference's own packed bytes."""
    for j in range(int(gs["scount"])):
        Z = gs[f"s{j}_Z"]
        np.testing.assert_array_equal(P.pack_sign_of(Z).bits, gs[f"s{j}_signs"])
        S = gs[f"s{j}_S"]
        r, c = Z.shape
        T = P.transpose_signs(P.SignMatrix(r, c, S.copy()))
        assert (T.rows, T.cols) == (c, r)
        np.testing.assert_array_equal(T.bits, gs[f"s{j}_ST"])
