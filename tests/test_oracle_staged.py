"""The oracle restatement of the staged-gradient consumers (oracle/dbf_oracle.py) against golden
vectors produced by the reference itself (tests/golden/make_golden_staged.py): channel_scores
(budget.py:145-173) and _staged_loss_grads (factorize.py:310-326)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import dbf_oracle as npo

G = Path(__file__).resolve().parent / "golden" / "golden_staged.npz"


@pytest.fixture(scope="module")
def gs():
    with np.load(G) as z:
        return {k: z[k] for k in z.files}


def test_oracle_staged_matches_reference(gs):
    for i in range(int(gs["count"])):
        p = lambda s: gs[f"c{i}_{s}"]  # noqa: E731
        sc = npo.channel_scores([p("X0"), p("X1")], [p("Y0"), p("Y1")], p("Abits"), p("Bbits"), p("a"), p("mid"), p("b"))
        np.testing.assert_allclose(sc, p("scores"), rtol=1e-12, atol=0)
        loss, ga, gm, gb = npo.staged_loss_grads(p("X0"), p("Y0"), p("Abits"), p("Bbits"), p("a"), p("mid"), p("b"))
        assert loss == pytest.approx(float(p("loss")), rel=1e-12)
        for got, ref in ((ga, p("ga")), (gm, p("gm")), (gb, p("gb"))):
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_sign_projection_restatement_matches_reference(gs):
    """numpy restatement of the svid sign projection (the checker for pack_sign_of)."""
    for j in range(int(gs["scount"])):
        Z = gs[f"s{j}_Z"]
        np.testing.assert_array_equal(np.packbits(Z >= 0.0, axis=1, bitorder="little"), gs[f"s{j}_signs"])
        r, c = Z.shape
        S = npo.unpack_bits(gs[f"s{j}_S"], c)
        np.testing.assert_array_equal(npo.pack_bits(S.T), gs[f"s{j}_ST"])
