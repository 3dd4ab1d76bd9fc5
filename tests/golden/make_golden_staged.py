"""Golden fixtures of the staged-gradient consumers, produced by the REFERENCE package itself:
budget.channel_scores (budget.py:145-173), factorize._staged_loss_grads (factorize.py:310-326) and
factorize.refine_scales (factorize.py:335-370), on layers drawn like the reference's tests draw
theirs (pkg/tests/conftest.py:17-24, test_budget.py:94-145, test_factorize.py:231-290).

    python tests/golden/make_golden_staged.py      (build container; writes golden_staged.npz)
"""

from __future__ import annotations

# also: svid sign projection + packed transpose fixtures

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    import dbf
    from dbf.factorize import _staged_loss_grads

    rng = np.random.default_rng(20251018)
    g: dict[str, np.ndarray] = {}
    cases = [(6, 4, 5, 9), (8, 6, 8, 10), (40, 24, 70, 16), (100, 64, 257, 12), (33, 31, 129, 7)]
    for i, (n, k, m, batch) in enumerate(cases):
        A = rng.integers(0, 2, (n, k)) * 2.0 - 1.0
        B = rng.integers(0, 2, (k, m)) * 2.0 - 1.0
        a = np.abs(rng.standard_normal(n).astype(np.float32).astype(np.float64)) + 0.1
        mid = np.abs(rng.standard_normal(k).astype(np.float32).astype(np.float64)) + 0.1
        b = np.abs(rng.standard_normal(m).astype(np.float32).astype(np.float64)) + 0.1
        layer = dbf.DbfLayer(a=a, A=dbf.pack(A), mid=mid, B=dbf.pack(B), b=b)
        Xs = [rng.standard_normal((batch, m)) for _ in range(2)]
        Ys = [rng.standard_normal((batch, n)) for _ in range(2)]
        g[f"c{i}_Abits"], g[f"c{i}_Bbits"] = layer.A.bits, layer.B.bits
        g[f"c{i}_a"], g[f"c{i}_mid"], g[f"c{i}_b"] = a, mid, b
        g[f"c{i}_X0"], g[f"c{i}_X1"], g[f"c{i}_Y0"], g[f"c{i}_Y1"] = Xs[0], Xs[1], Ys[0], Ys[1]
        g[f"c{i}_scores"] = dbf.channel_scores(layer, Xs, Ys).scores
        loss, ga, gm, gb = _staged_loss_grads(Xs[0], Ys[0], dbf.unpack(layer.A), dbf.unpack(layer.B), a, mid, b)
        g[f"c{i}_loss"], g[f"c{i}_ga"], g[f"c{i}_gm"], g[f"c{i}_gb"] = np.array(loss), ga, gm, gb
        # refine: perturbation recovery (test_factorize.py:262-278)
        Xr = rng.standard_normal((4 * batch, m))
        Yr = dbf.forward(Xr, layer)
        pert = dbf.DbfLayer(a=a * (1 + 0.1 * rng.standard_normal(n)), A=layer.A,
                            mid=mid * (1 + 0.1 * rng.standard_normal(k)), B=layer.B,
                            b=b * (1 + 0.1 * rng.standard_normal(m)))
        out = dbf.refine_scales(pert, Xr, Yr, steps=20, lr=1e-3)
        g[f"c{i}_Xr"], g[f"c{i}_Yr"] = Xr, Yr
        g[f"c{i}_pa"], g[f"c{i}_pmid"], g[f"c{i}_pb"] = pert.a, pert.mid, pert.b
        g[f"c{i}_ra"], g[f"c{i}_rmid"], g[f"c{i}_rb"] = out.a, out.mid, out.b
        g[f"c{i}_rloss"] = np.array(float(np.sum((dbf.forward(Xr, out) - Yr) ** 2)))
        g[f"c{i}_ploss"] = np.array(float(np.sum((dbf.forward(Xr, pert) - Yr) ** 2)))
    g["count"] = np.array(len(cases))
    # sign packing inside the factorization loop: svid's sign projection
    # (svid.py:99-103) and _assemble's transpose (factorize.py:193-195)
    shapes = [(1, 1), (7, 9), (33, 31), (64, 100), (130, 257)]
    for j, (r, c) in enumerate(shapes):
        Z = rng.standard_normal((r, c))
        Z[rng.random((r, c)) < 0.05] = 0.0  # zeros project to +1
        g[f"s{j}_Z"] = Z
        g[f"s{j}_signs"] = dbf.svid(Z).signs.bits
        S = dbf.pack(rng.integers(0, 2, (r, c)) * 2.0 - 1.0)
        g[f"s{j}_S"] = S.bits
        g[f"s{j}_ST"] = dbf.pack(dbf.unpack(S).T).bits
    g["scount"] = np.array(len(shapes))
    np.savez_compressed(OUT / "golden_staged.npz", **g)
    print(f"wrote {OUT / 'golden_staged.npz'} ({len(g)} arrays)")


if __name__ == "__main__":
    main()
