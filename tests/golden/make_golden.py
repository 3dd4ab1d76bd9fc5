"""Generate the golden fixtures of the DBF hot path from the REFERENCE package itself.

Run in the build container (the reference is importable from /root/reference/pkg/src; it does
not exist on the GPU box, so its outputs are frozen here as small .npz fixtures):

    python tests/golden/make_golden.py

Every output array below is produced by the reference's own functions -- dbf.pack
(bitcore.py:72-85), dbf.unpack (88-91), dbf.sign_matvec (kernel.py:24-45), dbf.forward
(kernel.py:48-62), dbf.save_dbf (bitcore.py:149-170), dbf.middle_dim (budget.py:113-132) -- on
inputs drawn like the reference tests draw theirs (pkg/tests/conftest.py:7-24,
test_kernel.py:20-45, test_acceptance.py:79-96, 241-245).
"""

from __future__ import annotations

import io
import sys
import warnings
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _import_reference():
    sys.path.insert(0, str(REF))
    import dbf  # noqa: E402

    return dbf


def random_signs(rng, rows, cols):
    """conftest.py:7-8"""
    return rng.integers(0, 2, size=(rows, cols)).astype(np.float64) * 2.0 - 1.0


def f32_vector(rng, size, positive=False):
    """conftest.py:11-14"""
    vals = rng.standard_normal(size).astype(np.float32).astype(np.float64)
    return np.abs(vals) + 0.1 if positive else vals


def f16_scales(rng, size, div):
    """U(0.5,1.5)/div rounded through fp16."""
    return ((rng.uniform(0.5, 1.5, size) / div).astype(np.float16)).astype(np.float64)


def main():
    dbf = _import_reference()
    rng = np.random.default_rng(20250517)
    g: dict[str, np.ndarray] = {}

    # ---- pack / unpack -----------------------------------------------------------------
    packs = [np.array([[1, -1, -1, 1, 1, 1, -1, 1]], dtype=float), np.ones((2, 2))]
    for _ in range(60):
        packs.append(random_signs(rng, int(rng.integers(1, 25)), int(rng.integers(1, 71))))
    for cols in (1, 7, 8, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 300):
        packs.append(random_signs(rng, 5, cols))
    for i, d in enumerate(packs):
        s = dbf.pack(d)
        g[f"pack{i}_dense"] = d.astype(np.int8)
        g[f"pack{i}_bits"] = s.bits.copy()
        assert np.array_equal(dbf.unpack(s), d)
    g["pack_count"] = np.array(len(packs))
    # first-offending-index error cases (bitcore.py:79-82)
    bad = []
    for shape, pos, val in (((3, 4), (1, 2), 0.5), ((2, 2), (0, 0), 0.0), ((4, 9), (3, 8), np.nan), ((5, 5), (2, 1), -2.0)):
        M = np.ones(shape)
        M[pos] = val
        if val != 0.0:
            M[-1, -1] = 0.0  # a later offender must not win
        try:
            dbf.pack(M)
        except ValueError as e:
            msg = str(e)
        bad.append((shape, pos, msg))
    g["packbad_msgs"] = np.array([m for _, _, m in bad])
    g["packbad_pos"] = np.array([p for _, p, _ in bad])

    # ---- sign_matvec ---------------------------------------------------------------------
    smv = []
    for cols in (7, 8, 64, 65, 130):  # test_kernel.py:20-26
        S = random_signs(rng, 11, cols)
        smv.append((S, rng.standard_normal(cols)))
    S = random_signs(rng, 9, 333)  # test_kernel.py:28-33 (integer inputs)
    smv.append((S, rng.integers(-1000, 1001, size=333).astype(np.float64)))
    for _ in range(24):
        rows, cols = int(rng.integers(1, 48)), int(rng.integers(1, 700))
        smv.append((random_signs(rng, rows, cols), rng.standard_normal(cols) * rng.uniform(0.01, 100)))
    smv.append((random_signs(rng, 70, 4100), rng.standard_normal(4100)))  # > 16 chunks
    smv.append((random_signs(rng, 33, 2976), rng.standard_normal(2976)))  # 7B 1-bpw k (not /256)
    for i, (S, x) in enumerate(smv):
        s = dbf.pack(S)
        g[f"smv{i}_bits"] = s.bits.copy()
        g[f"smv{i}_cols"] = np.array(S.shape[1])
        g[f"smv{i}_x"] = x
        g[f"smv{i}_out"] = dbf.sign_matvec(s, x)
    g["smv_count"] = np.array(len(smv))
    g["smv_integer_case"] = np.array(5)

    # ---- forward -----------------------------------------------------------------------
    fw = []
    fw.append(dict(a=np.array([2.0]), A=np.array([[1.0]]), mid=np.array([3.0]), B=np.array([[-1.0]]),
                   b=np.array([5.0]), X=np.array([[1.0]])))  # test_kernel.py:59-66 -> -30
    r5 = np.random.default_rng(5)
    for case in range(100):  # test_acceptance.py:79-96 regimes
        n, m = int(r5.integers(3, 40)), int(r5.integers(3, 40))
        regime = case % 3
        if regime == 0:
            k = int(r5.integers(1, max(2, min(n, m))))
        elif regime == 1:
            k = n
        else:
            k = max(n, m) + int(r5.integers(1, 9))
        fw.append(dict(a=f32_vector(r5, n), A=random_signs(r5, n, k), mid=f32_vector(r5, k),
                       B=random_signs(r5, k, m), b=f32_vector(r5, m), X=r5.standard_normal((4, m))))
    for n, k, m, batch in ((300, 160, 520, 3), (1000, 512, 700, 2), (257, 300, 129, 17)):
        fw.append(dict(a=f32_vector(rng, n), A=random_signs(rng, n, k), mid=f32_vector(rng, k),
                       B=random_signs(rng, k, m), b=f32_vector(rng, m), X=rng.standard_normal((batch, m))))
    # fp16-exact layer for the fp16 tolerance test
    n, k, m = 512, 320, 768
    fw.append(dict(a=f16_scales(rng, n, k**0.5), A=random_signs(rng, n, k), mid=f16_scales(rng, k, 1.0),
                   B=random_signs(rng, k, m), b=f16_scales(rng, m, m**0.5),
                   X=rng.standard_normal((2, m)).astype(np.float16).astype(np.float64)))
    for i, c in enumerate(fw):
        layer = dbf.DbfLayer(a=c["a"], A=dbf.pack(c["A"]), mid=c["mid"], B=dbf.pack(c["B"]), b=c["b"])
        for key in ("a", "mid", "b", "X"):
            g[f"fw{i}_{key}"] = c[key]
        g[f"fw{i}_Abits"] = layer.A.bits.copy()
        g[f"fw{i}_Bbits"] = layer.B.bits.copy()
        g[f"fw{i}_out"] = dbf.forward(c["X"], layer)
        if i < 101:
            g[f"fw{i}_recon"] = dbf.reconstruct(layer)
    g["fw_count"] = np.array(len(fw))
    g["fw_fp16_case"] = np.array(len(fw) - 1)

    # ---- DBF1 file bytes (bitcore.py:149-211) ------------------------------------------------
    layer = dbf.DbfLayer(a=f32_vector(rng, 7), A=dbf.pack(random_signs(rng, 7, 5)), mid=f32_vector(rng, 5),
                         B=dbf.pack(random_signs(rng, 5, 11)), b=f32_vector(rng, 11))
    buf = io.BytesIO()
    dbf.save_dbf(layer, buf)
    g["dbf1_bytes"] = np.frombuffer(buf.getvalue(), dtype=np.uint8).copy()
    g["dbf1_X"] = rng.standard_normal((3, 11))
    g["dbf1_out"] = dbf.forward(g["dbf1_X"], dbf.load_dbf(io.BytesIO(buf.getvalue())))

    # ---- middle_dim for every configuration shape (budget.py:113-132) ------------------------
    shapes = [(4096, 4096), (11008, 4096), (4096, 11008), (5120, 5120), (13824, 5120), (5120, 13824),
              (8192, 8192), (1024, 8192), (28672, 8192), (8192, 28672), (4096, 14336), (8192, 28672)]
    bits = [1.0, 1.3, 1.5, 1.7, 2.0, 2.3]
    table = []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for n, m in shapes:
            for b in bits:
                table.append((n, m, b, dbf.middle_dim(n, m, b, 32)))
    g["middle_dim_table"] = np.array(table, dtype=np.float64)

    np.savez_compressed(OUT / "golden.npz", **g)
    print(f"wrote {OUT / 'golden.npz'} ({(OUT / 'golden.npz').stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
