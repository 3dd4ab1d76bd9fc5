"""Host-side behaviour that needs no GPU: reference error conventions, DBF1 format, budget rule,
the engine planner and the k-shard bookkeeping.  The product never falls back to the CPU."""

import io

import numpy as np
import pytest

import paper_2505_11076_b200 as P
from paper_2505_11076_b200 import sharded
from paper_2505_11076_b200.engine import distribute, levels_of
from conftest import random_signs


def _bits(M):
    return np.packbits(M > 0, axis=1, bitorder="little")


def test_sign_matrix_validates_buffer_shape():  # test_bitcore.py:195-198
    with pytest.raises(ValueError, match="packed buffer"):
        P.SignMatrix(2, 10, np.zeros((2, 1), dtype=np.uint8))
    with pytest.raises(ValueError, match="at least 1x1"):
        P.SignMatrix(0, 4, np.zeros((0, 1), dtype=np.uint8))


def test_layer_shape_and_scale_validation(rng):  # test_bitcore.py:101-119
    S = lambda r, c: P.SignMatrix(r, c, _bits(random_signs(rng, r, c)))
    with pytest.raises(ValueError, match="mid"):
        P.DbfLayer(a=np.ones(3), A=S(3, 4), mid=np.ones(5), B=S(4, 2), b=np.ones(2))
    with pytest.raises(ValueError, match="B has"):
        P.DbfLayer(a=np.ones(3), A=S(3, 4), mid=np.ones(4), B=S(5, 2), b=np.ones(2))
    a = np.ones(3)
    a[1] = np.nan
    with pytest.raises(ValueError):
        P.DbfLayer(a=a, A=S(3, 2), mid=np.ones(2), B=S(2, 2), b=np.ones(2))


def test_forward_and_sign_matvec_argument_errors_come_first(rng):
    S = P.SignMatrix(3, 5, _bits(random_signs(rng, 3, 5)))
    with pytest.raises(ValueError, match="length"):
        P.sign_matvec(S, np.ones(6))
    layer = P.DbfLayer(a=np.ones(4), A=P.SignMatrix(4, 3, _bits(random_signs(rng, 4, 3))), mid=np.ones(3),
                       B=P.SignMatrix(3, 6, _bits(random_signs(rng, 3, 6))), b=np.ones(6))
    with pytest.raises(ValueError, match="columns"):
        P.forward(np.ones((2, 5)), layer)
    with pytest.raises(ValueError, match="2-D"):
        P.forward(np.ones(6), layer)
    with pytest.raises(ValueError, match="non-finite"):
        P.forward(np.full((1, 6), np.inf), layer)


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.pack(np.ones((2, 2)))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.forward(np.ones((1, 2)), P.DbfLayer(a=np.ones(2), A=P.SignMatrix(2, 2, np.ones((2, 1), np.uint8)),
                                              mid=np.ones(2), B=P.SignMatrix(2, 2, np.ones((2, 1), np.uint8)),
                                              b=np.ones(2)))


def test_dbf1_roundtrip_against_reference_bytes(golden):
    data = golden["dbf1_bytes"].tobytes()
    layer = P.load_dbf(io.BytesIO(data))
    assert (layer.n, layer.k, layer.m_dim) == (7, 5, 11)
    assert P.dumps_dbf(layer) == data  # byte-identical re-serialisation (bitcore.py:149-211)
    with pytest.raises(P.DbfFormatError, match="truncated"):
        P.load_dbf(io.BytesIO(data[:-3]))
    with pytest.raises(P.DbfFormatError, match="trailing"):
        P.load_dbf(io.BytesIO(data + b"\0"))
    with pytest.raises(P.DbfFormatError, match="magic"):
        P.load_dbf(io.BytesIO(b"NOPE" + data[4:]))


def test_middle_dim_matches_reference(golden):
    for n, m, b, k in golden["middle_dim_table"]:
        assert P.middle_dim(int(n), int(m), float(b)) == int(k)
    with pytest.warns(UserWarning):
        assert P.middle_dim(4, 4, 0.5) == 32


class _Op:
    def __init__(self, layer, src, dst):
        self.layer, self.src, self.dst = layer, src, dst


def test_engine_levels_follow_the_decoder_dataflow():
    # h=0 q=1 k=2 v=3 o=4 gate=5 up=6; two blocks
    ops = []
    for _ in range(2):
        ops += [_Op(0, 0, 1), _Op(0, 0, 2), _Op(0, 0, 3), _Op(0, 3, 4), _Op(0, 4, 5), _Op(0, 4, 6), _Op(0, 5, 0)]
    assert levels_of(ops, 0) == [0, 0, 0, 1, 2, 2, 3, 4, 4, 4, 5, 6, 6, 7]


@pytest.mark.parametrize("n,grid,rot", [(768, 148, 0), (100, 148, 37), (148, 148, 5), (1376, 132, 99)])
def test_engine_distribution_is_balanced_and_complete(n, grid, rot):
    units = [(0, i) for i in range(n)]
    per = distribute(units, grid, rot)
    flat = sorted(u for lst in per for u in lst)
    assert flat == units
    sizes = [len(x) for x in per]
    assert max(sizes) - min(sizes) <= 1
    for lst in per:  # each CTA's share is a contiguous run of row blocks
        rbs = [u[1] for u in lst]
        assert rbs == list(range(rbs[0], rbs[0] + len(rbs))) if rbs else True


@pytest.mark.parametrize("k,world", [(12736, 4), (12736, 8), (1792, 8), (4096, 2), (100, 2), (5952, 3)])
def test_shard_bounds_are_word_aligned_and_cover_k(k, world):
    b = sharded.shard_bounds(k, world)
    assert b[0][0] == 0 and b[-1][1] == k
    for (a0, a1), (c0, c1) in zip(b, b[1:]):
        assert a1 == c0
    assert all(k0 % 32 == 0 for k0, _ in b)
    sizes = [k1 - k0 for k0, k1 in b]
    assert max(sizes) - min(sizes) <= 32
    if (k, world) == (12736, 4):
        assert sizes == [3200, 3200, 3168, 3168] or max(sizes) - min(sizes) <= 32


def test_slice_columns_matches_numpy(rng):
    M = random_signs(rng, 9, 300)
    bits = _bits(M)
    for c0, c1 in [(0, 32), (32, 300), (64, 100), (296, 300), (0, 300)]:
        assert np.array_equal(sharded.slice_columns(bits, 300, c0, c1), _bits(M[:, c0:c1]))


@pytest.mark.parametrize("grid,rot", [(148, 0), (148, 77), (64, 3), (7, 2)])
def test_multi_segment_stage_gives_each_cta_one_segment(grid, rot):
    # q/k/v of a 7B block: three segments of 256 units, equal bytes
    units = [(s, i) for s in range(3) for i in range(256)]
    per = distribute(units, grid, rot, {0: 8192, 1: 8192, 2: 8192})
    assert sorted(u for lst in per for u in lst) == sorted(units)
    for lst in per:
        assert len({u[0] for u in lst}) <= 1  # never two segments on one CTA
        rbs = [u[1] for u in lst]
        assert rbs == list(range(rbs[0], rbs[0] + len(rbs))) if rbs else True
    sizes = [len(x) for x in per]
    assert max(sizes) <= -(-256 // (grid // 3))  # each segment spread over its share of the CTAs
