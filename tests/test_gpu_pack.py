"""GPU pack/unpack/repack parity: bit-exact against the reference's own bytes (golden.npz)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2505_11076_b200 as P  # noqa: E402
from paper_2505_11076_b200 import _lib  # noqa: E402


def test_pack_bytes_equal_reference(golden):
    for i in range(int(golden["pack_count"])):
        dense = golden[f"pack{i}_dense"].astype(np.float64)
        s = P.pack(dense)
        assert s.bits.shape == golden[f"pack{i}_bits"].shape
        assert np.array_equal(s.bits, golden[f"pack{i}_bits"]), i


def test_pack_from_fp16_and_fp32_device_tensors(golden):
    import torch

    for i in range(0, int(golden["pack_count"]), 5):
        dense = golden[f"pack{i}_dense"]
        for dt in (torch.float16, torch.float32, torch.bfloat16):
            t = torch.from_numpy(dense.astype(np.float32)).to("cuda", dt)
            ds = P.DeviceSignMatrix.pack(t)
            assert np.array_equal(ds.to_host().bits, golden[f"pack{i}_bits"])


def test_unpack_equals_reference(golden):
    for i in range(int(golden["pack_count"])):
        dense = golden[f"pack{i}_dense"].astype(np.float64)
        s = P.SignMatrix(dense.shape[0], dense.shape[1], golden[f"pack{i}_bits"].copy())
        assert np.array_equal(P.unpack(s), dense)


def test_pack_rejects_first_offender(golden):
    shapes = [(3, 4), (2, 2), (4, 9), (5, 5)]
    vals = [0.5, 0.0, np.nan, -2.0]
    for shape, pos, val, msg in zip(shapes, golden["packbad_pos"], vals, golden["packbad_msgs"]):
        M = np.ones(shape)
        M[tuple(pos)] = val
        if val != 0.0:
            M[-1, -1] = 0.0
        with pytest.raises(ValueError) as e:
            P.pack(M)
        assert str(e.value) == str(msg)  # identical message, incl. the value repr


def test_pack_rejects_zero_and_matches_index_regex():
    M = np.ones((3, 4))
    M[1, 2] = 0.5
    with pytest.raises(ValueError, match=r"\(1, 2\)"):  # test_bitcore.py:40-44
        P.pack(M)
    with pytest.raises(ValueError):
        P.pack(np.zeros((2, 2)))


def test_roundtrip_property_random(rng):
    for _ in range(200):  # test_acceptance.py:241-245 style
        rows, cols = int(rng.integers(1, 25)), int(rng.integers(1, 300))
        M = rng.integers(0, 2, size=(rows, cols)).astype(np.float64) * 2 - 1
        assert np.array_equal(P.unpack(P.pack(M)), M)


def test_large_pack_matches_numpy_packbits(rng):
    M = rng.integers(0, 2, size=(1000, 4100)).astype(np.float64) * 2 - 1
    bits = np.packbits((M > 0).astype(np.uint8), axis=1, bitorder="little")
    assert np.array_equal(P.pack(M).bits, bits)


def test_repack_clears_padding_bits(rng):
    M = rng.integers(0, 2, size=(6, 13)).astype(np.float64) * 2 - 1
    s = P.pack(M)
    flipped = s.bits.copy()
    flipped[:, -1] ^= 0b11100000  # test_kernel.py:35-45: touch only padding bits
    ds = P.DeviceSignMatrix.from_host(P.SignMatrix(6, 13, flipped))
    assert np.array_equal(ds.to_host().bits, s.bits)


def test_canonical_words_are_reference_bytes_little_endian(rng):
    M = rng.integers(0, 2, size=(9, 200)).astype(np.float64) * 2 - 1
    s = P.pack(M)
    ds = P.DeviceSignMatrix.from_host(s)
    words = ds.words.cpu().numpy().view(np.uint8)[:, : s.bits.shape[1]]
    assert np.array_equal(words, s.bits)
    assert _lib.lib.dbf_canonical_pitch_words(200) == 8
