"""Host-side arithmetic of the prefill path (no GPU): the paired layout and the one-shift
sign expansion the tcgen05 kernel applies, restated in numpy and checked against the
reference's packing (bitcore.py:7-9, LSB-first, bit 1 <=> +1)."""

import numpy as np

from paper_2505_11076_b200 import _lib
from conftest import random_signs


def pair_words(words):
    """numpy model of dbf_pair_signs (csrc/pack.cu)."""
    out = np.zeros_like(words)
    for q in range(16):
        out |= ((words >> (2 * q)) & 1) << q
        out |= ((words >> (2 * q + 1)) & 1) << (16 + q)
    return out


def expand_word(w, ks):
    """numpy model of prefill.cu expand_word: 16 words of fp16 pairs +-ks from one paired word."""
    nw = (~w) & 0xFFFFFFFF
    return np.array([(((nw << (15 - q)) & 0xFFFFFFFF) & 0x80008000) ^ ks[q] for q in range(16)], dtype=np.uint32)


def test_expansion_reproduces_signs_times_scale(rng):
    rows, cols = 5, 64
    D = random_signs(rng, rows, cols)
    bits = np.packbits(D > 0, axis=1, bitorder="little")
    words = np.ascontiguousarray(bits).view("<u4")
    paired = pair_words(words.astype(np.uint64)).astype(np.uint32)
    scale = rng.uniform(0.5, 1.5, cols).astype(np.float16)
    ks_all = scale.view(np.uint16).astype(np.uint32)
    for r in range(rows):
        for j in range(cols // 32):
            ks = ks_all[32 * j:32 * j + 32:2] | (ks_all[32 * j + 1:32 * j + 32:2] << 16)
            v = expand_word(int(paired[r, j]), ks)
            halves = v.view(np.uint16).view(np.float16).astype(np.float64)  # little-endian: col 2q, 2q+1
            np.testing.assert_array_equal(halves, D[r, 32 * j:32 * j + 32] * scale[32 * j:32 * j + 32])


def test_unit_scale_expansion_is_plus_minus_one(rng):
    w = int(rng.integers(0, 2**32))
    v = expand_word(w, [0x3C003C00] * 16).view(np.uint16).view(np.float16)
    cols = np.array([(w >> (q if c % 2 == 0 else 16 + q)) & 1 for q in range(16) for c in (0, 1)])
    np.testing.assert_array_equal(v.astype(np.float64), np.where(cols == 1, 1.0, -1.0))


def test_prefill_workspace_queries():
    L = _lib.lib
    assert L.dbf_prefill_ld(1) == 64 and L.dbf_prefill_ld(64) == 64 and L.dbf_prefill_ld(2976) == 3008
    assert L.dbf_prefill_workspace_bytes(2976, 2048) == 2048 * 3008 * 2
    assert L.dbf_forward_prefill(None, 4, None, 4, None, None, None, 1, 1, 1, None, 1, 1, None, 1, None, 0, None) \
        == _lib.ERR_INVALID_ARGUMENT
    assert L.dbf_pair_signs(None, 1, 4, None, None) == _lib.ERR_INVALID_ARGUMENT
