"""Device-resident DBF operands.

``DeviceSignMatrix`` keeps a sign matrix in HBM in the two layouts of include/dbf_b200.h:
the canonical uint32 words (the reference bytes viewed little-endian, 16-byte row pitch) and
the tiled decode layout consumed by the tensor-core GEMV.  ``DeviceLayer`` is the device image
of a reference ``DbfLayer`` (bitcore.py:94-131): tiled A and B plus the three scale vectors in
fp16 (performance path) or fp32/fp64 (parity path).  Device objects are immutable after upload
and may be shared by several streams, like the reference's read-only containers
(bitcore.py:57, 108-111).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .bitcore import SignMatrix, row_bytes


def _tile(words, rows: int, cols: int):
    import torch

    nbytes = _lib.lib.dbf_tiled_bytes(rows, cols)
    tiled = torch.empty(nbytes, dtype=torch.uint8, device=words.device)
    _lib.check(
        _lib.lib.dbf_tile_signs(words.data_ptr(), rows, cols, words.shape[1], tiled.data_ptr(), _lib.stream_ptr()),
        "dbf_tile_signs",
    )
    return tiled


class DeviceSignMatrix:
    """A rows x cols sign matrix resident on the GPU."""

    def __init__(self, rows: int, cols: int, words=None, tiled=None):
        if rows < 1 or cols < 1:
            raise ValueError(f"sign matrix must be at least 1x1, got {rows}x{cols}")
        if words is None and tiled is None:
            raise ValueError("DeviceSignMatrix needs canonical words or a tiled buffer")
        self.rows, self.cols = int(rows), int(cols)
        self.words = words
        self.tiled = tiled

    # -- construction ---------------------------------------------------------------------
    @classmethod
    def from_words(cls, words, rows: int, cols: int, tile: bool = True, keep_words: bool = True):
        """From canonical device words (int32/uint32 tensor rows x pitch, padding bits zero)."""
        tiled = _tile(words, rows, cols) if tile else None
        return cls(rows, cols, words if (keep_words or not tile) else None, tiled)

    @classmethod
    def from_host(cls, s, device=None, tile: bool = True, keep_words: bool = True):
        """Upload a reference-layout SignMatrix (ours or the reference package's)."""
        import torch

        _lib.require_cuda()
        rows, cols = int(s.rows), int(s.cols)
        bits = np.ascontiguousarray(np.asarray(s.bits, dtype=np.uint8))
        if bits.shape != (rows, row_bytes(cols)):
            raise ValueError(f"packed buffer must be uint8 with shape {(rows, row_bytes(cols))}, got {bits.shape}")
        dev = torch.device(device) if device is not None else torch.device("cuda")
        raw = torch.from_numpy(bits.copy()).to(dev)
        pitch = _lib.lib.dbf_canonical_pitch_words(cols)
        words = torch.empty((rows, pitch), dtype=torch.int32, device=dev)
        _lib.check(
            _lib.lib.dbf_repack_u8(raw.data_ptr(), rows, cols, words.data_ptr(), pitch, _lib.stream_ptr()),
            "dbf_repack_u8",
        )
        return cls.from_words(words, rows, cols, tile=tile, keep_words=keep_words)

    @classmethod
    def pack(cls, dense, tile: bool = True, keep_words: bool = True):
        """GPU pack of a dense +-1 matrix (host array or CUDA tensor) straight to the device."""
        from .bitcore import pack_words

        words, rows, cols = pack_words(dense)
        return cls.from_words(words, rows, cols, tile=tile, keep_words=keep_words)

    @classmethod
    def random(cls, rows: int, cols: int, generator=None, device="cuda", keep_words: bool = False):
        """Uniform random signs generated on the device (benchmarks; layout-valid padding)."""
        import torch

        pitch = _lib.lib.dbf_canonical_pitch_words(cols)
        words = torch.randint(-(2**31), 2**31 - 1, (rows, pitch), dtype=torch.int32, device=device, generator=generator)
        full = cols // 32
        if cols % 32:
            words[:, full] &= (1 << (cols % 32)) - 1
            full += 1
        if full < pitch:
            words[:, full:] = 0
        return cls.from_words(words, rows, cols, tile=True, keep_words=keep_words)

    # -- views ------------------------------------------------------------------------------
    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    def nbytes_logical(self) -> int:
        return self.rows * row_bytes(self.cols)

    def _need_words(self):
        if self.words is None:
            raise ValueError("this DeviceSignMatrix was built without canonical words (keep_words=False)")
        return self.words

    @property
    def paired(self):
        """The paired prefill layout (dbf_pair_signs), built once from the canonical words."""
        import torch

        if getattr(self, "_paired", None) is None:
            w = self._need_words()
            out = torch.empty_like(w)
            _lib.check(
                _lib.lib.dbf_pair_signs(w.data_ptr(), self.rows, w.shape[1], out.data_ptr(), _lib.stream_ptr()),
                "dbf_pair_signs",
            )
            self._paired = out
        return self._paired

    def transposed(self) -> "DeviceSignMatrix":
        """S^T as its own device sign matrix (canonical words + tiled), built once on the GPU."""
        import torch

        if getattr(self, "_transposed", None) is None:
            w = self._need_words()
            pitch = _lib.lib.dbf_canonical_pitch_words(self.rows)
            out = torch.empty((self.cols, pitch), dtype=torch.int32, device=w.device)
            _lib.check(
                _lib.lib.dbf_transpose_signs(w.data_ptr(), self.rows, self.cols, w.shape[1], out.data_ptr(), pitch,
                                             _lib.stream_ptr()),
                "dbf_transpose_signs",
            )
            self._transposed = DeviceSignMatrix.from_words(out, self.cols, self.rows, tile=True, keep_words=True)
        return self._transposed

    def to_host(self) -> SignMatrix:
        from .bitcore import words_to_bytes

        return SignMatrix(self.rows, self.cols, words_to_bytes(self._need_words(), self.rows, self.cols))

    def unpack(self, dtype=None):
        """+-1 dense tensor (bitcore.py:88-91) on the device."""
        import torch

        dtype = dtype or torch.float32
        w = self._need_words()
        out = torch.empty((self.rows, self.cols), dtype=dtype, device=w.device)
        _lib.check(
            _lib.lib.dbf_unpack_signs(
                w.data_ptr(), self.rows, self.cols, w.shape[1], out.data_ptr(), _lib.dtype_code(dtype),
                self.cols, _lib.stream_ptr(),
            ),
            "dbf_unpack_signs",
        )
        return out


class DeviceLayer:
    """Device image of a DbfLayer: y = a * (A . (mid * (B . (b * x))))."""

    def __init__(self, a, A: DeviceSignMatrix, mid, B: DeviceSignMatrix, b):
        if a.numel() != A.rows:
            raise ValueError(f"a has length {a.numel()}, expected {A.rows}")
        if mid.numel() != A.cols:
            raise ValueError(f"mid has length {mid.numel()}, expected {A.cols}")
        if B.rows != A.cols:
            raise ValueError(f"B has {B.rows} rows, expected {A.cols}")
        if b.numel() != B.cols:
            raise ValueError(f"b has length {b.numel()}, expected {B.cols}")
        if not (a.dtype == mid.dtype == b.dtype):
            raise ValueError("scale vectors must share one dtype")
        if A.tiled is None or B.tiled is None:
            raise ValueError("DeviceLayer needs tiled sign matrices")
        self.a, self.A, self.mid, self.B, self.b = a.contiguous(), A, mid.contiguous(), B, b.contiguous()

    @property
    def n(self) -> int:
        return self.A.rows

    @property
    def k(self) -> int:
        return self.A.cols

    @property
    def m_dim(self) -> int:
        return self.B.cols

    @property
    def scale_dtype(self):
        return self.a.dtype

    @classmethod
    def from_host(cls, layer, scale_dtype=None, device=None, keep_words: bool = True):
        """Upload a reference DbfLayer (ours or the reference package's)."""
        import torch

        _lib.require_cuda()
        scale_dtype = scale_dtype or torch.float32
        dev = torch.device(device) if device is not None else torch.device("cuda")

        def vec(v):
            return torch.as_tensor(np.array(v, dtype=np.float64)).to(device=dev, dtype=scale_dtype)

        A = DeviceSignMatrix.from_host(layer.A, dev, keep_words=keep_words)
        B = DeviceSignMatrix.from_host(layer.B, dev, keep_words=keep_words)
        return cls(vec(layer.a), A, vec(layer.mid), B, vec(layer.b))

    def bytes_logical(self, batch: int = 1, act_bytes: int = 2) -> int:
        """Algorithmic HBM bytes of one decode forward."""
        n, k, m = self.n, self.k, self.m_dim
        sb = self.a.element_size()
        return n * row_bytes(k) + k * row_bytes(m) + sb * (n + k + m) + act_bytes * batch * (m + n)

    def reconstruct(self, dtype=None):
        """Dense W = (a*A*mid) @ (B*b) on the device (bitcore.py:134-138)."""
        import torch

        dtype = dtype or torch.float32
        left = self.a.to(dtype)[:, None] * self.A.unpack(dtype) * self.mid.to(dtype)[None, :]
        right = self.B.unpack(dtype) * self.b.to(dtype)[None, :]
        return left @ right

    def forward(self, X, out_dtype=None):
        from .kernel import forward_device

        return forward_device(X, self, out_dtype=out_dtype)
