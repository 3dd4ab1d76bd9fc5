"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatements of the reference DBF hot path used to CHECK the product:
``dbf_oracle`` (numpy, bit-identical to the reference) and ``liboracle.so`` (plain C, built from
``dbf_oracle.c`` by ``build()``).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"


def build() -> Path:
    src = HERE / "dbf_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    return LIB


_lib = None


def clib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        P, I = ctypes.c_void_p, ctypes.c_int64
        L.dbf_oracle_pack.restype = I
        L.dbf_oracle_pack.argtypes = [P, I, I, P]
        L.dbf_oracle_unpack.restype = None
        L.dbf_oracle_unpack.argtypes = [P, I, I, P]
        L.dbf_oracle_sign_matvec.restype = None
        L.dbf_oracle_sign_matvec.argtypes = [P, I, I, P, P]
        L.dbf_oracle_forward.restype = None
        L.dbf_oracle_forward.argtypes = [P, I, P, P, P, P, P, I, I, I, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def c_pack(dense) -> tuple[np.ndarray | None, int]:
    d = np.ascontiguousarray(dense, dtype=np.float64)
    rows, cols = d.shape
    bits = np.zeros((rows, (cols + 7) // 8), dtype=np.uint8)
    bad = clib().dbf_oracle_pack(_p(d), rows, cols, _p(bits))
    return (None if bad >= 0 else bits), int(bad)


def c_unpack(bits, cols: int) -> np.ndarray:
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    out = np.empty((b.shape[0], cols))
    clib().dbf_oracle_unpack(_p(b), b.shape[0], cols, _p(out))
    return out


def c_sign_matvec(bits, cols: int, x) -> np.ndarray:
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    xv = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(b.shape[0])
    clib().dbf_oracle_sign_matvec(_p(b), b.shape[0], cols, _p(xv), _p(out))
    return out


def c_forward(X, a, A_bits, mid, B_bits, b) -> np.ndarray:
    X = np.ascontiguousarray(np.atleast_2d(X), dtype=np.float64)
    a, mid, b = (np.ascontiguousarray(v, dtype=np.float64) for v in (a, mid, b))
    A_bits = np.ascontiguousarray(A_bits, dtype=np.uint8)
    B_bits = np.ascontiguousarray(B_bits, dtype=np.uint8)
    n, k, m = len(a), len(mid), len(b)
    out = np.empty((X.shape[0], n))
    tmp = np.empty(max(m, k) + k + n)
    clib().dbf_oracle_forward(_p(X), X.shape[0], _p(a), _p(A_bits), _p(mid), _p(B_bits), _p(b), n, k, m, _p(out), _p(tmp))
    return out
