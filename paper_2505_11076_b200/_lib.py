"""ctypes binding of the C ABI declared in ``include/dbf_b200.h``.

This is the only place the package touches native code.  There is no CPU fallback: if
``libdbf_b200.so`` is missing the import of this module raises, and every compute entry point
additionally requires a CUDA device (``require_cuda``).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("DBF_B200_LIB", _PKG / "libdbf_b200.so"))

# dtype codes (dbf_dtype)
F16, F32, F64, BF16 = 0, 1, 2, 3

# status codes (dbf_status)
OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_SHAPE = 2
ERR_WORKSPACE = 3
ERR_CUDA = 4
ERR_UNSUPPORTED = 5

_c = ctypes
_vp, _i64, _int, _sz = _c.c_void_p, _c.c_int64, _c.c_int, _c.c_size_t

# name -> (restype, argtypes); mirrors include/dbf_b200.h one to one
SIGNATURES: dict[str, tuple] = {
    "dbf_abi_version": (_int, []),
    "dbf_status_string": (_c.c_char_p, [_int]),
    "dbf_last_cuda_error": (_int, []),
    "dbf_last_cuda_error_string": (_c.c_char_p, []),
    "dbf_row_bytes": (_i64, [_i64]),
    "dbf_canonical_pitch_words": (_i64, [_i64]),
    "dbf_tiled_bytes": (_i64, [_i64, _i64]),
    "dbf_pack_signs": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _vp]),
    "dbf_unpack_signs": (_int, [_vp, _i64, _i64, _i64, _vp, _int, _i64, _vp]),
    "dbf_pack_sign_of": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _i64, _vp]),
    "dbf_repack_u8": (_int, [_vp, _i64, _i64, _vp, _i64, _vp]),
    "dbf_words_to_u8": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "dbf_tile_signs": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "dbf_transpose_signs": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp]),
    "dbf_sign_gemm_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp]),
    "dbf_forward_workspace_bytes": (_sz, [_i64, _i64, _i64, _i64]),
    "dbf_forward_batched_workspace_bytes": (_sz, [_i64, _i64, _i64, _i64]),
    "dbf_batched_frag_bytes": (_sz, [_i64, _i64]),
    "dbf_batched_debug_reset": (_int, [_int]),
    "dbf_batched_debug_trace": (_int, [_vp, _int]),
    "dbf_batched_quantize": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _int, _vp, _vp]),
    "dbf_forward_batched_frag_workspace_bytes": (_sz, [_i64, _i64, _i64, _i64]),
    "dbf_forward_batched_frag": (
        _int,
        [_vp, _vp, _vp, _vp, _int, _i64, _i64, _i64, _vp, _i64, _vp, _int, _i64, _vp, _int, _vp, _sz, _vp, _vp],
    ),
    "dbf_forward_batched": (
        _int,
        [_vp, _vp, _vp, _vp, _vp, _int, _i64, _i64, _i64, _vp, _int, _i64, _i64, _vp, _int, _i64, _vp, _sz, _vp, _vp],
    ),
    "dbf_sign_matvec": (_int, [_vp, _i64, _i64, _vp, _int, _i64, _i64, _vp, _int, _i64, _vp, _sz, _vp]),
    "dbf_forward": (
        _int,
        [_vp, _vp, _vp, _vp, _vp, _int, _i64, _i64, _i64, _vp, _int, _i64, _i64, _vp, _int, _i64, _vp, _sz, _vp],
    ),
    "dbf_forward_partial": (
        _int,
        [_vp, _vp, _vp, _vp, _int, _i64, _i64, _i64, _vp, _int, _i64, _i64, _vp, _vp, _sz, _vp],
    ),
    "dbf_finalize_partial": (_int, [_vp, _vp, _int, _i64, _i64, _vp, _int, _i64, _vp]),
    "dbf_allreduce_recv_bytes": (_sz, [_i64, _i64, _int]),
    "dbf_allreduce_flag_bytes": (_sz, [_i64, _int]),
    "dbf_forward_allreduce": (
        _int,
        [_vp, _vp, _vp, _vp, _vp, _int, _i64, _i64, _i64, _vp, _int, _i64, _i64, _vp, _int, _i64, _vp, _vp,
         _int, _int, _vp, _vp, _sz, _vp],
    ),
    "dbf_sign_matvec_xor": (_int, [_vp, _i64, _i64, _i64, _vp, _int, _vp, _vp]),
    "dbf_engine_smem_bytes": (_int, [_c.c_int32, _c.c_int32, _c.POINTER(_sz)]),
    "dbf_engine_occupancy": (_int, [_c.c_int32, _c.POINTER(_c.c_int32), _c.POINTER(_c.c_int32)]),
    "dbf_engine_build_runs": (_int, [_vp, _c.c_int32, _vp, _c.c_int32, _vp, _c.c_int32, _c.c_int32, _vp, _vp]),
    "dbf_engine_launch": (_int, [_vp, _vp]),
    "dbf_engine_run_limits": (_int, [_c.c_int32, _c.POINTER(_c.c_int32), _c.POINTER(_c.c_int64)]),
    "dbf_engine_run_limits_cols": (_int, [_c.c_int32, _c.c_int32, _c.POINTER(_c.c_int32), _c.POINTER(_c.c_int64)]),
    "dbf_engine_qscratch_bytes": (_sz, [_c.c_int32, _c.c_int32]),
    "dbf_pair_signs": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "dbf_prefill_debug_trace": (_int, [_vp, _int]),
    "dbf_prefill_ld": (_i64, [_i64]),
    "dbf_prefill_workspace_bytes": (_sz, [_i64, _i64]),
    "dbf_prefill_workspace_bytes_nkm": (_sz, [_i64, _i64, _i64, _i64]),
    "dbf_sign_gemm": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _i64, _vp]),
    "dbf_forward_prefill": (
        _int,
        [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _sz, _vp],
    ),
    "dbf_forward_prefill_ex": (
        _int,
        [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _sz, _int, _vp],
    ),
    "dbf_prefill_layer_path": (_int, [_i64, _i64, _i64, _i64]),
}


class DbfOverflowError(FloatingPointError):
    """The decode engine saw a non-finite input or overflowed fp16 (EngineProgram.check)."""


class DbfNativeError(RuntimeError):
    """A native call returned a non-OK dbf_status."""


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is not built; run `python paper_2505_11076_b200/_build.py` "
            "(nvcc, sm_100a).  There is no CPU fallback."
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    missing = [name for name in SIGNATURES if not hasattr(lib, name)]
    if missing:
        raise ImportError(f"{LIB_PATH} is stale (missing {missing}); rebuild with "
                          "`python paper_2505_11076_b200/_build.py`")
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def status_message(status: int) -> str:
    msg = lib.dbf_status_string(status).decode()
    if status == ERR_CUDA:
        msg += f" ({lib.dbf_last_cuda_error_string().decode()})"
    return msg


def check(status: int, what: str) -> None:
    if status != OK:
        raise DbfNativeError(f"{what} failed: {status_message(status)} (status {status})")


def require_cuda():
    """Raise unless a CUDA device is usable: the product path has no CPU fallback."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2505_11076_b200 runs the DBF forward on a B200 (sm_100a) GPU only; "
            "no CUDA device is available and there is no CPU fallback"
        )


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dtype) -> int:
    import torch

    table = {torch.float16: F16, torch.float32: F32, torch.float64: F64, torch.bfloat16: BF16}
    try:
        return table[dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {dtype}; expected float16/bfloat16/float32/float64") from None
