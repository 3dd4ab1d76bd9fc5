"""B200-native Double Binary Factorization (DBF) forward -- drop-in for the reference ``dbf``
package's hot path (pack / unpack / sign_matvec / forward, /root/reference/pkg/src/dbf).

Everything computes on an sm_100a GPU through the C ABI in ``include/dbf_b200.h``
(``libdbf_b200.so``); importing this package fails if the library is not built, and compute
calls fail without a CUDA device -- there is no CPU fallback.
"""

from ._lib import DbfNativeError, DbfOverflowError
from .bitcore import (
    DbfFormatError,
    DbfLayer,
    SignMatrix,
    dumps_dbf,
    load_dbf,
    pack,
    pack_sign_of,
    reconstruct,
    row_bytes,
    save_dbf,
    transpose_signs,
    unpack,
)
from .budget import middle_dim, storage_bits
from .device import DeviceLayer, DeviceSignMatrix
from .staged import ChannelScores, channel_scores, refine_scales, staged_loss_grads
from .kernel import (
    BENCH_CSV_HEADER,
    BenchRow,
    bench_forward,
    forward,
    forward_device,
    forward_batched,
    forward_engine,
    forward_prefill,
    random_device_layer,
    sign_matvec,
    sign_matvec_device,
)

__version__ = "0.1.0"

__all__ = [
    "BENCH_CSV_HEADER",
    "BenchRow",
    "ChannelScores",
    "channel_scores",
    "refine_scales",
    "staged_loss_grads",
    "DbfFormatError",
    "DbfLayer",
    "DbfNativeError",
    "DbfOverflowError",
    "DeviceLayer",
    "DeviceSignMatrix",
    "SignMatrix",
    "bench_forward",
    "dumps_dbf",
    "forward",
    "forward_device",
    "forward_batched",
    "forward_engine",
    "forward_prefill",
    "load_dbf",
    "middle_dim",
    "pack",
    "pack_sign_of",
    "random_device_layer",
    "reconstruct",
    "row_bytes",
    "save_dbf",
    "sign_matvec",
    "sign_matvec_device",
    "storage_bits",
    "transpose_signs",
    "unpack",
]
