"""The DBF forward on the GPU: drop-in ``forward`` / ``sign_matvec`` / ``bench_forward``.

Restates the public surface of /root/reference/pkg/src/dbf/kernel.py:24-133.  Host (numpy)
inputs keep the reference contract -- float64 in, float64 out, same ``ValueError`` messages --
and run through the C ABI (``dbf_forward`` / ``dbf_sign_matvec``) on device copies.  CUDA tensor
inputs stay on the device (the fast path used by the decode engine and the benchmarks).

Numerics: every input row is quantized once to a 22-bit fixed-point grid relative
to its max |value|; the sign products are then exact integer sums on the int8 tensor cores.  The
result is bitwise reproducible (kernel.py:26-28) and agrees with the float64 reference to ~1e-7
relative, well inside the reference's own 1e-5 / 1e-4 tolerances (test_kernel.py:26, 80).
"""

from __future__ import annotations

import ctypes
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bitcore import SignMatrix
from .device import DeviceLayer, DeviceSignMatrix
from .validation import as_matrix, as_vector

# ---------------------------------------------------------------------------------------------
# workspace + device-object caches
# ---------------------------------------------------------------------------------------------
_workspaces: dict = {}


def _workspace(nbytes: int, device):
    import torch

    key = (str(device), torch.cuda.current_stream(device).cuda_stream)
    buf = _workspaces.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _workspaces[key] = buf
    return buf


_device_cache: dict[int, object] = {}


def _cached(obj, build):
    """Device image of an immutable host object, cached by identity until it is collected."""
    key = id(obj)
    hit = _device_cache.get(key)
    if hit is not None and hit[0]() is obj:
        return hit[1]
    dev = build()
    try:
        ref = weakref.ref(obj, lambda _r, k=key: _device_cache.pop(k, None))
    except TypeError:
        return dev
    _device_cache[key] = (ref, dev)
    return dev


def as_device_layer(layer, scale_dtype=None) -> DeviceLayer:
    import torch

    if isinstance(layer, DeviceLayer):
        return layer
    sd = scale_dtype or torch.float64
    return _cached(layer, lambda: DeviceLayer.from_host(layer, scale_dtype=sd))


def as_device_signs(s) -> DeviceSignMatrix:
    if isinstance(s, DeviceSignMatrix):
        return s
    return _cached(s, lambda: DeviceSignMatrix.from_host(s))


# ---------------------------------------------------------------------------------------------
# device fast path
# ---------------------------------------------------------------------------------------------
PREFILL_MIN_TOKENS = 64


def _prefill_eligible(X2, layer: DeviceLayer, out_dtype) -> bool:
    import torch

    return (
        X2.shape[0] >= PREFILL_MIN_TOKENS
        and X2.dtype == torch.float16
        and out_dtype == torch.float16
        and layer.scale_dtype == torch.float16
        and layer.A.words is not None
        and layer.B.words is not None
    )


PREFILL_PATHS = {"auto": 0, "two_launches": 1, "one_launch": 2}


def forward_prefill(X, layer: DeviceLayer, out=None, path: str = "auto"):
    """Y = forward(X, layer) for a token batch on the tcgen05 tensor cores (prefill path).

    X: CUDA fp16 tensor tokens x m; layer: fp16 scales with canonical words kept.  The two sign
    GEMMs run with fp32 accumulation in tensor memory and an fp16 intermediate t.
    path: "auto" (dbf_prefill_layer_path), "two_launches" (one per-tile launch per GEMM) or
    "one_launch" (both GEMMs in one persistent launch, T > 256); all give the same bits."""
    import torch

    if X.ndim != 2:
        raise ValueError(f"X must be 2-D, got ndim={X.ndim}")
    if X.shape[1] != layer.m_dim:
        raise ValueError(f"X has {X.shape[1]} columns, expected {layer.m_dim}")
    if X.dtype != torch.float16 or layer.scale_dtype != torch.float16:
        raise ValueError("the prefill path computes in fp16: X and the layer scales must be float16")
    T, m = X.shape
    if X.stride(1) != 1 or X.stride(0) % 8 or X.data_ptr() % 16:
        # TMA needs a 16-byte aligned base and a row pitch that is a multiple of 16 bytes
        ld = (m + 7) // 8 * 8
        Xp = torch.empty((T, ld), dtype=X.dtype, device=X.device)
        Xp[:, :m] = X
        X = Xp[:, :m]
    Y = out if out is not None else torch.empty((T, layer.n), dtype=torch.float16, device=X.device)
    A, B = layer.A.paired, layer.B.paired
    name = "dbf_forward_prefill_ex"
    if path not in PREFILL_PATHS:
        raise ValueError(f"path must be one of {sorted(PREFILL_PATHS)}, got {path!r}")
    # room for the split-K partials of small token counts / the one-launch kernel's tile counters
    ws_bytes = _lib.lib.dbf_prefill_workspace_bytes_nkm(layer.n, layer.k, layer.m_dim, T)
    ws = _workspace(ws_bytes, X.device)
    _lib.check(
        getattr(_lib.lib, name)(
            A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1],
            layer.a.data_ptr(), layer.mid.data_ptr(), layer.b.data_ptr(), layer.n, layer.k, layer.m_dim,
            X.data_ptr(), T, X.stride(0), Y.data_ptr(), Y.stride(0), ws.data_ptr(), ws.numel(),
            PREFILL_PATHS[path], _lib.stream_ptr(),
        ),
        name,
    )
    return Y


BATCHED_MAX_TOKENS = 32


def forward_engine(X, layer: DeviceLayer, out=None, out_dtype=None):
    """Y = forward(X, layer) for 1-4 fp16 / fp32 token rows through the persistent decode engine as
    a one-layer program: ONE launch runs GEMV1, the LL handoff of t and GEMV2 (forward_device takes
    two GEMV launches).  Engine numerics: a 13-bit grid per 256-column input chunk,
    t rounded to fp16 -- within the fp16 tolerance of the oracle, not bitwise forward_device.  The
    program is built once per (batch, input dtype, output dtype) and cached on the layer; each call
    then reads X and writes Y through the launch-time I/O overrides (dbf_engine_program
    x_override / y_override) and costs one kernel launch."""
    import torch

    from .engine import EngineProgram
    from .plan import DecodePlan, PlanOp

    squeeze = X.ndim == 1
    X2 = (X.unsqueeze(0) if squeeze else X).contiguous()
    if X2.ndim != 2 or X2.shape[1] != layer.m_dim:
        raise ValueError(f"X must be (batch, {layer.m_dim}), got {tuple(X.shape)}")
    batch = X2.shape[0]
    if not 1 <= batch <= 4 or X2.dtype not in (torch.float16, torch.float32):
        raise ValueError("forward_engine runs 1..4 fp16 / fp32 token rows (forward_device / forward_batched for others)")
    odt = out.dtype if out is not None else (out_dtype or X2.dtype)
    key = (batch, X2.dtype, odt, X2.device)
    progs = layer.__dict__.setdefault("_engine_progs", {})
    if key not in progs:
        bufs = [torch.zeros((batch, layer.m_dim), dtype=X2.dtype, device=X2.device),
                torch.zeros((batch, layer.n), dtype=odt, device=X2.device)]
        plan = DecodePlan([layer], [PlanOp(0, 0, 1, "forward")], bufs, input_buffer=0, output_buffer=1)
        progs[key] = EngineProgram(plan)
    Y = out if out is not None else torch.empty((batch, layer.n), dtype=odt, device=X2.device)
    progs[key].launch_io(X2, Y)
    return Y[0] if squeeze else Y


def forward_batched(X, layer: DeviceLayer, out=None, status=None):
    """Y = forward(X, layer) (/root/reference/pkg/src/dbf/kernel.py:48-62) for a CUDA batch of
    1-32 token rows with ONE pass over each sign matrix for all tokens (dbf_forward_batched,
    csrc/batched.cu): every extracted sign fragment feeds one int8 IMMA per group of 4 tokens.
    Numerics are the decode engine's (13-bit grid per token and 256-column chunk, exact chunk sums,
    fp32 accumulation and intermediate); ``status`` (a 1-element int32 CUDA tensor, optional) gets
    bit 1 for a non-finite output and bit 2 for an fp16 overflow."""
    import torch

    if X.ndim != 2:
        raise ValueError(f"X must be 2-D, got ndim={X.ndim}")
    if X.shape[1] != layer.m_dim:
        raise ValueError(f"X has {X.shape[1]} columns, expected {layer.m_dim}")
    batch = X.shape[0]
    if not 1 <= batch <= BATCHED_MAX_TOKENS:
        raise ValueError(f"forward_batched takes 1-{BATCHED_MAX_TOKENS} token rows, got {batch}")
    if X.stride(1) != 1:
        X = X.contiguous()
    Y = out if out is not None else torch.empty((batch, layer.n), dtype=X.dtype, device=X.device)
    if Y.stride(1) != 1:
        raise ValueError("out must have unit column stride")
    ws_bytes = _lib.lib.dbf_forward_batched_workspace_bytes(layer.n, layer.k, layer.m_dim, batch)
    ws = _workspace(ws_bytes, X.device)
    _lib.check(
        _lib.lib.dbf_forward_batched(
            layer.A.tiled.data_ptr(), layer.B.tiled.data_ptr(),
            layer.a.data_ptr(), layer.mid.data_ptr(), layer.b.data_ptr(), _lib.dtype_code(layer.a.dtype),
            layer.n, layer.k, layer.m_dim,
            X.data_ptr(), _lib.dtype_code(X.dtype), batch, X.stride(0),
            Y.data_ptr(), _lib.dtype_code(Y.dtype), Y.stride(0),
            ws.data_ptr(), ws.numel(), status.data_ptr() if status is not None else None, _lib.stream_ptr(),
        ),
        "dbf_forward_batched",
    )
    return Y


class _BatchedConsumer(ctypes.Structure):
    """dbf_batched_consumer (include/dbf_b200.h)."""
    _fields_ = [("b", ctypes.c_void_p), ("frag", ctypes.c_void_p)]


def batched_frag(cols: int, batch: int, device):
    """A fragment buffer: one layer's first-GEMV input (cols columns, batch tokens) as quantized
    B fragments (dbf_batched_frag_bytes)."""
    import torch

    return torch.empty(int(_lib.lib.dbf_batched_frag_bytes(cols, batch)), dtype=torch.uint8, device=device)


def batched_quantize(X, layer: DeviceLayer, frag):
    """X (batch x m) times the layer's input scale b -> its first-GEMV fragments (dbf_batched_quantize)."""
    _lib.check(
        _lib.lib.dbf_batched_quantize(X.data_ptr(), _lib.dtype_code(X.dtype), X.stride(0), X.shape[0], layer.m_dim,
                                      layer.b.data_ptr(), _lib.dtype_code(layer.b.dtype), frag.data_ptr(),
                                      _lib.stream_ptr()),
        "dbf_batched_quantize",
    )


def forward_batched_frag(frag, layer: DeviceLayer, batch: int, out, consumers=(), status=None):
    """forward_batched from a pre-quantized input (``frag``, from batched_quantize or a previous
    layer's finalize) into ``out`` (batch x n); ``consumers`` = [(layer_c, frag_c), ...] (<= 4):
    layers reading ``out`` next, whose fragments this call's finalize writes (dbf_forward_batched_frag)."""
    if len(consumers) > 4:
        raise ValueError("at most 4 consumers per layer")
    arr = (_BatchedConsumer * max(1, len(consumers)))()
    for i, (lc, fc) in enumerate(consumers):
        arr[i].b = lc.b.data_ptr()
        arr[i].frag = fc.data_ptr()
    ws = _workspace(_lib.lib.dbf_forward_batched_frag_workspace_bytes(layer.n, layer.k, layer.m_dim, batch),
                    out.device)
    _lib.check(
        _lib.lib.dbf_forward_batched_frag(
            layer.A.tiled.data_ptr(), layer.B.tiled.data_ptr(), layer.a.data_ptr(), layer.mid.data_ptr(),
            _lib.dtype_code(layer.a.dtype), layer.n, layer.k, layer.m_dim, frag.data_ptr(), batch,
            out.data_ptr(), _lib.dtype_code(out.dtype), out.stride(0), ctypes.cast(arr, ctypes.c_void_p),
            len(consumers), ws.data_ptr(), ws.numel(), status.data_ptr() if status is not None else None,
            _lib.stream_ptr(),
        ),
        "dbf_forward_batched_frag",
    )
    return out


def forward_device(X, layer: DeviceLayer, out=None, out_dtype=None):
    """Y = forward(X, layer) for a CUDA tensor X (batch x m or m); returns a CUDA tensor.

    fp16 batches of >= PREFILL_MIN_TOKENS tokens on an fp16 layer run the tcgen05 prefill path
    (forward_prefill); everything else -- decode batches, fp32/fp64 parity inputs -- runs the
    exact-integer tensor-core GEMV (dbf_forward)."""
    import torch

    squeeze = X.ndim == 1
    X2 = X.unsqueeze(0) if squeeze else X
    if X2.ndim != 2:
        raise ValueError(f"X must be 2-D, got ndim={X.ndim}")
    if X2.shape[1] != layer.m_dim:
        raise ValueError(f"X has {X2.shape[1]} columns, expected {layer.m_dim}")
    if X2.stride(1) != 1:
        X2 = X2.contiguous()
    batch = X2.shape[0]
    out_dtype = out_dtype or X2.dtype
    if _prefill_eligible(X2, layer, out_dtype) and (out is None or (out.stride(1) == 1 and out.dtype == torch.float16)):
        return forward_prefill(X2, layer, out=out)
    Y = out if out is not None else torch.empty((batch, layer.n), dtype=out_dtype, device=X2.device)
    ws_bytes = _lib.lib.dbf_forward_workspace_bytes(layer.n, layer.k, layer.m_dim, batch)
    ws = _workspace(ws_bytes, X2.device)
    _lib.check(
        _lib.lib.dbf_forward(
            layer.A.tiled.data_ptr(), layer.B.tiled.data_ptr(),
            layer.a.data_ptr(), layer.mid.data_ptr(), layer.b.data_ptr(), _lib.dtype_code(layer.a.dtype),
            layer.n, layer.k, layer.m_dim,
            X2.data_ptr(), _lib.dtype_code(X2.dtype), batch, X2.stride(0),
            Y.data_ptr(), _lib.dtype_code(Y.dtype), Y.stride(0),
            ws.data_ptr(), ws.numel(), _lib.stream_ptr(),
        ),
        "dbf_forward",
    )
    return Y[0] if squeeze else Y


def sign_matvec_device(s: DeviceSignMatrix, x, out_dtype=None):
    """S @ x for a CUDA tensor x (cols or batch x cols); returns a CUDA tensor."""
    import torch

    squeeze = x.ndim == 1
    X2 = x.unsqueeze(0) if squeeze else x
    if X2.shape[-1] != s.cols:
        raise ValueError(f"x has length {X2.shape[-1]}, expected {s.cols}")
    if X2.stride(1) != 1:
        X2 = X2.contiguous()
    batch = X2.shape[0]
    Y = torch.empty((batch, s.rows), dtype=out_dtype or X2.dtype, device=X2.device)
    _lib.check(
        _lib.lib.dbf_sign_matvec(
            s.tiled.data_ptr(), s.rows, s.cols, X2.data_ptr(), _lib.dtype_code(X2.dtype), batch, X2.stride(0),
            Y.data_ptr(), _lib.dtype_code(Y.dtype), Y.stride(0), None, 0, _lib.stream_ptr(),
        ),
        "dbf_sign_matvec",
    )
    return Y[0] if squeeze else Y


def _is_cuda_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


# ---------------------------------------------------------------------------------------------
# reference-compatible surface (kernel.py:24-62)
# ---------------------------------------------------------------------------------------------
def sign_matvec(s, x):
    """kernel.py:24-45: ``s @ x`` for a packed sign matrix; float64 numpy in/out for host inputs."""
    if _is_cuda_tensor(x):
        return sign_matvec_device(as_device_signs(s), x)
    x = as_vector(x, "x")
    if x.size != s.cols:
        raise ValueError(f"x has length {x.size}, expected {s.cols}")
    _lib.require_cuda()
    import torch

    ds = as_device_signs(s)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return sign_matvec_device(ds, xd, out_dtype=torch.float64).cpu().numpy()


def forward(X, layer):
    """kernel.py:48-62: ``X @ W_hat^T`` staged as b, B, mid, A, a -- on the GPU."""
    if _is_cuda_tensor(X):
        return forward_device(X, as_device_layer(layer))
    X = as_matrix(X, "X")
    if X.shape[1] != layer.m_dim:
        raise ValueError(f"X has {X.shape[1]} columns, expected {layer.m_dim}")
    _lib.require_cuda()
    import torch

    dl = as_device_layer(layer)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    return forward_device(Xd, dl, out_dtype=torch.float64).cpu().numpy()


# ---------------------------------------------------------------------------------------------
# bench harness (kernel.py:65-133), timed with CUDA events instead of perf_counter
# ---------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class BenchRow:
    n: int
    m_dim: int
    bits: float
    k: int
    t_dense_us: float
    t_dbf_us: float
    ratio: float

    def csv(self) -> str:
        return (
            f"{self.n}x{self.m_dim},{self.bits:g},"
            f"{self.t_dense_us:.3f},{self.t_dbf_us:.3f},{self.ratio:.4f}"
        )


BENCH_CSV_HEADER = "shape,bits,t_dense_us,t_dbf_us,ratio"


def _median_us(fn, repeats: int) -> float:
    import torch

    fn()
    times = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(times))


def bench_forward(shapes, bits, repeats: int = 3, seed: int = 0) -> list[BenchRow]:
    """kernel.py:94-118 on the GPU: median time of a dense fp16 matvec (cuBLAS) vs the DBF
    forward (fp16 activations and scales), one row per (shape, bits).  Informational only."""
    import torch

    from .budget import middle_dim

    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")
    _lib.require_cuda()
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    rows = []
    for n, m in shapes:
        dense = torch.randn((n, m), generator=g, device="cuda", dtype=torch.float16)
        x = torch.randn((m,), generator=g, device="cuda", dtype=torch.float16)
        t_dense = _median_us(lambda: torch.mv(dense, x), repeats)
        for b in bits:
            raw = b * n * m / (n + m)
            k = middle_dim(n, m, b, 32) if raw >= 32 else max(1, int(raw))
            layer = random_device_layer(n, k, m, generator=g)
            xm = x.reshape(1, m)
            t_dbf = _median_us(lambda: forward_device(xm, layer), repeats)
            ratio = t_dbf / t_dense if t_dense > 0 else float("inf")
            rows.append(BenchRow(n, m, float(b), k, t_dense, t_dbf, ratio))
    return rows


def random_device_layer(n: int, k: int, m: int, generator=None, scale_dtype=None, device="cuda",
                        keep_words: bool = False) -> DeviceLayer:
    """Synthetic layer on the device: uniform signs, a = U(.5,1.5)/sqrt(k),
    mid = U(.5,1.5), b = U(.5,1.5)/sqrt(m), all rounded through the scale dtype."""
    import torch

    sd = scale_dtype or torch.float16

    def u(size, div):
        return ((torch.rand(size, generator=generator, device=device, dtype=torch.float64) + 0.5) / div).to(sd)

    A = DeviceSignMatrix.random(n, k, generator=generator, device=device, keep_words=keep_words)
    B = DeviceSignMatrix.random(k, m, generator=generator, device=device, keep_words=keep_words)
    return DeviceLayer(u(n, k**0.5), A, u(k, 1.0), B, u(m, m**0.5))
