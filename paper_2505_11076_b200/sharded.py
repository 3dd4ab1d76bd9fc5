"""Middle-dimension (k) sharding of one DBF layer across the GPUs of a node.

    y = a * (A . (mid * (B . (b * x))))  =  a * sum_g  A[:, K_g] . (mid[K_g] * (B[K_g, :] . (b * x)))

Rank g owns rows K_g of B, columns K_g of A and mid[K_g]; x, b and a are replicated.  Each rank
computes its fp32 partial ``P_g = A_g . (mid_g * (B_g . (b * x)))`` with no communication
(``dbf_forward_partial``), one SUM all-reduce combines the partials over NVLink (NCCL through
``torch.distributed``), and ``y = a * P`` is applied after the reduce (``dbf_finalize_partial``).
``FusedAllReduce`` + ``DeviceShard.forward_allreduce`` fuse that exchange into GEMV2 instead
(``dbf_forward_allreduce``): partial row blocks are pushed into every peer's symmetric-memory
receive buffer from the kernel epilogue and combined per row block as soon as all ranks released it.

Shard boundaries are multiples of 32 columns so every shard of A is a word-aligned slice of the
packed rows (the reference's LSB-first layout, bitcore.py:7-9): k = 12736 over 4 ranks gives
3200/3200/3200/3136 (12736/4 = 3184 is not word-aligned).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .bitcore import SignMatrix, row_bytes


def shard_bounds(k: int, world: int, align: int = 32) -> list[tuple[int, int]]:
    """Contiguous [k0, k1) ranges covering 0..k, boundaries multiples of ``align``, sizes
    balanced to within one alignment block; trailing ranks may be empty if k is tiny."""
    if k < 1 or world < 1 or align < 1:
        raise ValueError("k, world and align must be >= 1")
    blocks = -(-k // align)
    bounds = []
    for r in range(world):
        b0 = (r * blocks) // world
        b1 = ((r + 1) * blocks) // world
        bounds.append((min(b0 * align, k), min(b1 * align, k)))
    return bounds


def slice_columns(bits: np.ndarray, cols: int, c0: int, c1: int) -> np.ndarray:
    """Reference row bytes of columns [c0, c1) (c0 a multiple of 8) of a packed sign matrix."""
    if c0 % 8:
        raise ValueError("column slices must start on a byte boundary")
    if not (0 <= c0 < c1 <= cols):
        raise ValueError(f"bad column range [{c0}, {c1}) for {cols} columns")
    out = np.ascontiguousarray(bits[:, c0 // 8 : c0 // 8 + row_bytes(c1 - c0)]).copy()
    tail = (c1 - c0) % 8
    if tail:
        out[:, -1] &= (1 << tail) - 1  # padding bits beyond c1 must be zero
    return out


@dataclass(frozen=True)
class LayerShard:
    """Host-side shard of a DbfLayer for rank `rank` of `world` (k range [k0, k1))."""

    rank: int
    world: int
    k0: int
    k1: int
    a: np.ndarray
    A: SignMatrix  # n x (k1 - k0)
    mid: np.ndarray  # (k1 - k0,)
    B: SignMatrix  # (k1 - k0) x m
    b: np.ndarray

    @property
    def n(self) -> int:
        return self.A.rows

    @property
    def k_shard(self) -> int:
        return self.k1 - self.k0

    @property
    def m_dim(self) -> int:
        return self.B.cols


def shard_layer(layer, rank: int, world: int, align: int = 32) -> LayerShard:
    """Cut the k-shard of `rank` out of a host DbfLayer (ours or the reference's)."""
    k = layer.A.cols
    k0, k1 = shard_bounds(k, world, align)[rank]
    if k1 <= k0:
        raise ValueError(f"rank {rank} has an empty shard of k={k} over {world} ranks")
    A_bits = slice_columns(np.asarray(layer.A.bits), k, k0, k1)
    B_bits = np.ascontiguousarray(np.asarray(layer.B.bits)[k0:k1]).copy()
    return LayerShard(
        rank, world, k0, k1,
        np.asarray(layer.a, dtype=np.float64),
        SignMatrix(layer.A.rows, k1 - k0, A_bits),
        np.asarray(layer.mid, dtype=np.float64)[k0:k1].copy(),
        SignMatrix(k1 - k0, layer.B.cols, B_bits),
        np.asarray(layer.b, dtype=np.float64),
    )


@dataclass(frozen=True)
class _LayerView:
    """The fields EngineProgram reads from a layer (a = None: no output scale)."""

    A: object
    B: object
    a: object
    mid: object
    b: object
    n: int
    k: int
    m_dim: int


@dataclass(frozen=True)
class _ShardShape:
    rank: int
    world: int
    k0: int
    k1: int
    n: int
    m_dim: int

    @property
    def k_shard(self) -> int:
        return self.k1 - self.k0


class DeviceShard:
    """Device image of a LayerShard (tiled A_g, B_g; scales in `scale_dtype`)."""

    def __init__(self, shard: LayerShard, scale_dtype=None, device=None):
        import torch

        from .device import DeviceSignMatrix

        sd = scale_dtype or torch.float32
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.shard = shard
        self.A = DeviceSignMatrix.from_host(shard.A, dev, keep_words=False)
        self.B = DeviceSignMatrix.from_host(shard.B, dev, keep_words=False)
        self.a = torch.as_tensor(np.array(shard.a)).to(dev, sd)
        self.mid = torch.as_tensor(np.array(shard.mid)).to(dev, sd)
        self.b = torch.as_tensor(np.array(shard.b)).to(dev, sd)

    @classmethod
    def from_device_layer(cls, layer, rank: int, world: int, k0: int = 0):
        """Wrap a DeviceLayer that already holds one rank's shard (A_g n x k_g, B_g k_g x m) --
        e.g. synthetic shards generated on each GPU for benchmarks."""
        self = cls.__new__(cls)
        self.shard = _ShardShape(rank, world, k0, k0 + layer.k, layer.n, layer.B.cols)
        self.A, self.B, self.a, self.mid, self.b = layer.A, layer.B, layer.a, layer.mid, layer.b
        return self

    def partial(self, X):
        """fp32 partial P_g (batch x n) for a CUDA tensor X (batch x m)."""
        import torch

        from . import _lib
        from .kernel import _workspace

        sh = self.shard
        X2 = X if X.ndim == 2 else X.unsqueeze(0)
        X2 = X2.contiguous()
        P = torch.empty((X2.shape[0], sh.n), dtype=torch.float32, device=X2.device)
        ws_bytes = _lib.lib.dbf_forward_workspace_bytes(sh.n, sh.k_shard, sh.m_dim, X2.shape[0])
        ws = _workspace(ws_bytes, X2.device)
        _lib.check(
            _lib.lib.dbf_forward_partial(
                self.A.tiled.data_ptr(), self.B.tiled.data_ptr(), self.mid.data_ptr(), self.b.data_ptr(),
                _lib.dtype_code(self.a.dtype), sh.n, sh.k_shard, sh.m_dim, X2.data_ptr(), _lib.dtype_code(X2.dtype),
                X2.shape[0], X2.stride(0), P.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(),
            ),
            "dbf_forward_partial",
        )
        return P

    def partial_engine(self, X):
        """The same fp32 partial through the persistent decode engine (batch <= 4, fp16 / fp32
        input): one cooperative launch runs GEMV1 and GEMV2 with the LL handoff of t between them
        (engine numerics: 13-bit input grid per 256-column chunk, t rounded to fp16; the partial
        itself is not rounded).  The program is built once per (batch, dtype) and then reads X and
        writes P through the launch-time I/O overrides, so calls cost one engine launch."""
        import torch

        X2 = X if X.ndim == 2 else X.unsqueeze(0)
        X2 = X2.contiguous()
        prog = self._engine_program(X2)
        P = torch.empty((X2.shape[0], self.shard.n), dtype=torch.float32, device=X2.device)
        prog.launch_io(X2, P)
        return P

    def _engine_program(self, X2):
        import torch

        from .engine import EngineProgram
        from .plan import DecodePlan, PlanOp

        batch = X2.shape[0]
        if not 1 <= batch <= 4 or X2.dtype not in (torch.float16, torch.float32):
            raise ValueError("partial_engine runs 1..4 fp16/fp32 tokens (use partial for others)")
        key = (batch, X2.dtype, X2.device)
        progs = self.__dict__.setdefault("_engine_progs", {})
        if key not in progs:
            sh = self.shard
            view = _LayerView(self.A, self.B, None, self.mid, self.b, sh.n, sh.k_shard, sh.m_dim)
            bufs = [torch.zeros((batch, sh.m_dim), dtype=X2.dtype, device=X2.device),
                    torch.zeros((batch, sh.n), dtype=torch.float32, device=X2.device)]
            plan = DecodePlan([view], [PlanOp(0, 0, 1, "partial")], bufs, input_buffer=0, output_buffer=1)
            progs[key] = (EngineProgram(plan), plan)
        return progs[key][0]

    def forward_allreduce_engine(self, X, peer_recv, peer_flags, epoch_counter, out_dtype=None):
        """The layer through the decode engine with the one-shot all-reduce fused into its last
        stage (one launch per call): GEMV1 -> LL t -> GEMV2, whose finalize pushes the fp32 partial
        rows into every rank's receive buffer, raises the row blocks' flags, waits for every rank's
        and writes y = a * sum over ranks.  Same buffers, flags and call counter as
        ``forward_allreduce`` (``FusedAllReduce``); batch 1..4, fp16 / fp32 X."""
        import torch

        sh = self.shard
        X2 = X if X.ndim == 2 else X.unsqueeze(0)
        X2 = X2.contiguous()
        prog = self._engine_program(X2)
        Y = torch.empty((X2.shape[0], sh.n), dtype=out_dtype or X2.dtype, device=X2.device)
        prog.launch_allreduce(X2, Y, peer_recv, peer_flags, epoch_counter, sh.world, sh.rank, self.a)
        return Y

    def finalize(self, P, out_dtype=None):
        import torch

        from . import _lib

        Y = torch.empty(P.shape, dtype=out_dtype or torch.float16, device=P.device)
        _lib.check(
            _lib.lib.dbf_finalize_partial(
                P.data_ptr(), self.a.data_ptr(), _lib.dtype_code(self.a.dtype), P.shape[1], P.shape[0],
                Y.data_ptr(), _lib.dtype_code(Y.dtype), Y.stride(0), _lib.stream_ptr(),
            ),
            "dbf_finalize_partial",
        )
        return Y

    def forward(self, X, group=None, out_dtype=None, engine: bool = False):
        """y = a * all_reduce_sum(P_g): one NCCL SUM all-reduce of n x batch fp32 values
        (engine=True computes P_g with partial_engine)."""
        import torch.distributed as dist

        P = self.partial_engine(X) if engine else self.partial(X)
        if dist.is_initialized():  # a single process without a group has nothing to reduce
            dist.all_reduce(P, op=dist.ReduceOp.SUM, group=group)
        return self.finalize(P, out_dtype=out_dtype or X.dtype)


    def forward_allreduce(self, X, peer_recv, peer_flags, epoch_counter, out_dtype=None):
        """dbf_forward_allreduce: the layer with its all-reduce fused into GEMV2's epilogue.

        ``peer_recv`` / ``peer_flags``: int64 CUDA tensors holding every rank's receive-buffer and
        flag-array device addresses (``FusedAllReduce`` builds them from symmetric memory);
        ``epoch_counter``: a 1-element int32 CUDA tensor the call advances on the device."""
        import torch

        from . import _lib
        from .kernel import _workspace

        sh = self.shard
        X2 = X if X.ndim == 2 else X.unsqueeze(0)
        X2 = X2.contiguous()
        Y = torch.empty((X2.shape[0], sh.n), dtype=out_dtype or X2.dtype, device=X2.device)
        ws = _workspace(_lib.lib.dbf_forward_workspace_bytes(sh.n, sh.k_shard, sh.m_dim, X2.shape[0]), X2.device)
        _lib.check(
            _lib.lib.dbf_forward_allreduce(
                self.A.tiled.data_ptr(), self.B.tiled.data_ptr(), self.a.data_ptr(), self.mid.data_ptr(),
                self.b.data_ptr(), _lib.dtype_code(self.a.dtype), sh.n, sh.k_shard, sh.m_dim, X2.data_ptr(),
                _lib.dtype_code(X2.dtype), X2.shape[0], X2.stride(0), Y.data_ptr(), _lib.dtype_code(Y.dtype),
                Y.stride(0), peer_recv.data_ptr(), peer_flags.data_ptr(), sh.world, sh.rank, epoch_counter.data_ptr(),
                ws.data_ptr(), ws.numel(), _lib.stream_ptr(),
            ),
            "dbf_forward_allreduce",
        )
        return Y


class FusedAllReduce:
    """Receive buffers and flags of ``dbf_forward_allreduce`` in torch symmetric memory: every
    rank maps every peer's buffers, so GEMV2's epilogue stores partials straight into them over
    NVLink.  One instance serves every call with at most (n, batch); calls are counted on the
    device, so a captured CUDA graph of ``forward`` replays correctly."""

    def __init__(self, n: int, batch: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        from . import _lib

        if batch > 16:
            raise ValueError("the fused all-reduce handles batch <= 16")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n, self.batch = n, batch
        self.counter = torch.zeros(1, dtype=torch.int32, device=dev)
        if not dist.is_initialized():  # one process, no group: the buffers are local
            self.world, self.rank = 1, 0
            self.recv = torch.empty(_lib.lib.dbf_allreduce_recv_bytes(n, batch, 1) // 4, dtype=torch.float32,
                                    device=dev)
            self.flags = torch.zeros(_lib.lib.dbf_allreduce_flag_bytes(n, 1) // 4, dtype=torch.int32, device=dev)
            self.peer_recv = torch.tensor([self.recv.data_ptr()], dtype=torch.int64, device=dev)
            self.peer_flags = torch.tensor([self.flags.data_ptr()], dtype=torch.int64, device=dev)
            return
        grp = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(grp)
        self.rank = dist.get_rank(grp)
        rb = _lib.lib.dbf_allreduce_recv_bytes(n, batch, self.world)
        fb = _lib.lib.dbf_allreduce_flag_bytes(n, self.world)
        self.recv = symm_mem.empty(rb // 4, dtype=torch.float32, device=dev)
        self.flags = symm_mem.empty(fb // 4, dtype=torch.int32, device=dev)
        self.flags.zero_()
        torch.cuda.synchronize(dev)
        hr = symm_mem.rendezvous(self.recv, grp)
        hf = symm_mem.rendezvous(self.flags, grp)
        self.peer_recv = torch.tensor(list(hr.buffer_ptrs), dtype=torch.int64, device=dev)
        self.peer_flags = torch.tensor(list(hf.buffer_ptrs), dtype=torch.int64, device=dev)
        self._handles = (hr, hf)
        dist.barrier(group=grp)  # every rank's flags are zero before anyone pushes

    def forward(self, shard: "DeviceShard", X, out_dtype=None, engine: bool = False):
        """engine=True: the decode-engine path (``forward_allreduce_engine``, batch <= 4)."""
        if (X.shape[0] if X.ndim == 2 else 1) > self.batch or shard.shard.n != self.n:
            raise ValueError("layer/batch larger than this FusedAllReduce was sized for")
        if shard.shard.world != self.world or shard.shard.rank != self.rank:
            raise ValueError("shard rank/world do not match the process group")
        fwd = shard.forward_allreduce_engine if engine else shard.forward_allreduce
        return fwd(X, self.peer_recv, self.peer_flags, self.counter, out_dtype=out_dtype)


def reduce_partials_host(partials, a) -> np.ndarray:
    """Host restatement of the combine step (used by the CPU multi-process tests)."""
    total = np.sum(np.stack(partials), axis=0)
    return total * np.asarray(a)[None, :]
