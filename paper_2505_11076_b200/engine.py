"""Host side of the decode engine (include/dbf_b200.h ``dbf_engine_*``).

Compiles a ``DecodePlan`` (ordered layer forwards + activation dataflow) into one persistent
kernel program:

* every layer forward becomes two SEGMENTS -- B (iscale = b, oscale = mid) writing the LL
  vector t, then A (oscale = a) writing the LL vector y -- exactly the staging of
  kernel.py:59-61;
* ops are grouped into dependency LEVELS (q/k/v of a block share the block input, gate/up
  share o's output), and each level becomes two STAGES (all GEMV1s, then all GEMV2s), so the
  independent layers of a level fill the GPU together;
* each stage's 16-row UNITS are block-distributed over the CTAs (one per SM), rotating the
  start from stage to stage so bytes stay balanced over the run; a CTA's list is in stage
  order, which is what makes the in-kernel LL waits deadlock-free.

The program is plain device arrays; ``EngineProgram.launch()`` is one cooperative launch.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import DbfOverflowError

SEG_DTYPE = np.dtype(
    {
        "names": ["tiled", "rows", "cols", "in_vec", "out_vec", "iscale", "oscale", "scale_dtype", "out_dtype", "out_plain"],
        "formats": ["<u8", "<i4", "<i4", "<i4", "<i4", "<u8", "<u8", "<i4", "<i4", "<u8"],
        "offsets": [0, 8, 12, 16, 20, 24, 32, 40, 44, 48],
        "itemsize": 56,
    }
)
VEC_DTYPE = np.dtype(
    {
        "names": ["data", "len", "kind", "dtype", "producers"],
        "formats": ["<u8", "<i4", "<i4", "<i4", "<i4"],
        "offsets": [0, 8, 12, 16, 20],
        "itemsize": 24,
    }
)


class _Program(ctypes.Structure):
    _fields_ = [
        ("runs", ctypes.c_void_p),
        ("cta_offsets", ctypes.c_void_p),
        ("run_counter", ctypes.c_void_p),
        ("trace", ctypes.c_void_p),
        ("nvectors", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("max_cols", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("x_override", ctypes.c_void_p),
        ("y_override", ctypes.c_void_p),
        ("qscratch", ctypes.c_void_p),
        ("qscratch_cta_bytes", ctypes.c_int64),
        ("ar_recv", ctypes.c_void_p),
        ("ar_flags", ctypes.c_void_p),
        ("ar_epoch", ctypes.c_void_p),
        ("ar_a", ctypes.c_void_p),
        ("ar_world", ctypes.c_int32),
        ("ar_rank", ctypes.c_int32),
        ("ar_bt", ctypes.c_int32),
        ("ar_sdt", ctypes.c_int32),
        ("ar_ydt", ctypes.c_int32),
        ("ar_pad", ctypes.c_int32),
        ("ar_ldy", ctypes.c_int64),
    ]


_lib.lib.dbf_engine_smem_bytes.restype = ctypes.c_int
_lib.lib.dbf_engine_smem_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]
_lib.lib.dbf_engine_occupancy.restype = ctypes.c_int
_lib.lib.dbf_engine_occupancy.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
_lib.lib.dbf_engine_build_runs.restype = ctypes.c_int
_lib.lib.dbf_engine_build_runs.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32,
                                           ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                           ctypes.c_void_p]
_lib.lib.dbf_engine_launch.restype = ctypes.c_int
_lib.lib.dbf_engine_launch.argtypes = [ctypes.POINTER(_Program), ctypes.c_void_p]


def occupancy(max_cols: int) -> tuple[int, int]:
    """(engine CTAs per SM, registers per thread) for a program whose widest segment is max_cols."""
    b, r = ctypes.c_int32(0), ctypes.c_int32(0)
    _lib.check(_lib.lib.dbf_engine_occupancy(max_cols, ctypes.byref(b), ctypes.byref(r)), "dbf_engine_occupancy")
    return b.value, r.value


def run_limits(batch: int = 1, max_cols: int = 0) -> tuple[int, int]:
    """(units per run, packed-sign bytes per run) the engine accepts at this batch for a program
    whose widest segment has max_cols columns."""
    u, b = ctypes.c_int32(0), ctypes.c_int64(0)
    _lib.check(_lib.lib.dbf_engine_run_limits_cols(max_cols, batch, ctypes.byref(u), ctypes.byref(b)),
               "dbf_engine_run_limits_cols")
    return u.value, b.value


def levels_of(ops, input_buffer: int) -> list[int]:
    """Dependency level of each op: 1 + level of the op that last wrote its source buffer."""
    writer_level: dict[int, int] = {}
    lv = []
    for op in ops:
        level = writer_level.get(op.src, -1) + 1
        lv.append(level)
        writer_level[op.dst] = level
    return lv


def distribute(units: list[tuple[int, int]], grid: int, rotate: int,
               unit_bytes: dict | None = None) -> list[list[tuple[int, int]]]:
    """Distribution of a stage's units over CTAs, starting at CTA `rotate`.

    A stage with several segments (q/k/v, gate/up) gives every segment its own set of CTAs, sized
    in proportion to the segment's bytes, and block-distributes each segment's units over its set:
    no CTA then holds units of two segments, which would make it run two runs back to back and
    finish the stage last.  A single segment (or more segments than CTAs) is block-distributed."""
    out: list[list[tuple[int, int]]] = [[] for _ in range(grid)]
    segs: dict[int, list[tuple[int, int]]] = {}
    for u in units:
        segs.setdefault(u[0], []).append(u)
    if len(segs) == 1 or len(segs) > grid:
        n = len(units)
        for c in range(grid):
            lo, hi = (c * n) // grid, ((c + 1) * n) // grid
            out[(c + rotate) % grid].extend(units[lo:hi])
        return out
    order = list(segs)
    weight = [len(segs[sg]) * ((unit_bytes or {}).get(sg, 1)) for sg in order]
    total = float(sum(weight))
    # largest-remainder apportionment of the CTAs, at least one per segment
    quota = [max(1.0, grid * w / total) for w in weight]
    counts = [max(1, int(q)) for q in quota]
    while sum(counts) > grid:
        i = max(range(len(counts)), key=lambda j: (counts[j] - quota[j], counts[j]))
        counts[i] -= 1
    while sum(counts) < grid:
        i = max(range(len(counts)), key=lambda j: quota[j] - counts[j])
        counts[i] += 1
    base = 0
    for sg, cnt in zip(order, counts):
        lst = segs[sg]
        n = len(lst)
        for c in range(cnt):
            lo, hi = (c * n) // cnt, ((c + 1) * n) // cnt
            out[(base + c + rotate) % grid].extend(lst[lo:hi])
        base += cnt
    return out


class EngineProgram:
    """A DecodePlan compiled for the persistent decode engine."""

    def __init__(self, plan, grid: int | None = None, device="cuda"):
        import torch

        _lib.require_cuda()
        self.plan = plan
        props = torch.cuda.get_device_properties(device)
        self.grid = int(grid or props.multi_processor_count)
        dev = torch.device(device)
        act = plan.buffers[plan.input_buffer]
        self.batch = int(act.shape[0])
        if not 1 <= self.batch <= 4:
            raise ValueError("the decode engine runs 1..4 tokens per step (use forward_device for larger batches)")
        act_code = _lib.dtype_code(act.dtype)
        if act_code not in (_lib.F16, _lib.F32):
            raise ValueError("engine activations must be float16 or float32")

        # ---- vectors ------------------------------------------------------------------------
        vecs = []  # (data tensor, len, kind, dtype)
        self._keep = []
        self._out_private = None

        def ll_vector(length: int) -> int:
            # uint32 {fp16, epoch16} words, padded to whole 256-column chunks (the kernel reads them),
            # one padded row per token
            t = torch.zeros(self.batch * (((length + 255) // 256) * 256), dtype=torch.int32, device=dev)
            self._keep.append(t)
            vecs.append((t.data_ptr(), length, 1, 0))
            return len(vecs) - 1

        vecs.append((act.data_ptr(), act.shape[1], 0, act_code))  # vector 0: the step input
        latest = {plan.input_buffer: 0}  # buffer id -> vector holding its current version

        lv = levels_of(plan.ops, plan.input_buffer)
        last_writer = {}
        consumed = [False] * len(plan.ops)  # is op i's output read by a later op?
        for i, op in enumerate(plan.ops):
            if op.src in last_writer:
                consumed[last_writer[op.src]] = True
            last_writer[op.dst] = i
        final_op = last_writer.get(plan.output_buffer)

        segs = []
        stage_units: dict[int, list[tuple[int, int]]] = {}
        for i, op in enumerate(plan.ops):
            layer = plan.layers[op.layer]
            sd = _lib.dtype_code(layer.mid.dtype)
            if sd not in (_lib.F16, _lib.F32):
                raise ValueError("engine scales must be float16 or float32")
            if op.src not in latest:  # read before any op wrote it: an external (plain) input
                buf = plan.buffers[op.src]
                vecs.append((buf.data_ptr(), buf.shape[1], 0, _lib.dtype_code(buf.dtype)))
                latest[op.src] = len(vecs) - 1
            src_vec = latest[op.src]
            t_vec = ll_vector(layer.k)
            # outputs read by a later op are published as LL words; the final output and outputs
            # nobody reads in the plan (e.g. q, k of the benchmark's block, whose consumer --
            # attention -- is outside this path) are plain stores into the destination buffer
            y_vec = ll_vector(layer.n) if consumed[i] else -1
            plain = i == final_op or not consumed[i]
            segs.append((layer.B.tiled.data_ptr(), layer.k, layer.m_dim, src_vec, t_vec, layer.b.data_ptr(),
                         layer.mid.data_ptr(), sd, _lib.F32, 0))
            out_plain = plan.buffers[op.dst].data_ptr() if plain else 0
            if plain and i == final_op and out_plain == act.data_ptr():
                # the step input is also the step output (a decoder's residual stream h): the
                # final stage writes a private buffer that launch() copies back after the kernel,
                # so no CTA can read vector 0 after another has overwritten it
                self._out_private = torch.empty_like(plan.buffers[op.dst])
                self._out_user = plan.buffers[op.dst]
                out_plain = self._out_private.data_ptr()
            out_code = _lib.dtype_code(plan.buffers[op.dst].dtype) if plain else act_code
            if out_code not in (_lib.F16, _lib.F32):
                raise ValueError("engine outputs must be float16 or float32")
            # layer.a None: no output scale (a k-shard's partial; the scale follows the all-reduce)
            segs.append((layer.A.tiled.data_ptr(), layer.n, layer.k, t_vec, y_vec, 0,
                         layer.a.data_ptr() if layer.a is not None else 0, sd, out_code, out_plain))
            latest[op.dst] = y_vec
            for stage, seg_idx, rows in ((2 * lv[i], len(segs) - 2, layer.k), (2 * lv[i] + 1, len(segs) - 1, layer.n)):
                stage_units.setdefault(stage, []).extend((seg_idx, rb) for rb in range((rows + 15) // 16))

        seg_unit_bytes = {j: ((sg[2] + 255) // 256) * 512 for j, sg in enumerate(segs)}
        per_cta: list[list[tuple[int, int]]] = [[] for _ in range(self.grid)]
        rot = 0
        for stage in sorted(stage_units):
            units = stage_units[stage]
            for c, lst in enumerate(distribute(units, self.grid, rot, seg_unit_bytes)):
                per_cta[c].extend(lst)
            rot = (rot + len(units)) % self.grid
        # compress each CTA's unit list into runs: consecutive row blocks of one segment, at most
        # max_units units / max_run_bytes of packed signs each (dbf_engine_run_limits)
        max_units, max_bytes = run_limits(self.batch, max(sg[2] for sg in segs))
        unit_bytes = {j: ((sg[2] + 255) // 256) * 512 for j, sg in enumerate(segs)}
        per_cta_runs: list[list[tuple[int, int, int]]] = []
        for lst in per_cta:
            maximal: list[list[int]] = []
            for seg, rb in lst:
                if maximal and maximal[-1][0] == seg and maximal[-1][1] + maximal[-1][2] == rb:
                    maximal[-1][2] += 1
                else:
                    maximal.append([seg, rb, 1])
            runs_c: list[tuple[int, int, int]] = []
            for seg, rb, n in maximal:  # split evenly (e.g. 10 units -> 5 + 5, not 8 + 2)
                cap = max(1, min(max_units, max_bytes // unit_bytes[seg]))
                parts = -(-n // cap)
                start = rb
                for p in range(parts):
                    cnt = n * (p + 1) // parts - n * p // parts
                    runs_c.append((seg, start, cnt))
                    start += cnt
            per_cta_runs.append(runs_c)
        offsets = np.zeros(self.grid + 1, dtype=np.int32)
        offsets[1:] = np.cumsum([len(x) for x in per_cta_runs])
        flat = np.ascontiguousarray(np.array([r for lst in per_cta_runs for r in lst], dtype=np.int32).reshape(-1, 3))
        self.nunits = sum(len(x) for x in per_cta)

        seg_arr = np.zeros(len(segs), dtype=SEG_DTYPE)
        for j, sg in enumerate(segs):
            seg_arr[j] = sg
        vec_arr = np.zeros(len(vecs), dtype=VEC_DTYPE)
        for j, (ptr, ln, kind, dt) in enumerate(vecs):
            vec_arr[j] = (ptr, ln, kind, dt, 0)

        self.max_cols = max(sg[2] for sg in segs)
        # [epoch base, CTAs done, status bits, reserved] (dbf_engine_program.run_counter)
        self.run_counter = torch.zeros(4, dtype=torch.int32, device=dev)
        self.ready = torch.zeros(len(vecs), dtype=torch.int32, device=dev)
        records = np.zeros(len(flat) * 128, dtype=np.uint8)
        _lib.check(
            _lib.lib.dbf_engine_build_runs(
                seg_arr.ctypes.data, len(segs), vec_arr.ctypes.data, len(vecs), flat.ctypes.data, len(flat),
                self.batch, self.ready.data_ptr(), records.ctypes.data,
            ),
            "dbf_engine_build_runs",
        )

        def dev_bytes(a: np.ndarray):
            t = torch.from_numpy(np.frombuffer(a.tobytes(), dtype=np.uint8).copy()).to(dev)
            self._keep.append(t)
            return t.data_ptr()

        self.records = records  # host copy of the run records (diagnostics)
        self.nruns = len(flat)
        self.units_per_cta = np.array([len(x) for x in per_cta])
        self.nstages = len(stage_units)
        self.nsegments = len(segs)
        self._prog = _Program(
            dev_bytes(records), dev_bytes(offsets), self.run_counter.data_ptr(), None,
            len(vecs), self.grid, self.max_cols, self.batch,
        )
        self._offsets = offsets
        self._flat = flat
        qb = _lib.lib.dbf_engine_qscratch_bytes(self.max_cols, self.batch)
        if qb:  # quantized-input scratch for wide inputs at 2-4 tokens (L2-resident, per CTA)
            qb = (qb + 255) // 256 * 256
            self.qscratch = torch.empty(self.grid * qb, dtype=torch.uint8, device=dev)
            self._prog.qscratch, self._prog.qscratch_cta_bytes = self.qscratch.data_ptr(), qb
        size = ctypes.c_size_t(0)
        _lib.check(_lib.lib.dbf_engine_smem_bytes(self.max_cols, self.batch, ctypes.byref(size)), "dbf_engine_smem_bytes")
        self.smem_bytes = size.value

    def enable_trace(self):
        """Record 4 %globaltimer stamps per run (start, input ready, first weights ready, done)."""
        import torch

        self.trace = torch.zeros((max(self.nruns, 1), 4), dtype=torch.int64, device="cuda")
        self._prog.trace = self.trace.data_ptr()
        return self

    def launch(self, stream=None):
        _lib.check(_lib.lib.dbf_engine_launch(ctypes.byref(self._prog), _lib.stream_ptr(stream)), "dbf_engine_launch")
        if self._out_private is not None:
            import torch

            if stream is None:
                self._out_user.copy_(self._out_private)
            else:
                with torch.cuda.stream(stream):
                    self._out_user.copy_(self._out_private)

    def launch_io(self, x, y, stream=None):
        """Launch on caller buffers: x replaces the step input (vector 0: batch x len, contiguous,
        the dtype the program was built for) and y the final plain output."""
        inp = self.plan.buffers[self.plan.input_buffer]
        out = self.plan.buffers[self.plan.output_buffer]
        if x.shape != inp.shape or x.dtype != inp.dtype or not x.is_contiguous():
            raise ValueError(f"x must be a contiguous {tuple(inp.shape)} {inp.dtype} tensor")
        if y.shape != out.shape or y.dtype != out.dtype or not y.is_contiguous():
            raise ValueError(f"y must be a contiguous {tuple(out.shape)} {out.dtype} tensor")
        prog = _Program.from_buffer_copy(self._prog)
        prog.x_override, prog.y_override = x.data_ptr(), y.data_ptr()
        _lib.check(_lib.lib.dbf_engine_launch(ctypes.byref(prog), _lib.stream_ptr(stream)), "dbf_engine_launch")

    def launch_allreduce(self, x, y, peer_recv, peer_flags, epoch_counter, world: int, rank: int, a,
                         stream=None):
        """Launch on caller buffers with the one-shot all-reduce fused into the last stage
        (dbf_engine_program.ar_*): the final plain output is pushed to every rank's receive
        buffer and y = a * (sum over ranks) is written to ``y`` (batch x n, any io dtype)."""
        inp = self.plan.buffers[self.plan.input_buffer]
        out = self.plan.buffers[self.plan.output_buffer]
        if x.shape != inp.shape or x.dtype != inp.dtype or not x.is_contiguous():
            raise ValueError(f"x must be a contiguous {tuple(inp.shape)} {inp.dtype} tensor")
        if y.shape != out.shape or y.stride(1) != 1:
            raise ValueError(f"y must be a {tuple(out.shape)} tensor with unit column stride")
        if not 1 <= world <= 8 or not 0 <= rank < world:
            raise ValueError("world must be 1..8 and 0 <= rank < world")
        prog = _Program.from_buffer_copy(self._prog)
        prog.x_override, prog.y_override = x.data_ptr(), y.data_ptr()
        prog.ar_recv, prog.ar_flags, prog.ar_epoch = peer_recv.data_ptr(), peer_flags.data_ptr(), epoch_counter.data_ptr()
        prog.ar_a, prog.ar_sdt = a.data_ptr(), _lib.dtype_code(a.dtype)
        prog.ar_world, prog.ar_rank, prog.ar_bt = world, rank, x.shape[0]
        prog.ar_ydt, prog.ar_ldy = _lib.dtype_code(y.dtype), y.stride(0)
        _lib.check(_lib.lib.dbf_engine_launch(ctypes.byref(prog), _lib.stream_ptr(stream)), "dbf_engine_launch")

    def kernel_launches_per_step(self) -> int:
        return 1  # the engine kernel (its last CTA advances the launch counter)

    def status(self, clear: bool = True) -> int:
        """Sticky status bits of the launches since the last clear (reads device memory: syncs):
        STATUS_NONFINITE = an input chunk held inf/NaN (the outputs it fed are NaN),
        STATUS_OVERFLOW = a value published in fp16 overflowed (|v| > 65504)."""
        bits = int(self.run_counter[2].item())
        if clear and bits:
            self.run_counter[2].zero_()
        return bits

    def check(self):
        """Raise DbfOverflowError if any launch since the last check saw a non-finite input or
        an fp16 overflow (the engine never turns those into finite garbage: the outputs are NaN /
        inf, and this reports them)."""
        bits = self.status()
        if bits:
            what = []
            if bits & STATUS_NONFINITE:
                what.append("a non-finite (inf/NaN) input reached the engine; the outputs it feeds are NaN")
            if bits & STATUS_OVERFLOW:
                what.append("a value published in fp16 overflowed (|v| > 65504)")
            raise DbfOverflowError("; ".join(what))


STATUS_NONFINITE = 1
STATUS_OVERFLOW = 2


class EngineGroups:
    """Batches above 4 tokens: one EngineProgram per group of <= 4 token rows, launched back to
    back on the same stream (each group re-reads the weights; tokens never interact)."""

    def __init__(self, groups):
        self.groups = list(groups)

    def launch(self, stream=None):
        for g in self.groups:
            g.launch(stream)

    def kernel_launches_per_step(self) -> int:
        return sum(g.kernel_launches_per_step() for g in self.groups)

    def enable_trace(self):
        for g in self.groups:
            g.enable_trace()
        return self

    def check(self):
        for g in self.groups:
            g.check()

