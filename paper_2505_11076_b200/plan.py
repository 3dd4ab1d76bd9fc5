"""Multi-layer decode plans: a chain of DBF layer forwards replayed as one CUDA graph.

The reference applies one layer per ``forward`` call (kernel.py:48-62).  A decode step of a
factorized model applies every linear layer once per token, so the natural B200 unit of work is
the whole chain: ``DecodePlan`` records the layer order and the activation dataflow of a decoder
(q/k/v read the block input, o reads v's output as the attention stand-in, gate/up read o's
output, down reads gate's output and produces the next block input -- attention, norms and the
SiLU product are outside this path) and replays it as a single CUDA graph, so per-layer host
launch overhead disappears.

``run(x)`` accepts a host (numpy / CPU tensor) or device input and copies host inputs in and the
final output back inside the call -- the end-to-end path the benchmark's ``e2e`` number times.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import _lib
from .budget import middle_dim
from .device import DeviceLayer
from .kernel import (BATCHED_MAX_TOKENS, batched_frag, batched_quantize, forward_batched_frag, forward_device,
                     forward_prefill, random_device_layer)

# Llama-2 linear shapes (n = out_features, m = in_features), SURVEY.md §8a
LLAMA_SHAPES = {
    "llama2-7b": dict(hidden=4096, inter=11008, kv=4096, blocks=32),
    "llama2-13b": dict(hidden=5120, inter=13824, kv=5120, blocks=40),
    "llama2-70b": dict(hidden=8192, inter=28672, kv=1024, blocks=80),
}


def block_shapes(model: str) -> list[tuple[str, int, int]]:
    s = LLAMA_SHAPES[model]
    h, i, kv = s["hidden"], s["inter"], s["kv"]
    return [("q", h, h), ("k", kv, h), ("v", kv, h), ("o", h, h), ("gate", i, h), ("up", i, h), ("down", h, i)]


@dataclass
class PlanOp:
    layer: int  # index into DecodePlan.layers
    src: int  # activation buffer read
    dst: int  # activation buffer written
    name: str = ""


def batched_dataflow(ops, max_readers: int = 4):
    """Dataflow of a batched chain (DecodePlan.use_batched) from the op list alone.

    readers[w]: the ops whose first-GEMV fragments op w's finalize writes -- every op reading the
    buffer w wrote, until the next write to it (at most max_readers; more read it on their own).
    standalone: the ops that quantize their input themselves (input from outside the chain, or a
    reader beyond max_readers).  deps[i]: the ops op i must follow when independent ops run on
    concurrent streams -- the producer of its input, the previous writer of its output buffer and
    every op that read that buffer's previous contents (chained readers read fragments, not the
    buffer; they are ordered conservatively)."""
    last_writer, readers, standalone = {}, {i: [] for i in range(len(ops))}, set()
    for i, op in enumerate(ops):
        w = last_writer.get(op.src)
        if w is None or len(readers[w]) >= max_readers:
            standalone.add(i)
        else:
            readers[w].append(i)
        last_writer[op.dst] = i
    deps, last_w, reads_since = [], {}, {}
    for i, op in enumerate(ops):
        d = set()
        if op.src in last_w:
            d.add(last_w[op.src])
        if op.dst in last_w:
            d.add(last_w[op.dst])
        d.update(reads_since.get(op.dst, ()))
        d.discard(i)
        deps.append(sorted(d))
        reads_since.setdefault(op.src, []).append(i)
        last_w[op.dst] = i
        reads_since[op.dst] = []
    return readers, standalone, deps


@dataclass
class DecodePlan:
    layers: list
    ops: list
    buffers: list  # device activation tensors (batch x width)
    input_buffer: int = 0
    output_buffer: int = 0
    engine: object = field(default=None, repr=False)
    _graph: object = field(default=None, repr=False)
    _stream: object = field(default=None, repr=False)

    # ---- accounting -------------------------------------------------------------------------
    def bytes_per_step(self) -> int:
        """Algorithmic HBM bytes of one step (summed over ops)."""
        act = self.buffers[0].element_size()
        batch = self.buffers[0].shape[0]
        return sum(self.layers[op.layer].bytes_logical(batch=batch, act_bytes=act) for op in self.ops)

    def kernel_launches_per_step(self) -> int:
        if self.engine is not None:
            return self.engine.kernel_launches_per_step()
        if getattr(self, "_mode", None) == "batched":
            # per layer GEMV, quantize, GEMV, finalize (+ a quantize for inputs from outside the
            # chain); per group of <= 32 tokens
            groups = self._bgroups or [self]
            return sum(4 * len(g.ops) + len(g._bchain[2]) for g in groups)
        return 2 * len(self.ops)  # one GEMV launch per stage (B, then A)

    # ---- execution --------------------------------------------------------------------------
    def use_engine(self, grid: int | None = None):
        """Run the whole chain in the persistent decode engine (one kernel per step).  One engine
        launch carries up to 4 tokens (they share every tensor-core MMA); larger batches run as
        consecutive launches over groups of <= 4 token rows of the same buffers."""
        from .engine import EngineGroups, EngineProgram

        batch = int(self.buffers[self.input_buffer].shape[0])
        if batch <= 4:
            self.engine = EngineProgram(self, grid=grid)
        else:
            groups = []
            for t0 in range(0, batch, 4):
                sub = DecodePlan(self.layers, self.ops, [b[t0:t0 + 4] for b in self.buffers],
                                 input_buffer=self.input_buffer, output_buffer=self.output_buffer)
                groups.append(EngineProgram(sub, grid=grid))
            self.engine = EngineGroups(groups)
        self._graph = None
        return self

    def use_layer_kernels(self):
        """Run one dbf_forward (two GEMV launches) per layer instead of the engine."""
        self.engine = None
        self._mode = "layer"
        self._graph = None
        return self

    def use_batched(self):
        """Run every layer through the batched kernels (csrc/batched.cu): up to 32 tokens share one
        pass over each sign matrix (four short kernels per layer, layers chained by fragments and
        independent ones on concurrent streams); larger batches run as consecutive groups of
        <= 32 token rows of the same buffers (one weight pass per group)."""
        import torch

        batch = int(self.buffers[self.input_buffer].shape[0])
        self.engine = None
        self._mode = "batched"
        if getattr(self, "_bstatus", None) is None:
            self._bstatus = torch.zeros(1, dtype=torch.int32, device=self.buffers[0].device)
        if batch > BATCHED_MAX_TOKENS:
            self._bgroups = []
            for t0 in range(0, batch, BATCHED_MAX_TOKENS):
                sub = DecodePlan(self.layers, self.ops, [b[t0:t0 + BATCHED_MAX_TOKENS] for b in self.buffers],
                                 input_buffer=self.input_buffer, output_buffer=self.output_buffer)
                sub._bstatus = self._bstatus
                self._bgroups.append(sub.use_batched())
        else:
            self._bgroups = None
            self._bchain = self._batched_chain(batch)
        self._graph = None
        return self

    def _batched_chain(self, batch: int):
        """Fragment buffers (one per op: its first-GEMV input) and the dataflow of the batched
        chain (batched_dataflow)."""
        device = self.buffers[0].device
        readers, standalone, deps = batched_dataflow(self.ops)
        frags = [batched_frag(self.layers[op.layer].m_dim, batch, device) for op in self.ops]
        return frags, readers, standalone, deps

    def use_prefill(self):
        """Run every layer through the tcgen05 sign GEMMs (forward_prefill) whatever the batch:
        one pass over the weights for all tokens (fp16 activations; layers built with keep_words)."""
        self.engine = None
        self._mode = "prefill"
        self._graph = None
        return self

    def _prefill_ok(self) -> bool:
        import torch

        return self.buffers[self.input_buffer].dtype == torch.float16 and all(
            l.scale_dtype == torch.float16 and l.A.words is not None and l.B.words is not None
            for l in self.layers)

    def default_path(self) -> str:
        """The static path rule for a token batch: the decode engine for 1 token (and 2 below 8 GB
        of weights per step), the batched kernels for 2-64 tokens (one weight pass per group of
        <= 32), the tcgen05 prefill chain above (when its layout is available).  Measured
        (ms per step): engine / batched 7B 2 tokens 1.55 / 1.89, 3 tokens 2.22 /
        1.90; 13B 2 tokens 2.38 / 2.57; 70B 2 tokens 13.0 / 9.6; batched / prefill chain 7B 32
        tokens 4.2 / 8.7, 70B 32 tokens 30.4 / 62.8, 13B 64 tokens 11.5 / 11.9."""
        batch = int(self.buffers[self.input_buffer].shape[0])
        if batch == 1 or (batch == 2 and self.bytes_per_step() < 8e9):
            # 2 tokens: the engine wins on 7B / 13B, the batched kernels on 70B (17.6 GB)
            return "engine"
        if batch <= 2 * BATCHED_MAX_TOKENS:
            return "batched"
        return "prefill" if self._prefill_ok() else "batched"

    def use_fastest(self, steps: int = 5, grid: int | None = None, margin: float = 0.10):
        """Time the decode engine (groups of <= 4 tokens) against the tcgen05 prefill chain on this
        plan's own buffers (CUDA graph replays, CUDA events; the input is restored before every
        candidate's warm-up and timing) and keep the static rule's path (default_path) unless the
        other is faster by more than `margin` -- so timing noise near the crossover cannot flip the
        choice.  The two paths round differently (13-bit chunk grid vs fp16 products with fp32
        sums): outputs are each path's own, within the fp16 tolerance of each other.  The choice is
        in ``self.choice`` / ``self.choice_ms``."""
        import torch

        _lib.require_cuda()
        cands = [("engine", lambda: self.use_engine(grid))]
        cands.append(("batched", self.use_batched))
        if self._prefill_ok():
            cands.append(("prefill", self.use_prefill))
        saved = self.buffers[self.input_buffer].clone()
        timings = {}
        for name, select in cands:
            select()
            self.buffers[self.input_buffer].copy_(saved)
            self.capture()
            for _ in range(2):
                self.buffers[self.input_buffer].copy_(saved)
                self.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                self.replay()
            e1.record()
            e1.synchronize()
            timings[name] = e0.elapsed_time(e1) / steps
        choice = self.default_path()
        other = min(timings, key=timings.get)
        if other != choice and timings[other] < (1.0 - margin) * timings[choice]:
            choice = other
        self.choice, self.choice_ms = choice, timings
        dict(cands)[choice]()
        self.buffers[self.input_buffer].copy_(saved)
        return self

    def _eager(self):
        if self.engine is not None:
            self.engine.launch()
            return
        mode = getattr(self, "_mode", "layer")
        if mode == "batched":
            for sub in self._bgroups or [self]:
                sub._eager_batched()
            return
        run = forward_prefill if mode == "prefill" else forward_device
        for op in self.ops:
            run(self.buffers[op.src], self.layers[op.layer], out=self.buffers[op.dst])

    def _eager_batched(self):
        """The batched chain with independent layers on concurrent streams (q/k/v, gate/up of a
        Llama block run side by side): an op waits only for its dependencies (events), each stream
        keeps its own workspace, and the streams fork from and join back into the current stream
        (so graph capture records the branches)."""
        import torch

        frags, readers, standalone, deps = self._bchain
        batch = int(self.buffers[self.input_buffer].shape[0])
        main = torch.cuda.current_stream()
        if getattr(self, "_bstreams", None) is None:
            self._bstreams = [main] + [torch.cuda.Stream() for _ in range(2)]
        streams = [main] + self._bstreams[1:]
        fork = torch.cuda.Event()
        fork.record(main)
        for st in streams[1:]:
            st.wait_event(fork)
        done, last_on = {}, {id(st): None for st in streams}
        for i, op in enumerate(self.ops):
            # a stream whose last op is a dependency (in-order: no event needed for that one), else
            # the stream idle longest
            st = next((st for st in streams if last_on[id(st)] in deps[i]), None)
            if st is None:
                st = min(streams, key=lambda x: -1 if last_on[id(x)] is None else last_on[id(x)])
            for d in deps[i]:
                if last_on[id(st)] != d:
                    st.wait_event(done[d])
            with torch.cuda.stream(st):
                layer = self.layers[op.layer]
                if i in standalone:
                    batched_quantize(self.buffers[op.src], layer, frags[i])
                cons = [(self.layers[self.ops[j].layer], frags[j]) for j in readers[i]]
                forward_batched_frag(frags[i], layer, batch, self.buffers[op.dst], consumers=cons,
                                     status=self._bstatus)
                ev = torch.cuda.Event()
                ev.record(st)
            done[i] = ev
            last_on[id(st)] = i
        for st in streams[1:]:
            j = torch.cuda.Event()
            j.record(st)
            main.wait_event(j)

    def capture(self):
        import torch

        _lib.require_cuda()
        self._stream = torch.cuda.Stream()
        self._stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self._stream):
            self._eager()  # warm-up: sets kernel attributes outside the capture
        torch.cuda.current_stream().wait_stream(self._stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self._stream):
            self._eager()
        self._graph = g
        return self

    def replay(self):
        """One step on the device (inputs already resident)."""
        if self._graph is None:
            self.capture()
        self._graph.replay()

    def run(self, x):
        """End-to-end step: host/device input -> device chain -> output (host if x was host)."""
        import numpy as np
        import torch

        inp = self.buffers[self.input_buffer]
        host = not (isinstance(x, torch.Tensor) and x.is_cuda)
        if host:
            xt = torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x)
            inp.copy_(xt.reshape(inp.shape), non_blocking=True)
        else:
            inp.copy_(x.reshape(inp.shape))
        self.replay()
        out = self.buffers[self.output_buffer]
        if not host:
            return out
        # the engine's sticky status word (non-finite input / fp16 overflow) rides along with the
        # output copy: queued before it, valid once the output copy has synchronized
        st = self._status_words()
        res = out.cpu()
        if st is not None:
            self._raise_status(st)
        return res

    def _status_words(self):
        """Queue a copy of every engine program's status word into pinned host memory."""
        import torch

        progs = getattr(self.engine, "groups", [self.engine]) if self.engine is not None else []
        progs = [p for p in progs if hasattr(p, "run_counter")]
        words = [p.run_counter[2:3] for p in progs]
        if getattr(self, "_mode", None) == "batched" and self.engine is None:
            progs, words = [self], [self._bstatus]
        if not progs:
            return None
        if getattr(self, "_status_host", None) is None or self._status_host.numel() != len(progs):
            self._status_host = torch.zeros(len(progs), dtype=torch.int32).pin_memory()
        for i, w in enumerate(words):
            self._status_host[i:i + 1].copy_(w, non_blocking=True)
        return progs

    def _raise_status(self, progs):
        if int(self._status_host.max()) != 0:
            for p in progs:
                p.check()

    def check(self):
        """Raise engine.DbfOverflowError if a step since the last check saw a non-finite input or
        overflowed fp16 (device calls: replay()/_eager() do not synchronize to look)."""
        if self.engine is not None:
            self.engine.check()
        elif getattr(self, "_mode", None) == "batched":
            from .engine import DbfOverflowError, STATUS_NONFINITE, STATUS_OVERFLOW

            st = int(self._bstatus.item())
            if st:
                self._bstatus.zero_()
                what = [w for bit, w in ((STATUS_NONFINITE, "a non-finite value"),
                                         (STATUS_OVERFLOW, "a value beyond the fp16 range")) if st & bit]
                raise DbfOverflowError(f"batched decode produced {' and '.join(what)} (status {st:#x})")


def layerwise_ks(model: str = "llama2-13b", target_bpw: float = 1.5, floor_bpw: float = 1.0, cap_bpw: float = 2.3,
                 blocks: int | None = None, seed: int = 0) -> list[int]:
    """Non-uniform per-layer middle dimensions (BASELINE configs[4]: 1.0-2.3 bits/weight across the
    layers of a model) from the reference's greedy allocation (budget.allocate_middle_dims,
    /root/reference/pkg/src/dbf/budget.py:187-261) at a global target, with every layer's source k
    at cap_bpw and its floor at floor_bpw.  The channel scores are synthetic (no calibration data
    here): per layer an exponentially decaying spectrum whose decay rate and scale vary by layer
    type and depth (seeded, deterministic).  Returns k per linear in plan order."""
    import numpy as np

    from .budget import allocate_middle_dims

    s = LLAMA_SHAPES[model]
    nblocks = blocks if blocks is not None else s["blocks"]
    rng = np.random.default_rng(seed)
    layers, scores = [], {}
    for bi in range(nblocks):
        for ti, (name, n, m) in enumerate(block_shapes(model)):
            nm = f"{bi}.{name}"
            k_src = middle_dim(n, m, cap_bpw, 32)
            depth = bi / max(nblocks - 1, 1)
            rate = (2.0 + 6.0 * rng.uniform() + 4.0 * abs(depth - 0.5)) / k_src
            scale = (1.0 + ti % 3) * (0.5 + depth) * rng.uniform(0.5, 1.5)
            layers.append((nm, n, m))
            scores[nm] = scale * np.exp(-rate * np.arange(k_src))
    ks = allocate_middle_dims(layers, scores, target_bpw, floor_bpw=floor_bpw, granularity=32)
    return [ks[nm] for nm, _, _ in layers]


def llama_decode_plan(model: str = "llama2-7b", bpw: float = 2.0, batch: int = 1, blocks: int | None = None,
                      generator=None, act_dtype=None, scale_dtype=None, device="cuda",
                      keep_words: bool | None = None, ks: list[int] | None = None) -> DecodePlan:
    """Synthetic random-init DBF factors of every linear layer of a Llama-2 model (§8d); ``ks``
    optionally gives every linear its own middle dimension (plan order, e.g. layerwise_ks)."""
    import torch

    act_dtype = act_dtype or torch.float16
    s = LLAMA_SHAPES[model]
    nblocks = blocks if blocks is not None else s["blocks"]
    shapes = block_shapes(model)
    layers, ops = [], []
    widths = {"h": s["hidden"], "q": s["hidden"], "k": s["kv"], "v": s["kv"], "o": s["hidden"],
              "gate": s["inter"], "up": s["inter"]}
    # activation buffers: 0 = block input h (also the output of down), one per layer output
    names = ["h", "q", "k", "v", "o", "gate", "up"]
    buffers = [torch.zeros((batch, widths[nm]), dtype=act_dtype, device=device) for nm in names]
    idx = {nm: i for i, nm in enumerate(names)}
    src_of = {"q": "h", "k": "h", "v": "h", "o": "v", "gate": "o", "up": "o", "down": "gate"}
    dst_of = {"q": "q", "k": "k", "v": "v", "o": "o", "gate": "gate", "up": "up", "down": "h"}
    if ks is not None and len(ks) != nblocks * len(shapes):
        raise ValueError(f"ks has {len(ks)} entries, expected {nblocks * len(shapes)}")
    for bi in range(nblocks):
        for li, (name, n, m) in enumerate(shapes):
            k = middle_dim(n, m, bpw, 32) if ks is None else int(ks[bi * len(shapes) + li])
            layers.append(random_device_layer(n, k, m, generator=generator, scale_dtype=scale_dtype, device=device,
                                              keep_words=batch >= 64 if keep_words is None else keep_words))
            ops.append(PlanOp(len(layers) - 1, idx[src_of[name]], idx[dst_of[name]], name))
    if s["kv"] != s["hidden"]:
        # GQA (70B): v is narrower than o's input; o reads q's output instead
        for op in ops:
            if op.name == "o":
                op.src = idx["q"]
    return DecodePlan(layers, ops, buffers, input_buffer=idx["h"], output_buffer=idx["h"])
