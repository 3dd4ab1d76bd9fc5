#!/usr/bin/env python
"""Benchmark of the DBF decode hot path on B200 (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): Llama-2-7B, every linear layer DBF-factorized at ~2 bits
per weight (k = middle_dim(n, m, 2.0, 32): q/k/v/o 4096x4096 k=4096, gate/up 11008x4096 k=5952,
down 4096x11008 k=5952), decode batch 1, synthetic random-init factors.
One STEP = one decode token through all 7 x 32 = 224 linear layers, in decoder dataflow order
(paper_2505_11076_b200.plan), replayed as one CUDA graph.  The 1.63 GB of packed weights touched
per step are > 2 x the 126 MB L2, so no L2 flush is needed between steps.

value      = algorithmic HBM bytes per step (SURVEY.md §8d formula, summed over the 224 layers)
             / device time per step -> GB/s (whole job: summed over ranks for --gpus N)
e2e        = the same metric through the public plan API with the step input copied from
             pinned host memory and the step output copied back inside the timed region
roofline   = the dominant kernel (the tensor-core sign GEMV) against MEASURED_PEAKS.json hbm_gbs
cpu_baseline = the reference algorithm (oracle restatement, bit-identical to dbf.forward) on the
             host cores, bounded sample (rank 0, N=1 only)

--impl reference times the reference CPU path (oracle restatement of dbf.forward, all host
cores via a process pool) on the same metric; the reference package cannot travel to the GPU
box, so its restatement -- pinned bit-exact to the reference's own outputs -- is what runs.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DBF layer µs & HBM GB/s (Llama2-7B shapes, bs=1); speedup vs fp16 cuBLAS GEMV"
WORKLOAD = "llama2-7b linears, DBF 2.0 bpw, decode bs=1 (224 layers/step)"

# Llama-2 linear shapes (n = out_features, m = in_features), kept here so that the reference arm
# never imports the product package (it must not load libdbf_b200.so)
LLAMA = {"llama2-7b": (4096, 11008, 4096, 32), "llama2-13b": (5120, 13824, 5120, 40),
         "llama2-70b": (8192, 28672, 1024, 80)}


def block_shapes(model: str) -> list[tuple[str, int, int]]:
    h, i, kv, _ = LLAMA[model]
    return [("q", h, h), ("k", kv, h), ("v", kv, h), ("o", h, h), ("gate", i, h), ("up", i, h), ("down", h, i)]


def middle_dim(n: int, m: int, bits: float, granularity: int = 32) -> int:
    """/root/reference/pkg/src/dbf/budget.py:113-132"""
    return max(int(bits * n * m / (n + m) // granularity) * granularity, granularity)


def layer_bytes(n: int, k: int, m: int, batch: int = 1, scale_bytes: int = 2, act_bytes: int = 2) -> int:
    """Algorithmic HBM bytes of one decode forward: packed signs of A and B, the
    three scale vectors, the input and output activations."""
    return n * ((k + 7) // 8) + k * ((m + 7) // 8) + scale_bytes * (n + k + m) + act_bytes * batch * (m + n)


def step_layers(model: str, bpw: float) -> list[tuple[str, int, int, int]]:
    """(name, n, k, m) of every linear of one decode step of `model`, in dataflow order."""
    blocks = LLAMA[model][3]
    return [(nm, n, middle_dim(n, m, bpw), m) for _ in range(blocks) for nm, n, m in block_shapes(model)]


def sharded_headline(args, world: int) -> bool:
    return world > 1 or args.sharded_step


def base_config(args, world: int) -> dict:
    """The workload as BOTH arms report it (same dict, so the driver can pair the lines)."""
    if sharded_headline(args, world):
        layers = step_layers("llama2-70b", 2.0)
        if args.blocks:
            layers = layers[: 7 * args.blocks]
        return {"workload": f"llama2-70b linears k-sharded over {world} GPUs, DBF 2.0 bpw, decode bs=1 "
                            f"({len(layers)} layers/step)",
                "model": "llama2-70b", "bpw": 2.0, "global_batch": 1, "seq_len": 1,
                "parallelism": f"k-shard x{world}", "layers_per_step": len(layers),
                "bytes_per_step": sum(layer_bytes(n, k, m) for _, n, k, m in layers),
                "l2": "working set > 2x126 MB L2 per step; no flush"}
    layers = step_layers(args.model, args.bpw)
    return {"workload": WORKLOAD if (args.model, args.bpw, args.batch) == ("llama2-7b", 2.0, 1) else
            f"{args.model} linears, DBF {args.bpw} bpw, decode bs={args.batch} ({len(layers)} layers/step)",
            "model": args.model, "bpw": args.bpw, "global_batch": args.batch * world, "seq_len": 1,
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU", "layers_per_step": len(layers),
            "bytes_per_step": sum(layer_bytes(n, k, m, args.batch) for _, n, k, m in layers),
            "l2": "working set > 2x126 MB L2 per step; no flush"}


# ---------------------------------------------------------------------------------------------
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--bpw", type=float, default=2.0)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-layers", action="store_true")
    ap.add_argument("--no-sharded", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--layer-kernels", action="store_true", help="per-layer GEMV kernels instead of the engine")
    ap.add_argument("--sharded-step", action="store_true",
                    help="headline the k-sharded Llama-2-70B step (the default when WORLD_SIZE > 1)")
    ap.add_argument("--blocks", type=int, default=None, help="decoder blocks of the sharded step (default: all)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def tensor_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"]))
    return 1590.0, 1400.0


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while the GPU is loaded."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
        except FileNotFoundError:
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------------------------
class CpuReference:
    """Reference algorithm (oracle restatement, bit-identical to dbf.forward) on one decoder
    block of the workload (q,k,v,o + gate,up + down) per step, rows split over all host cores."""

    def __init__(self, model: str, bpw: float, procs: int | None = None):
        from oracle import dbf_oracle as npo

        rng = np.random.default_rng(0)
        shapes = block_shapes(model)
        self.layers = {}
        for _, n, m in shapes:
            name = f"{n}x{m}"
            if name not in self.layers:
                k = npo.middle_dim(n, m, bpw)
                self.layers[name] = (
                    rng.uniform(0.5, 1.5, n) / np.sqrt(k),
                    rng.integers(0, 256, (n, npo.row_bytes(k)), dtype=np.uint8),
                    rng.uniform(0.5, 1.5, k),
                    rng.integers(0, 256, (k, npo.row_bytes(m)), dtype=np.uint8),
                    rng.uniform(0.5, 1.5, m) / np.sqrt(m),
                )
        self.order = [f"{n}x{m}" for _, n, m in shapes]
        self.bytes_per_block = 0
        for name in self.order:
            a, A, mid, B, b = self.layers[name]
            self.bytes_per_block += A.size + B.size + 2 * (len(a) + len(mid) + len(b)) + 2 * (len(b) + len(a))
        self.xs = {name: rng.standard_normal((1, len(v[4]))) for name, v in self.layers.items()}
        self.pf = npo.ProcessForward(self.layers, procs=procs)
        self.procs = self.pf.procs
        self.pf.forward(self.order[0], self.xs[self.order[0]])  # warm the pool

    def step(self) -> float:
        t0 = time.perf_counter()
        for name in self.order:
            self.pf.forward(name, self.xs[name])
        return time.perf_counter() - t0

    def close(self):
        self.pf.close()


def cpu_desc(model, bpw, procs):
    shapes = ", ".join(f"{nm} {n}x{m} k={middle_dim(n, m, bpw)}" for nm, n, m in block_shapes(model))
    return (f"bounded sample: one {model} decoder block per step (7 of the step's layers: {shapes}; "
            f"{bpw} bpw), bs=1, GB/s = that block's algorithmic bytes / its time; dbf.forward algorithm "
            f"(oracle restatement, bit-identical to the reference on its golden vectors), rows split over "
            f"{procs} processes")


# ---------------------------------------------------------------------------------------------
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # N>1: rank 0 alone runs the CPU reference; others exit 0 without work
    model, bpw = ("llama2-70b", 2.0) if sharded_headline(args, args.gpus) else (args.model, args.bpw)
    ref = CpuReference(model, bpw)
    for _ in range(args.warmup):
        ref.step()
    times = [ref.step() for _ in range(args.steps)]
    ref.close()
    t = float(np.mean(times))
    gbs = ref.bytes_per_block / t / 1e9
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": gbs,
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (uniform signs, U(0.5,1.5)-scaled vectors, N(0,1) input)",
        "config": base_config(args, args.gpus),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": ref.procs, "kind": "port",
                         "sample": cpu_desc(model, bpw, ref.procs),
                         "us_per_layer": t * 1e6 / len(ref.order)},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def build_cublas_chain(plan, dtype):
    """Dense fp16 weights of the same 224 shapes, same dataflow, cuBLAS GEMV per layer."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    weights = []
    for layer in plan.layers:
        w = torch.empty((layer.n, layer.m_dim), dtype=dtype, device="cuda")
        w.normal_(0, 1.0 / layer.m_dim**0.5, generator=g)
        weights.append(w)
    bufs = [torch.zeros_like(b) for b in plan.buffers]

    def step_out():
        for op in plan.ops:
            torch.matmul(bufs[op.src], weights[op.layer].t(), out=bufs[op.dst])

    nbytes = sum(2 * w.numel() + 2 * (w.shape[0] + w.shape[1]) for w in weights)
    return step_out, nbytes, weights


def graph_of(fn, warm=2):
    import torch

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    return g


def time_graph(g, steps, warmup, barrier=lambda: None):
    import torch

    for _ in range(warmup):
        g.replay()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    return e0.elapsed_time(e1) / steps  # ms per step


def layer_bench(model: str, bpw: float, steps: int, warmup: int, shapes=None, layer_kernels: bool = False):
    """The metric at layer level (SURVEY §8d timing method): per distinct Llama-2 linear shape at
    `bpw`, batch 1 -- (1) throughput: N distinct layer instances (total > 2x L2) that all read the
    same input, run as ONE engine program without dependencies between them, µs/layer = time / N;
    (2) isolated latency: one layer alone as one engine launch (B stage -> LL handoff -> A stage);
    (3) cuBLAS fp16 GEMV of the dense n x m layer, the same N distinct instances in a CUDA graph."""
    import torch

    import paper_2505_11076_b200 as P
    from paper_2505_11076_b200.plan import DecodePlan, PlanOp

    rows = []
    seen = set()
    for name, n, m in (shapes or block_shapes(model)):
        if (n, m) in seen:
            continue
        seen.add((n, m))
        k = middle_dim(n, m, bpw, 32)
        g = torch.Generator(device="cuda")
        g.manual_seed(7)
        one = P.random_device_layer(n, k, m, generator=g)
        lb = one.bytes_logical(batch=1, act_bytes=2)
        inst = int(min(96, max(4, -(-260_000_000 // lb))))
        layers = [one] + [P.random_device_layer(n, k, m, generator=g) for _ in range(inst - 1)]
        x = torch.randn((1, m), generator=g, device="cuda").half()
        bufs = [x] + [torch.zeros((1, n), dtype=torch.half, device="cuda") for _ in range(inst)]
        ops = [PlanOp(i, 0, i + 1, name) for i in range(inst)]
        tp = DecodePlan(layers, ops, bufs, input_buffer=0, output_buffer=inst).use_engine()
        tp.capture()
        ms_t = time_graph(tp._graph, steps, warmup)
        iso = DecodePlan([one], [PlanOp(0, 0, 1, name)], [x, bufs[1]], input_buffer=0, output_buffer=1).use_engine()
        iso.capture()
        ms_i = time_graph(iso._graph, steps * 10, warmup)
        ws = [torch.empty((n, m), dtype=torch.half, device="cuda").normal_(0, m ** -0.5, generator=g)
              for _ in range(inst)]
        ys = [torch.empty((1, n), dtype=torch.half, device="cuda") for _ in range(inst)]
        gc = graph_of(lambda: [torch.matmul(x, w.t(), out=y) for w, y in zip(ws, ys)])
        ms_c = time_graph(gc, steps, warmup)
        dense = 2 * n * m + 2 * (n + m)
        row = {"layer": name, "n": n, "k": k, "m": m, "bytes": lb, "instances": inst,
               "us_per_layer": ms_t * 1e3 / inst, "gbs": lb * inst / (ms_t * 1e-3) / 1e9,
               "us_isolated": ms_i * 1e3, "gbs_isolated": lb / (ms_i * 1e-3) / 1e9,
               "cublas_fp16_us_per_layer": ms_c * 1e3 / inst,
               "cublas_fp16_gbs": dense * inst / (ms_c * 1e-3) / 1e9,
               "speedup_vs_cublas": ms_c / ms_t}
        if layer_kernels:  # the per-layer GEMV kernels (two launches: B then A), same instances
            gk = graph_of(lambda: [P.forward_device(x, l, out=b) for l, b in zip(layers, bufs[1:])])
            ms_k = time_graph(gk, steps, warmup)
            row.update({"us_per_layer_layer_kernels": ms_k * 1e3 / inst,
                        "gbs_layer_kernels": lb * inst / (ms_k * 1e-3) / 1e9})
            del gk
        rows.append(row)
        del tp, iso, gc, ws, ys, layers
        torch.cuda.empty_cache()
    return {"model": model, "bpw": bpw, "batch": 1,
            "note": "independent instances in one engine launch (throughput) / one layer per launch (isolated)",
            "rows": rows}


def prefill_bench(model: str, bpw: float, tokens: int, steps: int, warmup: int):
    """BASELINE configs[2]: every Llama-2 linear shape at ~1 bpw, a prefill of `tokens` tokens through
    the tcgen05 path (forward_prefill), timed per distinct shape with CUDA events, against the
    dense fp16 cuBLAS GEMM of the same shapes; FLOPs = 2 T k (n + m) per layer."""
    import torch

    import paper_2505_11076_b200 as P

    from paper_2505_11076_b200 import _lib

    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    rows, total_us, total_dense_us, total_flops = [], 0.0, 0.0, 0.0
    kept = []
    shapes = block_shapes(model)
    for name, n, m in shapes:
        k = middle_dim(n, m, bpw, 32)
        layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
        layer.A.paired, layer.B.paired  # build the prefill layout outside the timed region
        X = torch.randn((tokens, m), generator=g, device="cuda").half()
        Y = torch.empty((tokens, n), dtype=torch.half, device="cuda")
        W = torch.randn((n, m), generator=g, device="cuda").half()
        Yd = torch.empty_like(Y)

        def t_of(fn):
            for _ in range(warmup):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                fn()
            e1.record()
            e1.synchronize()
            return e0.elapsed_time(e1) * 1e3 / steps

        us = t_of(lambda: P.forward_prefill(X, layer, out=Y))
        us_dense = t_of(lambda: torch.matmul(X, W.t(), out=Yd))
        flops = 2.0 * tokens * k * (n + m)
        rows.append({"layer": name, "n": n, "k": k, "m": m, "us": us, "tflops": flops / us / 1e6,
                     "cublas_fp16_dense_us": us_dense,
                     "path": "one launch" if _lib.lib.dbf_prefill_layer_path(n, k, m, tokens) == 2 else "two launches"})
        total_us += us
        total_dense_us += us_dense
        total_flops += flops
        kept.append((layer, X, Y, W, Yd))

    def sustained(fn, seconds=2.0):
        """The whole block back to back for ~2 s with the SM clock sampled: the prefill draws the
        board to its power cap, so this is the figure to set against bf16_tflops_sustained."""
        fn()
        torch.cuda.synchronize()
        clk = ClockSampler(torch.cuda.current_device()).start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters, t_end = 0, time.time() + seconds
        e0.record()
        while time.time() < t_end:
            for _ in range(5):
                fn()
            iters += 5
            torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e3 / iters, clk.stop()

    def block():
        for layer, X, Y, _, _ in kept:
            P.forward_prefill(X, layer, out=Y)

    def block_dense():
        for _, X, _, W, Yd in kept:
            torch.matmul(X, W.t(), out=Yd)

    us_s, clk_s = sustained(block)
    us_sd, clk_sd = sustained(block_dense)
    del kept
    torch.cuda.empty_cache()
    return {"workload": f"{model} linears, DBF {bpw} bpw, prefill {tokens} tokens (tcgen05 path)",
            "tokens": tokens, "us_per_block": total_us, "tokens_per_s_linears_only": tokens / (total_us * 32 / 1e6),
            "tflops": total_flops / total_us / 1e6, "cublas_fp16_dense_us_per_block": total_dense_us,
            "speedup_vs_cublas_dense": total_dense_us / total_us, "layers": rows,
            "sustained": {"us_per_block": us_s, "tflops": total_flops / us_s / 1e6, "clocks": clk_s,
                          "cublas_fp16_dense_us_per_block": us_sd, "cublas_clocks": clk_sd,
                          "speedup_vs_cublas_dense": us_sd / us_s,
                          "note": "7 layers back to back for ~2 s (power-capped); per-layer rows above are short bursts"}}


def drop_in_call_us(n: int, k: int, m: int, calls: int = 20, replays: int = 10) -> dict:
    """configs[0] through the per-call drop-in API, one fp16 token: forward_device (two GEMV
    launches) and forward_engine (a one-layer engine program, one launch), `calls` calls captured in
    one CUDA graph so the host is out of the loop; device us per call."""
    import torch

    import paper_2505_11076_b200 as P

    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    layer = P.random_device_layer(n, k, m, generator=g)
    x = torch.randn((1, m), generator=g, device="cuda").half()
    y = torch.empty((1, n), dtype=torch.half, device="cuda")
    out = {}
    for api in ("forward_device", "forward_engine"):
        fn = getattr(P, api)
        fn(x, layer, out=y)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(calls):
                fn(x, layer, out=y)
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(replays):
            gr.replay()
        e1.record()
        e1.synchronize()
        out[f"us_per_call_{api}"] = e0.elapsed_time(e1) * 1e3 / (calls * replays)
    return out


def sweep_bench(steps: int):
    """BASELINE configs[3] / [4] at one GPU: the decode engine over Llama-2-70B shapes at 2 bpw
    (batch 1, 4, 16) and Llama-2-13B shapes across bits/weight (batch 1, 4, 8), plus 13B at batch 8
    through the int8 GEMV layer chain and batch 64 through the tcgen05 prefill chain, and the
    single-pass batched kernels at 8 and 16 tokens.  Up to 4 tokens share every MMA of one engine
    launch; larger batches run consecutive launches over groups of 4 (or the batched kernels: one
    weight pass for up to 16).  Every number is a full model step of linears."""
    import torch

    from paper_2505_11076_b200.plan import llama_decode_plan

    rows = []

    def one(model, bpw, batch, engine, prefill=False, batched=False):
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        plan = llama_decode_plan(model, bpw=bpw, batch=batch, generator=g, keep_words=prefill or None)
        plan.buffers[plan.input_buffer].normal_(generator=g)
        if prefill:
            plan.use_prefill()
        elif batched:
            plan.use_batched()
        else:
            plan.use_engine() if engine else plan.use_layer_kernels()
        plan.capture()
        ms = time_graph(plan._graph, steps, 3)
        b = plan.bytes_per_step()
        rows.append({"model": model, "bpw": bpw, "batch": batch,
                     "path": (("engine" if batch <= 4 else f"engine, {-(-batch // 4)} launches of <= 4 tokens")
                              if engine else ("tcgen05 prefill chain" if batch >= 64 or prefill else
                                              "single-pass batched kernels" if batched else
                                              "int8 GEMV chain (pre-quantized batch)")),
                     "ms_per_step": ms, "gbs": b / (ms * 1e-3) / 1e9,
                     "tokens_per_s_linears_only": batch * 1e3 / ms, "layers": len(plan.ops)})
        del plan
        torch.cuda.empty_cache()

    one("llama2-70b", 2.0, 1, True)
    one("llama2-70b", 2.0, 4, True)
    one("llama2-70b", 2.0, 16, True)
    one("llama2-70b", 2.0, 16, False, prefill=True)
    one("llama2-70b", 2.0, 16, False, batched=True)
    one("llama2-70b", 2.0, 8, False, batched=True)
    one("llama2-70b", 2.0, 32, False, batched=True)
    for bpw in (1.0, 1.5, 2.0, 2.3):
        one("llama2-13b", bpw, 1, True)
    one("llama2-7b", 2.0, 4, True)
    one("llama2-7b", 2.0, 4, False, batched=True)
    one("llama2-13b", 1.5, 4, True)
    one("llama2-13b", 1.5, 8, True)
    one("llama2-13b", 1.5, 8, False)
    one("llama2-13b", 1.5, 8, False, prefill=True)
    one("llama2-13b", 1.5, 8, False, batched=True)
    one("llama2-7b", 2.0, 8, False, batched=True)
    one("llama2-13b", 1.5, 64, False)
    # BASELINE configs[4] as specified: a NON-uniform layer-wise k (1.0-2.3 bits/weight across the
    # 280 linears, 1.5 on average, from the reference's greedy allocation -- plan.layerwise_ks)
    from paper_2505_11076_b200.plan import layerwise_ks

    ks = layerwise_ks("llama2-13b", target_bpw=1.5, floor_bpw=1.0, cap_bpw=2.3)
    shp = block_shapes("llama2-13b") * LLAMA["llama2-13b"][3]
    bpws = [k * (n + m) / (n * m) for k, (_, n, m) in zip(ks, shp)]
    for batch in (1, 8, 64):
        g = torch.Generator(device="cuda")
        g.manual_seed(6)
        plan = llama_decode_plan("llama2-13b", batch=batch, generator=g, ks=ks, keep_words=batch >= 64)
        plan.buffers[plan.input_buffer].normal_(generator=g)
        path = plan.default_path()
        {"prefill": plan.use_prefill, "batched": plan.use_batched, "engine": plan.use_engine}[path]()
        plan.capture()
        ms = time_graph(plan._graph, steps, 3)
        b = plan.bytes_per_step()
        rows.append({"model": "llama2-13b", "bpw": "layerwise", "bpw_min": min(bpws), "bpw_max": max(bpws),
                     "bpw_mean_sign_bits": sum(k * (n + m) for k, (_, n, m) in zip(ks, shp)) /
                                           sum(n * m for _, n, m in shp),
                     "batch": batch, "path": path if batch <= 4 or path != "engine" else
                     f"engine, {-(-batch // 4)} launches of <= 4 tokens",
                     "ms_per_step": ms, "gbs": b / (ms * 1e-3) / 1e9,
                     "tokens_per_s_linears_only": batch * 1e3 / ms, "layers": len(plan.ops)})
        del plan
        torch.cuda.empty_cache()
    return rows


def sharded_bench(world: int, rank: int, steps: int, warmup: int, barrier, dist=None):
    """BASELINE configs[3]: the Llama-2-70B linears at 2 bpw with the middle dimension
    k sharded over the `world` GPUs of the run (word-aligned uneven shards).  Per shape and batch:
    the local partial alone, the NCCL path (partial -> NCCL all-reduce -> finalize) and the fused
    path (dbf_forward_allreduce: partials pushed to every peer's symmetric-memory buffer from the
    GEMV2 epilogue); at batch <= 4 also the decode-engine partial, its NCCL path and the engine with
    the same all-reduce fused into its last stage (forward_allreduce_engine).  Each timing replays a CUDA graph over enough distinct layer instances to
    exceed 2x L2; µs are per layer, max over ranks."""
    import torch

    import paper_2505_11076_b200 as P
    from paper_2505_11076_b200 import sharded

    shapes = [("q,o", 8192, 8192, 8192), ("k,v", 1024, 1792, 8192), ("gate,up", 28672, 12736, 8192),
              ("down", 8192, 12736, 28672)]

    def mx(v):
        if dist is None:
            return v
        t = torch.tensor([v], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    rows = []
    for batch in (1, 16):
        for name, n, k, m in shapes:
            k0, k1 = sharded.shard_bounds(k, world)[rank]
            g = torch.Generator(device="cuda")
            g.manual_seed(77 + 1000 * rank)
            bytes_rank = (n * ((k1 - k0 + 7) // 8) + (k1 - k0) * ((m + 7) // 8) + 2 * (n + (k1 - k0) + m)
                          + 2 * batch * (m + n))
            inst = int(min(64, max(2, -(-260_000_000 // bytes_rank))))
            shards = [sharded.DeviceShard.from_device_layer(P.random_device_layer(n, k1 - k0, m, generator=g),
                                                            rank, world, k0) for _ in range(inst)]
            gx = torch.Generator(device="cuda")
            gx.manual_seed(5)  # x is replicated
            X = torch.randn((batch, m), generator=gx, device="cuda").half()
            ar = sharded.FusedAllReduce(n, batch)
            y_n = shards[0].forward(X)
            y_f = ar.forward(shards[0], X)
            torch.cuda.synchronize()
            diff = float(((y_f.float() - y_n.float()).abs().max() / y_n.float().abs().max().clamp_min(1e-30)).item())
            g_p = graph_of(lambda: [s.partial(X) for s in shards])
            g_n = graph_of(lambda: [s.forward(X) for s in shards])
            g_f = graph_of(lambda: [ar.forward(s, X) for s in shards])
            us = [mx(time_graph(gr, steps, warmup, barrier)) * 1e3 / inst for gr in (g_p, g_n, g_f)]
            row = {"layer": name, "n": n, "k": k, "m": m, "batch": batch, "k_shard": [k0, k1],
                   "instances": inst, "us_partial": us[0], "us_nccl_path": us[1], "us_fused": us[2],
                   "us_allreduce_nccl": us[1] - us[0], "us_allreduce_fused": us[2] - us[0],
                   "gbs_per_rank_fused": bytes_rank / (us[2] * 1e-6) / 1e9,
                   "fused_vs_nccl_max_rel_diff": diff}
            if batch <= 4:  # the partial through the decode engine (one launch per shard layer)
                y_e = shards[0].forward(X, engine=True)
                torch.cuda.synchronize()
                row["engine_vs_nccl_max_rel_diff"] = float(
                    ((y_e.float() - y_n.float()).abs().max() / y_n.float().abs().max().clamp_min(1e-30)).item())
                y_fe = ar.forward(shards[0], X, engine=True)
                torch.cuda.synchronize()
                row["fused_engine_vs_engine_nccl_max_rel_diff"] = float(
                    ((y_fe.float() - y_e.float()).abs().max() / y_e.float().abs().max().clamp_min(1e-30)).item())
                g_pe = graph_of(lambda: [s.partial_engine(X) for s in shards])
                g_ne = graph_of(lambda: [s.forward(X, engine=True) for s in shards])
                g_fe = graph_of(lambda: [ar.forward(s, X, engine=True) for s in shards])
                ue = [mx(time_graph(gr, steps, warmup, barrier)) * 1e3 / inst for gr in (g_pe, g_ne, g_fe)]
                row.update({"us_partial_engine": ue[0], "us_nccl_path_engine": ue[1], "us_fused_engine": ue[2],
                            "us_allreduce_nccl_engine": ue[1] - ue[0], "us_allreduce_fused_engine": ue[2] - ue[0],
                            "gbs_per_rank_partial_engine": bytes_rank / (ue[0] * 1e-6) / 1e9,
                            "gbs_per_rank_fused_engine": bytes_rank / (ue[2] * 1e-6) / 1e9})
                del g_pe, g_ne, g_fe
            rows.append(row)
            del g_p, g_n, g_f, shards, ar
            torch.cuda.empty_cache()
    return {"world": world, "model": "llama2-70b", "bpw": 2.0,
            "note": "k-sharded layers, fp16 io; us per layer = max over ranks of graph time / instances",
            "rows": rows}


def sharded_step_bench(world: int, rank: int, steps: int, warmup: int, barrier, dist=None,
                       blocks: int | None = None):
    """BASELINE configs[3] as a decode STEP: every linear of Llama-2-70B (2 bpw, batch 1, decoder
    dataflow of plan.llama_decode_plan) with its middle dimension k sharded over the `world` ranks
    (word-aligned shards).  Per layer the rank's partial runs through the decode engine
    with the one-shot all-reduce fused into its last stage (FusedAllReduce: fp32 partial rows pushed
    into every peer's symmetric-memory buffer over NVLink, y = a * sum in rank order); the NCCL
    arm is the engine partial + an NCCL all-reduce + finalize.  Both are CUDA graphs of the whole
    step; times are max over ranks.  value = the whole model's algorithmic bytes / step time (all
    ranks together stream the model once per step: strong scaling)."""
    import torch

    import paper_2505_11076_b200 as P
    from paper_2505_11076_b200 import sharded

    model = "llama2-70b"
    h, inter, kv, nb = LLAMA[model]
    nb = blocks or nb
    src_of = {"q": "h", "k": "h", "v": "h", "o": "q", "gate": "o", "up": "o", "down": "gate"}
    g = torch.Generator(device="cuda")
    g.manual_seed(77 + 1000 * rank)
    layers, total_bytes = [], 0
    for _ in range(nb):
        for name, n, m in block_shapes(model):
            k = middle_dim(n, m, 2.0)
            k0, k1 = sharded.shard_bounds(k, world)[rank]
            dl = P.random_device_layer(n, k1 - k0, m, generator=g)
            layers.append((name, sharded.DeviceShard.from_device_layer(dl, rank, world, k0)))
            total_bytes += layer_bytes(n, k, m)
    ars = {n: sharded.FusedAllReduce(n, 1) for n in sorted({sh.shard.n for _, sh in layers})}
    gx = torch.Generator(device="cuda")
    gx.manual_seed(5)  # the step input is replicated
    x = (torch.randn((1, h), generator=gx, device="cuda") * 0.5).half()

    def step(fused: bool):
        bufs = {"h": x}
        for name, sh in layers:
            xin = bufs[src_of[name]]
            y = ars[sh.shard.n].forward(sh, xin, engine=True) if fused else sh.forward(xin, engine=True)
            bufs["h" if name == "down" else name] = y
        return bufs["h"]

    def mx(v):
        if dist is None:
            return v
        t = torch.tensor([v], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    y_f, y_n = step(True), step(False)
    torch.cuda.synchronize()
    diff = float(((y_f.float() - y_n.float()).abs().max() / y_n.float().abs().max().clamp_min(1e-30)).item())
    out = {}
    gf = graph_of(lambda: out.__setitem__("y", step(True)))
    ms_f = mx(time_graph(gf, steps, warmup, barrier))
    ms_n = mx(time_graph(graph_of(lambda: step(False)), steps, warmup, barrier))
    # end to end: the step input copied in from pinned host memory and the output read back,
    # inside the timed region
    host_x = x.cpu().pin_memory()
    host_y = torch.empty(out["y"].shape, dtype=out["y"].dtype).pin_memory()
    for _ in range(2):
        x.copy_(host_x, non_blocking=True)
        gf.replay()
        host_y.copy_(out["y"], non_blocking=True)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        x.copy_(host_x, non_blocking=True)
        gf.replay()
        host_y.copy_(out["y"], non_blocking=True)
    e1.record()
    e1.synchronize()
    ms_e = mx(e0.elapsed_time(e1) / steps)
    return {"ms_per_step_e2e": ms_e, "gbs_e2e": total_bytes / (ms_e * 1e-3) / 1e9,
            "h2d_bytes_per_step": host_x.numel() * host_x.element_size(),
            "d2h_bytes_per_step": host_y.numel() * host_y.element_size(),"model": model, "blocks": nb, "layers": len(layers), "world": world, "bytes_per_step": total_bytes,
            "ms_per_step_fused": ms_f, "ms_per_step_nccl": ms_n,
            "gbs_fused": total_bytes / (ms_f * 1e-3) / 1e9, "gbs_nccl": total_bytes / (ms_n * 1e-3) / 1e9,
            "us_per_layer_fused": ms_f * 1e3 / len(layers), "fused_vs_nccl_max_rel_diff": diff,
            "launches_per_step": len(layers)}


def main_sharded(args, world, rank, local, dist, barrier):
    """N > 1 (or --sharded-step): the headline is the k-sharded Llama-2-70B decode step."""
    import torch

    cfg = base_config(args, world)
    clocks = ClockSampler(local).start()
    r = sharded_step_bench(world, rank, args.steps, max(args.warmup, 3), barrier, dist, blocks=args.blocks)
    clk = clocks.stop()
    assert r["bytes_per_step"] == cfg["bytes_per_step"]
    peak, peak_src = peaks()
    ms = r["ms_per_step_fused"]
    per_rank = r["bytes_per_step"] / world
    if rank == 0:
        line = {
            "metric": METRIC, "value": r["gbs_fused"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int8-tc (exact i32 per 256-col chunk) / fp16 io, fp32 all-reduce",
            "data": "synthetic random-init DBF factors of Llama-2-70B shapes, k-sharded (uniform signs, fp16 scales)",
            "config": cfg,
            "detail": {k: v for k, v in r.items() if k != "bytes_per_step"},
            "roofline": {"bound": "hbm", "achieved": per_rank / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": per_rank / (ms * 1e-3) / 1e9 / peak, "traffic": None,
                         "kernel": "engine_kernel<1,*,AR> (one launch per k-sharded layer, all-reduce fused)",
                         "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": {"value": r["gbs_e2e"], "unit": "GB/s", "h2d_bytes_per_step": r["h2d_bytes_per_step"],
                    "d2h_bytes_per_step": r["d2h_bytes_per_step"], "ms_per_step": r["ms_per_step_e2e"]},
            "gpu_launches": r["launches_per_step"] * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    if sharded_headline(args, world):
        return main_sharded(args, world, rank, local, dist, barrier)

    import paper_2505_11076_b200 as P
    from paper_2505_11076_b200.plan import llama_decode_plan

    g = torch.Generator(device="cuda")
    g.manual_seed(1000 + rank)
    plan = llama_decode_plan(args.model, bpw=args.bpw, batch=args.batch, generator=g)
    plan.buffers[plan.input_buffer].normal_(generator=g)
    if not args.layer_kernels:
        plan.use_engine()
    plan.capture()
    bytes_step = plan.bytes_per_step()
    launches = plan.kernel_launches_per_step()
    cfg = base_config(args, world)
    assert cfg["bytes_per_step"] == bytes_step, (cfg["bytes_per_step"], bytes_step)

    clocks = ClockSampler(local).start()
    ms = time_graph(plan._graph, args.steps, max(args.warmup, 3), barrier)
    # keep the GPU loaded ~1.5 s more so the 200 ms clock sampler sees this kernel mix
    t_end = time.time() + 1.5
    while time.time() < t_end:
        for _ in range(20):
            plan._graph.replay()
        torch.cuda.synchronize()
    clk = clocks.stop()

    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * bytes_step / (ms * 1e-3) / 1e9

    # ---- e2e: pinned host input -> plan -> host output, copies inside the timed region --------
    inp = plan.buffers[plan.input_buffer]
    host_x = torch.empty(inp.shape, dtype=inp.dtype, pin_memory=True)
    host_x.copy_(inp.cpu())
    host_y = torch.empty(inp.shape, dtype=inp.dtype, pin_memory=True)
    for _ in range(3):
        inp.copy_(host_x, non_blocking=True)
        plan.replay()
        host_y.copy_(plan.buffers[plan.output_buffer], non_blocking=True)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        inp.copy_(host_x, non_blocking=True)
        plan.replay()
        host_y.copy_(plan.buffers[plan.output_buffer], non_blocking=True)
    e1.record()
    e1.synchronize()
    ms_e2e = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e = {"value": world * bytes_step / (ms_e2e * 1e-3) / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": host_x.numel() * host_x.element_size(),
           "d2h_bytes_per_step": host_y.numel() * host_y.element_size(),
           "ms_per_step": ms_e2e, "api": "paper_2505_11076_b200.plan.DecodePlan.run-equivalent (pinned H2D, graph replay, D2H)"}

    # ---- cuBLAS fp16 GEMV over the same 224 shapes and dataflow -----------------------------
    cublas = None
    if not args.no_cublas:
        step_fn, dense_bytes, weights = build_cublas_chain(plan, torch.float16)
        gc = graph_of(step_fn)
        ms_c = time_graph(gc, args.steps, max(args.warmup, 3), barrier)
        cublas = {"ms_per_step": ms_c, "gbs": dense_bytes / (ms_c * 1e-3) / 1e9,
                  "speedup_dbf_vs_cublas": ms_c / ms, "us_per_layer": ms_c * 1e3 / len(plan.ops)}
        del gc, weights
        torch.cuda.empty_cache()

    peak, peak_src = peaks()
    traffic = None
    tf = ROOT / "profiles" / "roofline_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("traffic_bytes_per_step")
        except Exception:
            traffic = None

    prefill = None
    if rank == 0 and not args.no_prefill:
        prefill = prefill_bench(args.model, 1.0, 2048, max(args.steps // 2, 5), 3)
        bf16_peak, bf16_sus = tensor_peaks()
        prefill["roofline"] = {"bound": "tensor", "achieved": prefill["tflops"], "peak": bf16_peak,
                               "unit": "TFLOP/s", "frac": prefill["tflops"] / bf16_peak,
                               "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: every layer is timed alone; "
                                              "dense fp16 = bf16 rate)"}
        sus = prefill["sustained"]
        sus["roofline"] = {"achieved": sus["tflops"], "peak": bf16_sus, "unit": "TFLOP/s",
                           "frac": sus["tflops"] / bf16_sus,
                           "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS under the power cap)"}

    layers = None
    cfg1 = None
    if rank == 0 and not args.no_layers:
        layers = layer_bench(args.model, args.bpw, max(args.steps // 2, 5), 3)
        # BASELINE configs[0]: one 4096 x 4096 layer, k = 2048 (~1 bit/weight), batch 1 -- the
        # decode engine (isolated: one launch per layer; throughput: independent instances), the
        # per-layer GEMV kernels, cuBLAS fp16 GEMV of the dense layer
        cfg1 = layer_bench(args.model, 1.0, max(args.steps // 2, 5), 3,
                           shapes=[("cfg1 4096x4096 k=2048", 4096, 4096)], layer_kernels=True)["rows"][0]
        cfg1.update(drop_in_call_us(4096, 2048, 4096))

    sweep = None
    if rank == 0 and not args.no_sweep:
        sweep = sweep_bench(max(args.steps // 4, 3))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ref = CpuReference(args.model, args.bpw)
        t = float(np.median([ref.step() for _ in range(args.cpu_reps)]))
        ref.close()
        cpu = {"value": ref.bytes_per_block / t / 1e9, "unit": "GB/s", "cores": ref.procs, "kind": "port",
               "sample": cpu_desc(args.model, args.bpw, ref.procs) + f", median of {args.cpu_reps} blocks",
               "ms_per_layer": t * 1e3 / len(ref.order)}

    # ---- k-sharded 70B layers: NCCL all-reduce vs the all-reduce fused into GEMV2 (all ranks) ---
    # last, after every other number is in hand: a failure here (e.g. a peer-memory problem at
    # N > 1) is reported in the line instead of losing it
    shard = None
    if not args.no_sharded:
        barrier()
        try:
            shard = sharded_bench(world, rank, max(args.steps // 2, 5), 3, barrier, dist)
        except Exception as e:  # noqa: BLE001 - report, keep the headline line
            shard = {"error": f"{type(e).__name__}: {e}"[:300]}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(args.warmup, 3),
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "int8-tc (exact i32 per 256-col chunk) / fp16 io",
            "data": "synthetic random-init DBF factors of Llama-2-7B shapes (uniform signs, fp16 scales)",
            "config": cfg,
            "detail": {
                "us_per_layer": ms * 1e3 / len(plan.ops), "tokens_per_s_linears_only": 1e3 / ms * world,
                "cublas_fp16": cublas,
                "path": "layer kernels (2 GEMV launches per layer)" if args.layer_kernels else
                        "decode engine: 1 persistent kernel per step (bulk-copy sign ring + int8 mma.sync + fp16 LL handoff)",
            },
            "roofline": {"bound": "hbm", "achieved": bytes_step / (ms * 1e-3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bytes_step / (ms * 1e-3) / 1e9 / peak, "traffic": traffic,
                         "kernel": ("gemv_i8_kernel, all launches of the step" if args.layer_kernels else
                                    "engine_kernel (one launch = the whole 224-layer step)"),
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "prefill": prefill,
            "layers": layers,
            "cfg1": cfg1,
            "sweep": sweep,
            "sharded": shard,
            "gpu_launches": launches * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
