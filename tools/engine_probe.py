"""Probe the decode engine's limits (not a benchmark of record; bench.py is).

  chain  : the real 7B decode dataflow (128 dependent levels)
  indep  : the same 224 layers, every op reading the step input -> 2 stages total
           (streaming capacity of the engine without inter-layer waits)
  layers : per-layer kernels (dbf_forward) for the chain
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2505_11076_b200.plan import llama_decode_plan


def timeit(plan, steps=20):
    plan.capture()
    for _ in range(3):
        plan.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        plan.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    plan = llama_decode_plan(model, bpw=2.0, generator=g)
    plan.buffers[plan.input_buffer].normal_(generator=g)
    nbytes = plan.bytes_per_step()
    for grid in (148, 132):
        ms = timeit(plan.use_engine(grid=grid))
        print(f"chain  grid={grid}: {ms:.3f} ms/step {nbytes/ms/1e6:.0f} GB/s  {ms*1e3/len(plan.ops):.2f} us/layer", flush=True)
    # independent: every op reads the step input, writes a scratch buffer
    scratch = len(plan.buffers)
    for op in plan.ops:
        plan.buffers.append(torch.zeros((1, plan.layers[op.layer].n), dtype=torch.float16, device="cuda"))
    saved = [(op.src, op.dst) for op in plan.ops]
    widths = {plan.layers[op.layer].m_dim for op in plan.ops}
    inputs = {w: torch.randn((1, w), device="cuda").half() for w in widths}
    for w, t in inputs.items():
        plan.buffers.append(t)
    wid = {w: len(plan.buffers) - len(inputs) + i for i, w in enumerate(inputs)}
    for i, op in enumerate(plan.ops):
        op.src = wid[plan.layers[op.layer].m_dim]
        op.dst = scratch + i
    plan.input_buffer = op.src
    plan.output_buffer = op.dst
    ms = timeit(plan.use_engine())
    print(f"indep  : {ms:.3f} ms/step {nbytes/ms/1e6:.0f} GB/s  {ms*1e3/len(plan.ops):.2f} us/layer", flush=True)
    for op, (s, d) in zip(plan.ops, saved):
        op.src, op.dst = s, d


if __name__ == "__main__":
    main()
