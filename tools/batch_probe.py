"""Run a 1-block 7B engine at a given batch and grid once (hang / correctness probe).
usage: batch_probe.py BATCH GRID"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2505_11076_b200.plan import llama_decode_plan

batch, grid = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda")
g.manual_seed(44)
plan = llama_decode_plan("llama2-7b", bpw=2.0, batch=batch, blocks=1, generator=g)
x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
plan.buffers[plan.input_buffer].copy_(x)
plan.use_engine(grid=grid)
print("runs", plan.engine.nruns, "smem", plan.engine.smem_bytes, flush=True)
plan._eager()
torch.cuda.synchronize()
print("ok", batch, grid, plan.buffers[plan.output_buffer].float().abs().mean().item(), flush=True)
