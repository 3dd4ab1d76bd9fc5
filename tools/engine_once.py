"""Run the 7B decode engine a few times (for ncu: the last launch is the profiled one).
usage: engine_once.py BLOCKS RUNS [indep] (ENGINE_BATCH=4 for a 4-token step)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2505_11076_b200.plan import llama_decode_plan

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 2
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
indep = len(sys.argv) > 3 and sys.argv[3] == "indep"
g = torch.Generator(device="cuda")
g.manual_seed(0)
import os
plan = llama_decode_plan(os.environ.get("DBF_MODEL", "llama2-7b"), bpw=2.0, blocks=blocks, generator=g, batch=int(os.environ.get("ENGINE_BATCH", "1")))
plan.buffers[plan.input_buffer].normal_(generator=g)
if indep:  # every op reads a fixed external input of its width, writes its own scratch buffer
    ins = {}
    for op in plan.ops:
        m = plan.layers[op.layer].m_dim
        if m not in ins:
            plan.buffers.append(torch.randn((1, m), device="cuda").half())
            ins[m] = len(plan.buffers) - 1
        op.src = ins[m]
        plan.buffers.append(torch.zeros((1, plan.layers[op.layer].n), device="cuda").half())
        op.dst = len(plan.buffers) - 1
    plan.input_buffer, plan.output_buffer = plan.ops[0].src, plan.ops[-1].dst
plan.use_engine()
for _ in range(runs):
    plan._eager()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); plan._eager(); e1.record(); e1.synchronize()
print(f"ok {e0.elapsed_time(e1)*1e3:.1f} us  {plan.bytes_per_step()/e0.elapsed_time(e1)/1e6:.0f} GB/s")
