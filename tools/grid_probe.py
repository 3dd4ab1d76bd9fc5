"""Batched engine: grid 148 vs grid 37 outputs (bitwise expected).  usage: grid_probe.py BATCH"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2505_11076_b200.plan import llama_decode_plan

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = torch.Generator(device="cuda")
g.manual_seed(40 + batch)
plan = llama_decode_plan("llama2-7b", bpw=2.0, batch=batch, blocks=1, generator=g)
x = torch.randn(plan.buffers[plan.input_buffer].shape, generator=g, device="cuda").half()
outs = {}
for grid in (148, 37):
    plan.buffers[plan.input_buffer].copy_(x)
    plan.use_engine(grid=grid)
    plan._eager()
    torch.cuda.synchronize()
    outs[grid] = plan.buffers[plan.output_buffer].clone()
d = (outs[148].float() - outs[37].float()).abs()
print("batch", batch, "equal", torch.equal(outs[148], outs[37]), "max diff", d.max().item(),
      "n diff per token", [(d[t] > 0).sum().item() for t in range(batch)])
if not torch.equal(outs[148], outs[37]):
    idx = (d > 0).nonzero()
    print("diff at", idx[:4].tolist(), "148:", outs[148][d > 0][:4].tolist(), "37:", outs[37][d > 0][:4].tolist())
    g1 = torch.Generator(device="cuda")
    g1.manual_seed(40 + batch)
    p1 = llama_decode_plan("llama2-7b", bpw=2.0, batch=1, blocks=1, generator=g1).use_engine(grid=148)
    p1.buffers[p1.input_buffer].copy_(x[:1])
    p1._eager()
    torch.cuda.synchronize()
    o1 = p1.buffers[p1.output_buffer]
    print("batch-1 engine token 0 == grid148:", torch.equal(o1, outs[148][:1]), "== grid37:", torch.equal(o1, outs[37][:1]))
    for grid in (148, 37, 64, 100, 147):
        plan.buffers[plan.input_buffer].copy_(x)
        plan.use_engine(grid=grid)
        plan._eager()
        torch.cuda.synchronize()
        o = plan.buffers[plan.output_buffer]
        print("grid", grid, "token0 == batch-1:", torch.equal(o[:1], o1))
