"""A/B timing of the decode engine build in use (DBF_B200_LIB selects a variant .so):
graph-replayed ms/step and GB/s for the 7B chain, the 7B layers without dependencies, a
13B chain and 16 blocks of the 70B chain.  usage: ab.py [label]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2505_11076_b200.plan import DecodePlan, PlanOp, llama_decode_plan


def timed(plan, steps=20):
    plan.capture()
    for _ in range(3):
        plan.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(steps):
            plan.replay()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / steps)
    return best, plan.bytes_per_step() / best / 1e6


def indep(chain):
    bufs = [torch.randn((1, 4096), device="cuda").half(), torch.randn((1, 11008), device="cuda").half()]
    ops = []
    for op in chain.ops:
        L = chain.layers[op.layer]
        bufs.append(torch.zeros((1, L.n), device="cuda").half())
        ops.append(PlanOp(op.layer, 0 if L.m_dim == 4096 else 1, len(bufs) - 1, op.name))
    return DecodePlan(chain.layers, ops, bufs, input_buffer=0, output_buffer=len(bufs) - 1)


g = torch.Generator(device="cuda")
g.manual_seed(0)
out = [sys.argv[1] if len(sys.argv) > 1 else os.environ.get("DBF_B200_LIB", "default")]
batch = int(os.environ.get("AB_BATCH", "1"))
for name, model, blocks in [("7b", "llama2-7b", None), ("13b", "llama2-13b", None), ("70b/16", "llama2-70b", 16)]:
    p = llama_decode_plan(model, bpw=2.0, blocks=blocks, batch=batch, generator=g)
    p.buffers[p.input_buffer].normal_(generator=g)
    ms, gbs = timed(p.use_engine())
    out.append(f"{name} {ms * 1e3:7.1f}us {gbs:6.0f}GB/s")
    if model == "llama2-7b" and batch == 1:
        ms, gbs = timed(indep(p).use_engine())
        out.append(f"7b-indep {ms * 1e3:7.1f}us {gbs:6.0f}GB/s")
    del p
    torch.cuda.empty_cache()
print(" | ".join(out), flush=True)
