"""Batched decode steps (CUDA graph, ms per step) on the configs[3] / [4] shapes, for A/B of batched
kernel variants (DBF_B200_LIB=...).  python tools/batched_sweep.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2505_11076_b200.plan import llama_decode_plan

for model, bpw, batch in (("llama2-70b", 2.0, 16), ("llama2-70b", 2.0, 8), ("llama2-13b", 1.5, 8), ("llama2-7b", 2.0, 4)):
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    plan = llama_decode_plan(model, bpw=bpw, batch=batch, generator=g, blocks=8 if "70b" in model else None)
    plan.buffers[plan.input_buffer].normal_(generator=g)
    plan.use_batched()
    plan.capture()
    for _ in range(3):
        plan.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.replay()
    e1.record()
    e1.synchronize()
    nb = 8 if "70b" in model else None
    print(f"{model} {bpw} bpw batch {batch}{' (8 blocks)' if nb else ''}: {e0.elapsed_time(e1) / 10:.3f} ms per step")
    del plan
    torch.cuda.empty_cache()
