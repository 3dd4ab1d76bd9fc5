"""7B chain ms/step at several engine grid sizes (one CTA per SM; fewer CTAs = more units each)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2505_11076_b200.plan import llama_decode_plan

sys.argv += []
g = torch.Generator(device="cuda")
g.manual_seed(0)
p = llama_decode_plan("llama2-7b", bpw=2.0, generator=g)
p.buffers[p.input_buffer].normal_(generator=g)
out = []
for grid in (148, 146, 144, 140, 136, 128):
    p.use_engine(grid=grid)
    p.capture()
    for _ in range(3):
        p.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        p.replay()
    e1.record()
    e1.synchronize()
    out.append(f"{grid}: {e0.elapsed_time(e1) / 20 * 1e3:.1f}us")
print(" | ".join(out))
