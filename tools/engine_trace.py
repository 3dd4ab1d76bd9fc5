"""Run the 7B decode chain once with per-run %globaltimer stamps and summarize where time goes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2505_11076_b200.plan import llama_decode_plan

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = torch.Generator(device="cuda")
g.manual_seed(0)
plan = llama_decode_plan("llama2-7b", bpw=2.0, blocks=blocks, generator=g)
plan.buffers[plan.input_buffer].normal_(generator=g)
plan.use_engine()
eng = plan.engine
eng.enable_trace()
for _ in range(3):
    plan._eager()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); plan._eager(); e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1)
print(f"blocks={blocks} layers={len(plan.ops)} kernel {ms*1e3:.1f} us  {plan.bytes_per_step()/ms/1e6:.0f} GB/s")
tr = eng.trace.cpu().numpy().astype(np.int64)
off = eng._offsets
t0 = tr[tr[:, 0] > 0, 0].min()
tr = tr - t0
prep = tr[:, 1] - tr[:, 0]
wait_w = np.maximum(tr[:, 2] - tr[:, 1], 0)
comp = tr[:, 3] - np.maximum(tr[:, 2], tr[:, 1])
print(f"runs={len(tr)}  prep mean {prep.mean():.0f} ns  weights-wait mean {wait_w.mean():.0f}  compute mean {comp.mean():.0f} max {comp.max()}")
for c in (0, 1, 77):
    lo, hi = off[c], off[c + 1]
    print(f"CTA {c}: runs {hi-lo}")
    for i in range(lo, min(hi, lo + 16)):
        seg, rb, n = eng._flat[i]
        print(f"   r{i-lo:3d} seg {seg:4d} rb {rb:4d} n {n:2d}  start {tr[i,0]:8d}  ready {tr[i,1]:8d}  wts {tr[i,2]:8d}  done {tr[i,3]:8d}")
