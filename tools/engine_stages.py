"""Per-stage critical-path breakdown of the decode engine from the per-run %globaltimer trace.

For each stage S: when its last unit was published (max finalize stamp), and for its runs the
spread of 'first input chunk ready' (warp 0), 'warp 0 compute done' and 'finalized' stamps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2505_11076_b200.engine import levels_of
from paper_2505_11076_b200.plan import llama_decode_plan

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 2
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = torch.Generator(device="cuda")
g.manual_seed(0)
import os
plan = llama_decode_plan(os.environ.get("DBF_MODEL", "llama2-7b"), bpw=2.0, blocks=blocks, batch=batch, generator=g)
plan.buffers[plan.input_buffer].normal_(generator=g)
plan.use_engine()
eng = plan.engine
eng.enable_trace()
for _ in range(3):
    plan._eager()
torch.cuda.synchronize()
tr = eng.trace.cpu().numpy().astype(np.int64)
t0 = tr[:, 0].min()
tr = tr - t0
lv = levels_of(plan.ops, plan.input_buffer)
seg_stage = []
for i in range(len(plan.ops)):
    seg_stage += [2 * lv[i], 2 * lv[i] + 1]
stage = np.array([seg_stage[s] for s in eng._flat[:, 0]])
prev_done = 0
print("stage  names         last_pub  | ready min/med/max   | w0done med/max | fin med/max  (us; 'lag' = ready_med - prev last_pub)")
names = {}
for i, op in enumerate(plan.ops):
    names.setdefault(2 * lv[i], []).append(op.name + ".B")
    names.setdefault(2 * lv[i] + 1, []).append(op.name + ".A")
for s in sorted(set(stage)):
    m = stage == s
    r, w, f = tr[m, 1] / 1e3, tr[m, 2] / 1e3, tr[m, 3] / 1e3
    print(f"{s:4d}  {','.join(names[s])[:14]:14s} {f.max():8.2f} | {r.min():6.2f} {np.median(r):6.2f} {r.max():6.2f} | "
          f"{np.median(w):6.2f} {w.max():6.2f} | {np.median(f):6.2f} {f.max():6.2f}  lag {np.median(r) - prev_done:5.2f}")
    prev_done = f.max()
