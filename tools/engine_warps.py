"""Per-warp clock64 breakdown of CTA 0's runs (debug stamps: start, first chunk quantized,
compute done, cycles spent waiting for weight pieces)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2505_11076_b200.plan import llama_decode_plan

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 1
indep = len(sys.argv) > 2 and sys.argv[2] == "indep"
g = torch.Generator(device="cuda")
g.manual_seed(0)
plan = llama_decode_plan("llama2-7b", bpw=2.0, blocks=blocks, generator=g)
plan.buffers[plan.input_buffer].normal_(generator=g)
if indep:
    ins = {}
    for op in plan.ops:
        m = plan.layers[op.layer].m_dim
        if m not in ins:
            plan.buffers.append(torch.randn((1, m), device="cuda").half())
            ins[m] = len(plan.buffers) - 1
        op.src = ins[m]
        plan.buffers.append(torch.zeros((1, plan.layers[op.layer].n), device="cuda").half())
        op.dst = len(plan.buffers) - 1
plan.use_engine()
eng = plan.engine
nr = eng.nruns
runs0 = eng._offsets[1] - eng._offsets[0]
eng.trace = torch.zeros(4 * nr + 16 * 4 * 64 + runs0 * 16 * 4 + 64, dtype=torch.int64, device="cuda")
eng._prog.trace = eng.trace.data_ptr()
eng._prog.pad = 4 * nr
for _ in range(3):
    plan._eager()
torch.cuda.synchronize()
t = eng.trace.cpu().numpy()
d = t[4 * nr: 4 * nr + runs0 * 64].reshape(runs0, 16, 4)
qd = t[4 * nr + 16 * 4 * 64: 4 * nr + 16 * 4 * 64 + runs0 * 64].reshape(runs0, 16, 4)
base = d[0, :, 0].min()
for j in range(runs0):
    seg, rb, n = eng._flat[j]
    s0 = d[j, :, 0] - base
    q = d[j, :, 1] - d[j, :, 0]
    c = d[j, :, 2] - d[j, :, 1]
    w = d[j, :, 3]
    print(f"run {j:2d} seg {seg:3d} n {n}: start {s0.min():7d}..{s0.max():7d}  quant(first) med {int(np.median(q)):6d} max {q.max():6d}"
          f"  compute med {int(np.median(c)):6d} max {c.max():6d}")
    ok = qd[j, :, 0] > 0
    if ok.any():
        a = (qd[j, ok, 0] - d[j, ok, 0]); b = qd[j, ok, 1] - qd[j, ok, 0]; cc = qd[j, ok, 2] - qd[j, ok, 1]; e = d[j, ok, 1] - qd[j, ok, 2]
        print(f"      quantize: loads {int(np.median(a))}  max-reduce {int(np.median(b))}  digits {int(np.median(cc))}  tail {int(np.median(e))}")
