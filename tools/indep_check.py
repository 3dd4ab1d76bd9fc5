"""Engine over the 224 Llama-2-7B DBF layers with NO dependency between layers (every op reads
the step input of its width, writes its own output): the GEMV kernel's bandwidth when it is not
bound by the chain's per-stage latency."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2505_11076_b200.plan import DecodePlan, PlanOp, llama_decode_plan

g = torch.Generator(device="cuda")
g.manual_seed(0)
chain = llama_decode_plan("llama2-7b", bpw=2.0, generator=g)
bufs = [torch.randn((1, 4096), generator=g, device="cuda").half(), torch.randn((1, 11008), generator=g, device="cuda").half()]
ops = []
for op in chain.ops:
    m = chain.layers[op.layer].m_dim
    n = chain.layers[op.layer].n
    bufs.append(torch.zeros((1, n), device="cuda").half())
    ops.append(PlanOp(op.layer, 0 if m == 4096 else 1, len(bufs) - 1, op.name))
plan = DecodePlan(chain.layers, ops, bufs, input_buffer=0, output_buffer=len(bufs) - 1)
t0 = time.time()
plan.use_engine()
plan.capture()
for _ in range(3):
    plan.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    plan.replay()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 20
b = plan.bytes_per_step()
print(f"independent layers: {ms:.3f} ms/step, {b / ms / 1e6:.0f} GB/s, {len(ops)} layers")

if len(sys.argv) > 1 and sys.argv[1] == "trace":  # needs DBF_B200_LIB=tools/_x/wt.so
    import numpy as np

    eng = plan.engine
    nr = eng.nruns
    eng.trace = torch.zeros(4 * nr + nr * 16 * 13, dtype=torch.int64, device="cuda")
    eng._prog.trace = eng.trace.data_ptr()
    plan._graph = None
    for _ in range(3):
        plan._eager()
    torch.cuda.synchronize()
    t = eng.trace.cpu().numpy().astype(np.int64)
    W = t[4 * nr:].reshape(nr, 16, 13)
    ok = W[:, :, 0] > 0

    def med(a, b):
        d = (W[:, :, b] - W[:, :, a])[ok & (W[:, :, b] > 0) & (W[:, :, a] > 0)]
        return int(np.median(d)), int(np.percentile(d, 90))

    tr = t[:4 * nr].reshape(nr, 4)
    runlen = tr[:, 3] - tr[:, 0]
    gaps = []
    offs = eng._offsets
    for c in range(len(offs) - 1):
        r = np.arange(offs[c], offs[c + 1])
        if len(r) > 1:
            gaps += list(tr[r[1:], 0] - tr[r[:-1], 3])
    print("per run (ns, median/p90): start->pieces", med(0, 1), "pieces->q0", med(1, 2), "q0->c0", med(2, 5),
          "c0->bar", med(5, 8), "bar->fin", med(8, 9))
    print("run length median", int(np.median(runlen)), "p90", int(np.percentile(runlen, 90)),
          "gap between runs median", int(np.median(gaps)), "units/run", float(np.mean(eng._flat[:, 2])))
