"""Per-warp critical-path breakdown of the decode engine (needs the DBF_ENGINE_WARP_TRACE build:
tools/build_variant.sh wt -DDBF_ENGINE_WARP_TRACE, then DBF_B200_LIB=tools/_x/wt.so).

For every stage of block 1 (the second block, steady state): over all CTAs' runs of the stage,
median / max of each phase per warp (ns): pieces wait, quantize of chunk j, compute of chunk j,
barrier wait, finalize; plus the CTA's start relative to the previous stage's last publish."""
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
nr = eng.nruns
eng.trace = torch.zeros(4 * nr + nr * 16 * 17, dtype=torch.int64, device="cuda")
eng._prog.trace = eng.trace.data_ptr()
for _ in range(3):
    plan._eager()
torch.cuda.synchronize()
t = eng.trace.cpu().numpy().astype(np.int64)
tr = t[: 4 * nr].reshape(nr, 4)
wt = t[4 * nr:].reshape(nr, 16, 17)
lv = levels_of(plan.ops, plan.input_buffer)
seg_stage = []
for i in range(len(plan.ops)):
    seg_stage += [2 * lv[i], 2 * lv[i] + 1]
stage = np.array([seg_stage[s] for s in eng._flat[:, 0]])
names = {}
for i, op in enumerate(plan.ops):
    names.setdefault(2 * lv[i], []).append(op.name + ".B")
    names.setdefault(2 * lv[i] + 1, []).append(op.name + ".A")
last_pub = {s: tr[stage == s, 3].max() for s in set(stage)}
nst = max(stage) + 1
per_block = nst // blocks
print("phase ns, median/max over (run, warp); q_j/c_j = quantize/compute of the warp's j-th chunk")
for s in range(per_block, 2 * per_block):
    runs = np.where(stage == s)[0]
    prev = last_pub.get(s - 1, tr[:, 0].min())
    W = wt[runs]  # (runs, 16, 10)

    def ph(a, b):
        d = (W[:, :, b] - W[:, :, a]).astype(np.float64)
        ok = (W[:, :, a] > 0) & (W[:, :, b] > 0)
        d = d[ok]
        return f"{int(np.median(d)):5d}/{int(d.max()):5d}" if d.size else "    -/    -"

    start = W[:, :, 0][W[:, :, 0] > 0] - prev
    cols = [ph(0, 1), ph(1, 2), ph(2, 5), ph(5, 3), ph(3, 6), ph(6, 4), ph(4, 7)]
    last_c = np.where(W[:, :, 7] > 0, W[:, :, 7], np.where(W[:, :, 6] > 0, W[:, :, 6], W[:, :, 5]))
    bar = (W[:, :, 8] - last_c)
    fin_all = (W[:, :, 9] - W[:, :, 8])
    nun = eng._flat[runs, 2]
    act = np.arange(16)[None, :] < nun[:, None]
    fa, fi = fin_all[act], fin_all[~act]
    fin = fa
    idle = f" idle-fin {int(np.median(fi)) if fi.size else -1}"
    print(f"{s:3d} {','.join(names[s]):22s} runs {len(runs):4d} start {int(np.median(start)):6d}/{int(start.max()):6d} "
          f"pieces {cols[0]} q0 {cols[1]} c0 {cols[2]} q1 {cols[3]} c1 {cols[4]} q2 {cols[5]} c2 {cols[6]} "
          f"bar {int(np.median(bar))}/{int(bar.max())} fin {int(np.median(fin))}/{int(fin.max())} "
          f"stage {last_pub[s] - prev}{idle}")

print("\ncritical CTA per stage (the last publisher): its phases relative to the previous stage's last publish (ns)")
cta_of_run = np.searchsorted(eng._offsets, np.arange(nr), side="right") - 1
prev_crit = None
for s in range(per_block, 2 * per_block):
    runs = np.where(stage == s)[0]
    prev = last_pub.get(s - 1, tr[:, 0].min())
    j = runs[np.argmax(tr[runs, 3])]
    c = cta_of_run[j]
    W = wt[j]
    act = W[:, 0] > 0
    q0 = W[act, 2].max() - prev
    lastc = np.max(np.where(W[act, 7] > 0, W[act, 7], np.where(W[act, 6] > 0, W[act, 6], W[act, 5]))) - prev
    print(f"{s:3d} {','.join(names[s]):22s} cta {c:3d} (prev crit {prev_crit}) runs-in-stage {np.sum(cta_of_run[runs] == c)} "
          f"start {W[act, 0].min() - prev:6d} pieces {W[act, 1].max() - prev:6d} q0(max warp) {q0:6d} "
          f"compute-done {lastc:6d} bar {W[act, 8].max() - prev:6d} pub {tr[j, 3] - prev:6d}")
    if batch > 1:
        Wa = W[act]
        print(f"      tokens: entry med {int(np.median(Wa[:, 10] - prev))} pair0 polled {int(np.median(Wa[:, 11] - prev))} "
              f"(polls max {Wa[:, 12].max()}) emitted {int(np.median(Wa[:, 13] - prev))} pair1 polled {int(np.median(Wa[:, 14] - prev))} "
              f"(polls max {Wa[:, 15].max()}) emitted {int(np.median(Wa[:, 16] - prev))} max {int((Wa[:, 16] - prev).max())}")
        prev_crit = c
        continue
    ws = int(np.argmax(W[act, 2]))
    print(f"      slowest-q0 warp {ws}: poll start {W[act, 10][ws] - prev} success {W[act, 11][ws] - prev} polls {W[act, 12][ws]}; "
          f"all warps: poll start med {int(np.median(W[act, 10] - prev))} success med {int(np.median(W[act, 11] - prev))} "
          f"max {int((W[act, 11] - prev).max())} polls med {int(np.median(W[act, 12]))} max {W[act, 12].max()}")
    prev_crit = c
