"""Kernel timeline of the batched decode chain (a -DDBF_BATCHED_TRACE build:
tools/build_variant.sh btr -DDBF_BATCHED_TRACE; DBF_B200_LIB=tools/_x/btr.so).  One graph replay of
`blocks` decoder blocks; per kernel launch: kind, first CTA start, last return from the grid
dependency wait, last warp end (µs from the first start), and the gap since the latest earlier end.
usage: batched_trace.py [model] [batch] [blocks]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2505_11076_b200 import _lib
from paper_2505_11076_b200.plan import llama_decode_plan

model = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 4
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = torch.Generator(device="cuda")
g.manual_seed(1)
plan = llama_decode_plan(model, bpw=2.0, batch=batch, blocks=blocks, generator=g).use_batched()
plan.buffers[plan.input_buffer].normal_(generator=g)
assert _lib.lib.dbf_batched_debug_reset(1) == 0, "needs a -DDBF_BATCHED_TRACE build"
plan.capture()  # the warm-up pass takes slots [0, n), the captured graph [n, 2n)
for _ in range(3):
    plan.replay()
torch.cuda.synchronize()
assert _lib.lib.dbf_batched_debug_reset(0) == 0
plan.replay()
torch.cuda.synchronize()
buf = np.zeros((8192, 5), dtype=np.uint64)
assert _lib.lib.dbf_batched_debug_trace(buf.ctypes.data, 8192) == 0
used = np.nonzero(buf[:, 3])[0]
t = buf[used].astype(np.float64)
t0 = t[:, 1].min()
names = {1: "quantize", 2: "gemv", 3: "finalize"}
mark = np.where(t[:, 4] > 0, (t[:, 4] - t0) / 1e3, np.nan)
rows = sorted(zip(used, t[:, 0], (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, mark, (t[:, 3] - t0) / 1e3),
              key=lambda r: r[2])
print("slot kind      start   waited  mark    end     dur    gap(start - latest earlier end)")
latest = 0.0
for s, k, st, wt, mk, en in rows:
    print(f"{s:5d} {names.get(int(k), k):9s} {st:7.2f} {wt:7.2f} {mk:7.2f} {en:7.2f} {en - st:6.2f} {st - latest:7.2f}")
    latest = max(latest, en)
span = max(r[5] for r in rows)
print(f"{len(rows)} launches, span {span:.1f} us, {span / blocks:.1f} us per block")
