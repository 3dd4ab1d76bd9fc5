"""LL handoff latency inside the decode engine (needs a DBF_LL_TRACE build with the batch-1
multi-token kernel: tools/build_variant.sh ll -DDBF_B1_OFF -DDBF_LL_TRACE; DBF_B200_LIB=tools/_x/ll.so).
For every run and warp whose first owned chunk is polled from an LL vector: the time from the
LAST publish among the chunk's 16 producer units to the warp having the chunk quantized, and the
time the warp started waiting relative to that publish."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2505_11076_b200.plan import llama_decode_plan

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = torch.Generator(device="cuda")
g.manual_seed(0)
plan = llama_decode_plan(os.environ.get("DBF_MODEL", "llama2-7b"), bpw=2.0, blocks=blocks, generator=g)
plan.buffers[plan.input_buffer].normal_(generator=g)
plan.use_engine()
eng = plan.engine
nr = eng.nruns
nv = eng._prog.nvectors
eng.trace = torch.zeros(4 * nr + nv * 2048 + nr * 16 * 2, dtype=torch.int64, device="cuda")
eng._prog.trace = eng.trace.data_ptr()
import ctypes

from paper_2505_11076_b200 import _lib

for _ in range(3):
    plan._eager()
torch.cuda.synchronize()
rtt = (ctypes.c_ulonglong * 2)()
if hasattr(_lib.lib, "dbf_debug_ll_rtt"):
    _lib.lib.dbf_debug_ll_rtt(rtt)
    print(f"LL poll round trip (load issue -> all lanes checked): mean {rtt[0] / max(rtt[1], 1):.0f} ns over {rtt[1]} polls")
t = eng.trace.cpu().numpy().astype(np.int64)
pub = t[4 * nr: 4 * nr + nv * 2048].reshape(nv, 2048)
arr = t[4 * nr + nv * 2048:].reshape(nr, 16, 2)
lat, waitpre = [], []
recs = eng.records.reshape(-1, 128)
in_vec = recs[:, 100:104].copy().view(np.int32)[:, 0]
in_kind = recs[:, 84:88].copy().view(np.int32)[:, 0]
for i in range(nr):
    if in_kind[i] != 1:
        continue
    for w in range(16):
        st, a = arr[i, w]
        if a == 0:
            continue
        p = pub[in_vec[i], 16 * w: 16 * w + 16]
        p = p[p > 0]
        if p.size == 0:
            continue
        lat.append(a - p.max())
        waitpre.append(p.max() - st)
lat, waitpre = np.array(lat), np.array(waitpre)
busy = waitpre > 0  # the warp was already waiting when the last unit was published
print(f"chunks {lat.size}; waiting-before-publish {busy.mean():.2f}")
for name, d in (("all", lat), ("warp waited", lat[busy]), ("warp late", lat[~busy])):
    if d.size:
        q = np.percentile(d, [10, 50, 90, 99])
        print(f"{name:12s} publish->quantized ns p10 {q[0]:6.0f} p50 {q[1]:6.0f} p90 {q[2]:6.0f} p99 {q[3]:6.0f}")
