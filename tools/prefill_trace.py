"""Per-K-block clock64 trace of CTA (0,0) of the prefill sign GEMM (a DBF_PREFILL_TRACE build)."""
import ctypes
import os
import sys
from pathlib import Path

# needs a -DDBF_PREFILL_TRACE build: tools/build_variant.sh ptr -DDBF_PREFILL_TRACE; DBF_B200_LIB=tools/_x/ptr.so
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2505_11076_b200 as P
from paper_2505_11076_b200 import _lib

T, n, k, m = (int(v) for v in sys.argv[1:5]) if len(sys.argv) >= 5 else (2048, 4096, 2048, 4096)
g = torch.Generator(device="cuda")
g.manual_seed(0)
layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
X = torch.randn((T, m), generator=g, device="cuda").half()
out = torch.empty((T, k), dtype=torch.half, device="cuda")
for _ in range(3):
    _lib.check(_lib.lib.dbf_sign_gemm(X.data_ptr(), T, m, m, layer.B.paired.data_ptr(), layer.B.paired.shape[1], k,
                                      layer.b.data_ptr(), layer.mid.data_ptr(), out.data_ptr(), k,
                                      _lib.stream_ptr()), "gemm")
nkb = (m + 63) // 64
buf = np.zeros(6 * nkb, dtype=np.int64)
f = _lib.lib.dbf_prefill_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert f(buf.ctypes.data, 6 * nkb) == 0
t = buf[: 4 * nkb].reshape(nkb, 4)
mma_go = buf[4 * nkb:5 * nkb]
tma_issue = buf[5 * nkb:]
t0 = t[0, 0]
print("kb  exp_ready  exp_empty  exp_st_done  mma_act  mma_go  tma_issue  (cycles rel. to kb0 exp_ready)")
for kb in range(nkb):
    print(kb, *(int(v - t0) for v in t[kb]), int(mma_go[kb] - t0), int(tma_issue[kb] - t0))
d = np.diff(mma_go)
print("mma_go deltas: median", np.median(d), "mean", d.mean())
lat = t[:, 3] - tma_issue
print("tma issue->mma_act latency: median", np.median(lat[4:]), "min", lat[4:].min())
