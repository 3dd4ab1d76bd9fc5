"""Per-CTA timeline of one prefill sign GEMM (a DBF_PREFILL_TRACE build): when each CTA started and
ended (globaltimer), and its setup / first MMA / last commit / accumulator / epilogue stamps
(clock64 relative to the CTA's start).  Shows wave quantization and the per-tile fixed costs.

  tools/build_variant.sh ptr -DDBF_PREFILL_TRACE
  DBF_B200_LIB=tools/_x/ptr.so python tools/prefill_ctas.py T rows K   (e.g. 2048 2048 4096)
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2505_11076_b200 as P
from paper_2505_11076_b200 import _lib

T, rows, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (2048, 2048, 4096)
kscale = len(sys.argv) < 5 or sys.argv[4] != "noks"
g = torch.Generator(device="cuda")
g.manual_seed(0)
pitch = ((K + 31) // 32 + 3) // 4 * 4
words = torch.randint(0, 2**31, (rows, pitch), generator=g, device="cuda", dtype=torch.int32)
X = torch.randn((T, K), generator=g, device="cuda").half()
ks = (torch.rand(K, generator=g, device="cuda") + 0.5).half()
rs = (torch.rand(rows, generator=g, device="cuda") + 0.5).half()
out = torch.empty((T, rows), dtype=torch.half, device="cuda")


def run():
    _lib.check(_lib.lib.dbf_sign_gemm(X.data_ptr(), T, K, K, words.data_ptr(), pitch, rows,
                                      ks.data_ptr() if kscale else None, rs.data_ptr(), out.data_ptr(), rows,
                                      _lib.stream_ptr()), "gemm")


for _ in range(5):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
print(f"T={T} rows={rows} K={K}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per launch "
      f"({2 * T * rows * K / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e12:.0f} TF/s)")
ntiles = ((rows + 127) // 128) * ((T + 255) // 256)
f = _lib.lib.dbf_prefill_debug_ctas
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(16 * ntiles, dtype=np.int64)
assert f(buf.ctypes.data, 16 * ntiles) == 0
c = buf.reshape(ntiles, 16)
t0 = c[:, 0].min()
start = (c[:, 0] - t0) / 1e3
end = (c[:, 1] - t0) / 1e3
clk0 = c[:, 4]
ghz = 1.965
rel = lambda i: (c[:, i] - clk0) / ghz / 1e3  # noqa: E731
print(f"kernel span {end.max():.1f} us; CTAs {ntiles}; SMs used {len(set(c[:, 3]))}")
order = np.argsort(start)
print("cta  sm  start   end   dur | setup firstMMA lastCommit accSeen staged barrier stored exit (us after CTA start)")
for i in list(order[:6]) + list(order[-6:]):
    print(f"{i:4d} {c[i, 3]:3d} {start[i]:6.1f} {end[i]:6.1f} {end[i] - start[i]:5.1f} | " +
          " ".join(f"{rel(j)[i]:6.2f}" for j in (5, 6, 7, 8, 10, 11, 12, 9)))
for name, j in (("setup", 5), ("first MMA", 6), ("last commit", 7), ("acc seen", 8), ("staged", 10),
                ("barrier", 11), ("stored", 12), ("exit", 9)):
    v = rel(j)
    print(f"  {name:12s} median {np.median(v):6.2f}  p90 {np.percentile(v, 90):6.2f} us")
dur = end - start
print(f"  CTA duration median {np.median(dur):.2f} us; K loop (first MMA -> last commit) median "
      f"{np.median(rel(7) - rel(6)):.2f} us")
# waves: start-time clusters
st = np.sort(start)
gaps = np.where(np.diff(st) > 2.0)[0]
print("  wave starts (us):", [round(st[0], 1)] + [round(st[i + 1], 1) for i in gaps])
