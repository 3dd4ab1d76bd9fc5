"""Per-call latency of the drop-in per-layer forward on BASELINE configs[0] (4096 x 4096, k = 2048,
batch 1) and the 7B shapes: forward_device (dbf_forward: two int8 tensor-core GEMV launches) and
forward_engine (a one-layer decode-engine program: one launch); N calls captured in one CUDA graph,
device time per call.  python tools/forward_latency.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2505_11076_b200 as P

g = torch.Generator(device="cuda")
g.manual_seed(0)
for name, n, k, m in (("cfg1", 4096, 2048, 4096), ("7B q 2bpw", 4096, 4096, 4096), ("7B gate", 11008, 5952, 4096),
                      ("7B down", 4096, 5952, 11008)):
    dl = P.random_device_layer(n, k, m, generator=g)
    x = torch.randn((1, m), generator=g, device="cuda").half()
    y = torch.empty((1, n), dtype=torch.half, device="cuda")
    for api in ("forward_device", "forward_engine"):
        fn = getattr(P, api)
        fn(x, dl, out=y)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(20):
                fn(x, dl, out=y)
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            gr.replay()
        e1.record()
        e1.synchronize()
        print(f"{name:10s} {api:15s} {e0.elapsed_time(e1) / 200 * 1e3:7.2f} us per call")
