"""Per-layer time of the batched decode GEMV (dbf_forward) for batch 1..16 at a 13B/70B shape."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2505_11076_b200 as P

n, k, m = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (5120, 3840, 5120)
g = torch.Generator(device="cuda")
g.manual_seed(0)
layer = P.random_device_layer(n, k, m, generator=g)
for batch in (1, 2, 4, 8, 16):
    X = torch.randn((batch, m), generator=g, device="cuda").half()
    Y = torch.empty((batch, n), dtype=torch.half, device="cuda")
    for _ in range(3):
        P.forward_device(X, layer, out=Y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        P.forward_device(X, layer, out=Y)
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(f"{n}x{m} k={k} batch {batch:2d}: {us:7.1f} us/layer  {layer.bytes_logical(batch) / us / 1e3:7.1f} GB/s")
