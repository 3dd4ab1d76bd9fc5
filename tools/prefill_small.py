"""Small-batch prefill timing: the 7 Llama-2-13B linears at 1.5 bpw, T tokens (default 64), one CUDA
graph per layer replayed; prints us per layer.  usage: prefill_small.py [T] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2505_11076_b200 as P
from paper_2505_11076_b200.budget import middle_dim
from paper_2505_11076_b200.plan import block_shapes

T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = torch.Generator(device="cuda")
g.manual_seed(0)
out = []
for name, n, m in block_shapes("llama2-13b"):
    k = middle_dim(n, m, 1.5, 32)
    L = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    X = torch.randn((T, m), generator=g, device="cuda").half()
    Y = torch.empty((T, n), dtype=torch.half, device="cuda")
    P.forward_prefill(X, L, out=Y)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        P.forward_prefill(X, L, out=Y)
        with torch.cuda.graph(gr, stream=s):
            P.forward_prefill(X, L, out=Y)
    torch.cuda.synchronize()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    fl = 2 * T * k * (n + m)
    out.append(f"{name} n={n} k={k} m={m}: {us:.1f} us {fl / us / 1e6:.0f} TF/s")
print(f"T={T}: " + " | ".join(out))
