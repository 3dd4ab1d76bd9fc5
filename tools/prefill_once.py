"""Run one Llama-2-7B-shape prefill layer a few times (for ncu captures): both the one-launch layer
kernel (forward_prefill) and the two per-tile launches.  python tools/prefill_once.py [q|gate|down] [T]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import torch

import paper_2505_11076_b200 as P
from test_gpu_prefill import _two_launch

SH = {"q": (4096, 2048, 4096), "gate": (11008, 2976, 4096), "down": (4096, 2976, 11008)}
n, k, m = SH[sys.argv[1] if len(sys.argv) > 1 else "gate"]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
g = torch.Generator(device="cuda")
g.manual_seed(0)
dl = P.random_device_layer(n, k, m, generator=g, keep_words=True)
X = torch.randn((T, m), generator=g, device="cuda").half()
for _ in range(3):
    P.forward_prefill(X, dl)
    _two_launch(X, dl)
torch.cuda.synchronize()
print("ok")
