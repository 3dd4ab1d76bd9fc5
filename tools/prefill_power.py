"""Clock / power while the prefill paths run back to back (nvidia-smi sampled every 50 ms):
is the one-launch kernel's slower K loop (in ns) a lower SM clock under its denser tensor load?
  python tools/prefill_power.py [q|gate|down]"""
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2505_11076_b200 as P

SH = {"q": (4096, 2048, 4096), "gate": (11008, 2976, 4096), "down": (4096, 2976, 11008)}
name = sys.argv[1] if len(sys.argv) > 1 else "gate"
n, k, m = SH[name]
T = 2048
g = torch.Generator(device="cuda")
g.manual_seed(0)
dl = P.random_device_layer(n, k, m, generator=g, keep_words=True)
X = torch.randn((T, m), generator=g, device="cuda").half()
Y = torch.empty((T, n), dtype=torch.half, device="cuda")
for path in ("two_launches", "one_launch", "two_launches", "one_launch"):
    for _ in range(5):
        P.forward_prefill(X, dl, out=Y, path=path)
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_end = time.time() + 2.0
    iters = 0
    e0.record()
    while time.time() < t_end:
        for _ in range(50):
            P.forward_prefill(X, dl, out=Y, path=path)
        iters += 50
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    smi.terminate()
    lines = [l.split(",") for l in smi.stdout.read().strip().splitlines()[2:-1]]
    mhz = sorted(float(l[0]) for l in lines)
    pw = sorted(float(l[1]) for l in lines)
    reasons = sorted({l[2].strip() for l in lines})
    us = e0.elapsed_time(e1) / iters * 1e3
    print(f"{name} {path:13s}: {us:7.1f} us/layer ({2.0 * T * k * (n + m) / us / 1e6:6.0f} TF/s)  SM clock median "
          f"{mhz[len(mhz) // 2]:.0f} MHz (min {mhz[0]:.0f})  power median {pw[len(pw) // 2]:.0f} W  reasons {reasons}")
