"""A/B of the prefill layer paths on the Llama-2-7B shapes at 1 bpw: forward_prefill (one persistent
launch per layer for T > 256) against two per-tile sign GEMM launches, CUDA events, TF/s per layer.

  python tools/prefill_ab.py [T]
With a DBF_PREFILL_TRACE build (DBF_B200_LIB=tools/_x/ptr.so) it also prints the per-tile timeline
of the last one-launch layer of each shape (claim -> first MMA -> last commit -> stored).
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch

import paper_2505_11076_b200 as P
from paper_2505_11076_b200 import _lib
from test_gpu_prefill import _two_launch

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
SHAPES = [("q", 4096, 2048, 4096), ("gate", 11008, 2976, 4096), ("down", 4096, 2976, 11008)]
g = torch.Generator(device="cuda")
g.manual_seed(0)


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


trace_fn = getattr(_lib.lib, "dbf_prefill_debug_layer", None)
for name, n, k, m in SHAPES:
    dl = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    X = torch.randn((T, m), generator=g, device="cuda").half()
    Y = torch.empty((T, n), dtype=torch.half, device="cuda")
    flops = 2.0 * T * k * (n + m)
    u1 = timed(lambda: P.forward_prefill(X, dl, out=Y, path="one_launch"))
    u2 = timed(lambda: P.forward_prefill(X, dl, out=Y, path="two_launches"))
    same = torch.equal(P.forward_prefill(X, dl, path="one_launch"), _two_launch(X, dl))
    print(f"{name:5s} T={T}: one launch {u1:7.1f} us ({flops / u1 / 1e6:6.0f} TF/s)   two launches {u2:7.1f} us "
          f"({flops / u2 / 1e6:6.0f} TF/s)   bitwise equal {same}")
    if trace_fn is not None:
        P.forward_prefill(X, dl, out=Y, path="one_launch")
        torch.cuda.synchronize()
        rt1, rt2, tbs = -(-k // 128), -(-n // 128), -(-T // 256)
        ntiles = (rt1 + rt2) * tbs
        buf = np.zeros(8 * ntiles, dtype=np.int64)
        trace_fn.restype = ctypes.c_int
        trace_fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
        assert trace_fn(buf.ctypes.data, 8 * ntiles) == 0
        tr = buf.reshape(ntiles, 8).astype(np.float64)
        t0 = tr[:, 0].min()
        tr = (tr - t0) / 1e3
        g1 = np.arange(ntiles) < rt1 * tbs
        for lab, sel in (("GEMM1", g1), ("GEMM2", ~g1)):
            d = tr[sel]
            print(f"   {lab}: tiles {sel.sum()}, claim->firstMMA median {np.median(d[:, 2] - d[:, 0]):.2f} us, "
                  f"K loop median {np.median(d[:, 3] - d[:, 2]):.2f}, commit->acc seen {np.median(d[:, 4] - d[:, 3]):.2f}, acc drained {np.median(d[:, 6] - d[:, 4]):.2f}, "
                  f"acc->stored {np.median(d[:, 5] - d[:, 4]):.2f}; first claim {d[:, 0].min():.1f}, last stored "
                  f"{d[:, 5].max():.1f} us")
        if (~g1).any():
            d = tr[~g1]
            print(f"   GEMM2 dependency wait (claim -> t ready) median {np.median(d[:, 1] - d[:, 0]):.2f} us, max "
                  f"{(d[:, 1] - d[:, 0]).max():.2f}")
        print(f"   span {tr[:, 5].max():.1f} us; sum of K loops / (148 x span) = "
              f"{(tr[:, 3] - tr[:, 2]).sum() / (148 * tr[:, 5].max()):.3f}")
        # per-K-block stamps of CTA 0 (clock64): TMA issue, activation box seen by the MMA issuer, signs
        # seen by the MMA issuer, expander warp 4 done (for the K-block pair)
        kt = np.zeros(4 * 1024, dtype=np.int64)
        off = 8 * ntiles
        full = np.zeros(off + 4 * 1024, dtype=np.int64)
        assert trace_fn(full.ctypes.data, off + 4 * 1024) == 0
        kt = full[off:].reshape(1024, 4).astype(np.float64)
        nk = int((kt[:, 1] > 0).sum())
        kt = kt[:nk]
        c0 = kt[0, 0]
        print("   CTA 0 per K block (cycles): g  tma_issue  act_seen  signs_seen  exp_done   [first 12, then deltas]")
        for gi in range(min(nk, 12)):
            print("     ", gi, *(int(v - c0) for v in kt[gi]))
        mma = np.diff(kt[:, 2])
        print(f"   MMA go deltas median {np.median(mma):.0f} cycles; waits: act after signs in "
              f"{(kt[:, 1] > kt[:, 2]).mean():.2f} of K blocks (signs later in the rest); "
              f"median (signs_seen - act_seen) {np.median(kt[:, 2] - kt[:, 1]):.0f}; "
              f"median (act_seen - tma_issue) {np.median(kt[:, 1] - kt[:, 0]):.0f}")
