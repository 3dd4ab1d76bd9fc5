"""Quick GPU check of the tcgen05 prefill sign GEMM against a torch fp32 reference, plus timing.

python tools/prefill_check.py [T n k m]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2505_11076_b200 as P
from paper_2505_11076_b200 import _lib


def main():
    T, n, k, m = (int(v) for v in sys.argv[1:5]) if len(sys.argv) >= 5 else (512, 384, 320, 512)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    layer = P.random_device_layer(n, k, m, generator=g, keep_words=True)
    X = torch.randn((T, m), generator=g, device="cuda").half()
    # single GEMM check: out = rscale * (X . (B*b)^T)
    Bd = layer.B.unpack(torch.float32)
    out = torch.empty((T, k), dtype=torch.half, device="cuda")
    _lib.check(_lib.lib.dbf_sign_gemm(X.data_ptr(), T, m, m, layer.B.paired.data_ptr(), layer.B.paired.shape[1], k,
                                      layer.b.data_ptr(), layer.mid.data_ptr(), out.data_ptr(), k,
                                      _lib.stream_ptr()), "dbf_sign_gemm")
    ref = layer.mid.float()[None, :] * ((X.float() * layer.b.float()[None, :]) @ Bd.t())
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
    print(f"gemm1 T={T} rows={k} K={m}: max rel err {err:.3e}")
    # full forward
    ws = torch.empty(_lib.lib.dbf_prefill_workspace_bytes(k, T), dtype=torch.uint8, device="cuda")
    Y = torch.empty((T, n), dtype=torch.half, device="cuda")

    def run():
        _lib.check(_lib.lib.dbf_forward_prefill(
            layer.A.paired.data_ptr(), layer.A.paired.shape[1], layer.B.paired.data_ptr(), layer.B.paired.shape[1],
            layer.a.data_ptr(), layer.mid.data_ptr(), layer.b.data_ptr(), n, k, m, X.data_ptr(), T, m,
            Y.data_ptr(), n, ws.data_ptr(), ws.numel(), _lib.stream_ptr()), "dbf_forward_prefill")

    run()
    Ad = layer.A.unpack(torch.float32)
    t = ref.half().float()
    refY = layer.a.float()[None, :] * (t @ Ad.t())
    torch.cuda.synchronize()
    errY = (Y.float() - refY).abs().max().item() / refY.abs().max().item()
    nrm = ((Y.float() - refY).norm() / refY.norm()).item()
    print(f"forward: max rel err {errY:.3e}  norm rel err {nrm:.3e}")
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    flops = 2.0 * T * k * (n + m)
    print(f"forward {us:.1f} us  {flops / us / 1e6:.1f} TFLOP/s")

    Yf = P.forward_prefill(X, layer)
    torch.cuda.synchronize()
    errF = (Yf.float() - refY).abs().max().item() / refY.abs().max().item()
    for _ in range(3):
        P.forward_prefill(X, layer, out=Yf)
    e0.record()
    for _ in range(reps):
        P.forward_prefill(X, layer, out=Yf)
    e1.record()
    e1.synchronize()
    usf = e0.elapsed_time(e1) * 1e3 / reps
    print(f"fused forward {usf:.1f} us  {flops / usf / 1e6:.1f} TFLOP/s  max rel err {errF:.3e}")

    def g1():
        _lib.lib.dbf_sign_gemm(X.data_ptr(), T, m, m, layer.B.paired.data_ptr(), layer.B.paired.shape[1], k,
                               layer.b.data_ptr(), layer.mid.data_ptr(), out.data_ptr(), k, _lib.stream_ptr())

    def g2():
        _lib.lib.dbf_sign_gemm(out.data_ptr(), T, k, k, layer.A.paired.data_ptr(), layer.A.paired.shape[1], n,
                               None, layer.a.data_ptr(), Y.data_ptr(), n, _lib.stream_ptr())

    for name, fn, fl in (("gemm1", g1, 2.0 * T * k * m), ("gemm2", g2, 2.0 * T * k * n)):
        for _ in range(3):
            fn()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        print(f"  {name} {us:.1f} us  {fl / us / 1e6:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
