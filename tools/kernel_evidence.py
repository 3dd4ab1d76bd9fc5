"""Bandwidth evidence for the kernels the benchmark does not headline (VERDICT r1 'evidence' items):

* dbf_pack_signs (bitcore.pack, /root/reference/pkg/src/dbf/bitcore.py:72-85): dense +-1 matrices
  of Llama-2-7B shapes (fp16 / fp32 / bf16) -> canonical words; bytes = dense read + words written
  (+ the 8-byte first-offender word); GB/s against MEASURED_PEAKS.json hbm_gbs.
* the north_star XOR + HADD2 decode (dbf_sign_matvec_xor, CUDA cores) against the int8
  tensor-core GEMV (dbf_sign_matvec) on the same sign matrices (batch 1, fp16 x): GB/s of packed
  signs, same matrix, CUDA events, many distinct instances per timing (> 2x L2).

usage: python tools/kernel_evidence.py [out.json]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

import paper_2505_11076_b200 as P
from paper_2505_11076_b200 import _lib


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3  # seconds per call


def timed_graph(fn, per_graph=20, replays=10):
    """Device time per call with the host out of the loop: `per_graph` calls captured in one CUDA
    graph, replayed (a short kernel launched from Python through ctypes is otherwise host-bound:
    round 2's first pack measurement timed ~20 us of launch overhead per call)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(per_graph):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / (replays * per_graph) * 1e-3


peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
out = {"peak_gbs": peak, "pack": [], "xor_vs_int8": []}
g = torch.Generator(device="cuda")
g.manual_seed(0)
for (rows, cols) in [(4096, 4096), (11008, 4096), (4096, 11008), (5952, 11008)]:
    for dt in (torch.float16, torch.float32, torch.bfloat16):
        dense = (torch.randint(0, 2, (rows, cols), generator=g, device="cuda", dtype=torch.int8) * 2 - 1).to(dt)
        pitch = _lib.lib.dbf_canonical_pitch_words(cols)
        words = torch.empty((rows, pitch), dtype=torch.int32, device="cuda")
        bad = torch.empty((), dtype=torch.int64, device="cuda")

        def run():
            _lib.check(_lib.lib.dbf_pack_signs(dense.data_ptr(), _lib.dtype_code(dt), rows, cols, cols,
                                               words.data_ptr(), pitch, bad.data_ptr(), _lib.stream_ptr()),
                       "dbf_pack_signs")

        t = timed_graph(run)
        nbytes = rows * cols * dense.element_size() + rows * pitch * 4 + 8
        out["pack"].append({"rows": rows, "cols": cols, "dtype": str(dt).split(".")[-1], "us": t * 1e6,
                            "gbs": nbytes / t / 1e9, "frac": nbytes / t / 1e9 / peak})
        back = torch.empty_like(dense)

        def run_unpack():
            _lib.check(_lib.lib.dbf_unpack_signs(words.data_ptr(), rows, cols, pitch, back.data_ptr(),
                                                 _lib.dtype_code(dt), cols, _lib.stream_ptr()), "dbf_unpack_signs")

        t = timed_graph(run_unpack)
        assert torch.equal(back, dense), "unpack(pack(x)) != x"
        out.setdefault("unpack", []).append({"rows": rows, "cols": cols, "dtype": str(dt).split(".")[-1],
                                             "us": t * 1e6, "gbs": nbytes / t / 1e9, "frac": nbytes / t / 1e9 / peak})
        del back
        del dense, words

for name, rows, cols in [("q.B / q.A 4096x4096", 4096, 4096), ("gate.A 11008x5952", 11008, 5952),
                         ("down.B 5952x11008", 5952, 11008)]:
    inst = max(4, -(-300_000_000 // (rows * cols // 8)))
    mats = [P.DeviceSignMatrix.random(rows, cols, generator=g, device="cuda", keep_words=True) for _ in range(inst)]
    x = torch.randn((1, cols), generator=g, device="cuda").half()
    ys = [torch.empty((rows,), dtype=torch.float32, device="cuda") for _ in range(inst)]

    def xor_all():
        for s, y in zip(mats, ys):
            _lib.check(_lib.lib.dbf_sign_matvec_xor(s.words.data_ptr(), rows, cols, s.words.shape[1], x.data_ptr(),
                                                    _lib.dtype_code(x.dtype), y.data_ptr(), _lib.stream_ptr()),
                       "dbf_sign_matvec_xor")

    def int8_all():
        for s in mats:
            P.sign_matvec_device(s, x[0], out_dtype=torch.float32)

    sign_bytes = rows * ((cols + 7) // 8)
    t_x = timed(xor_all, reps=5) / inst
    t_i = timed(int8_all, reps=5) / inst
    out["xor_vs_int8"].append({"matrix": name, "instances": inst, "xor_us": t_x * 1e6, "xor_gbs": sign_bytes / t_x / 1e9,
                               "int8_tc_us": t_i * 1e6, "int8_tc_gbs": sign_bytes / t_i / 1e9,
                               "int8_over_xor": t_x / t_i})
    del mats, ys
    torch.cuda.empty_cache()

s = json.dumps(out, indent=1)
print(s)
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(s)
