"""The C-ABI library loads on a CPU-only host and exports every symbol include/dbf_b200.h
declares; host-only entry points (layout queries, argument validation, the engine's run-record
builder) behave as documented.  No kernel is launched here."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2505_11076_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "dbf_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(dbf_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_abi_version_and_status_strings():
    assert _lib.lib.dbf_abi_version() == 1
    assert _lib.lib.dbf_status_string(0) == b"ok"
    assert b"workspace" in _lib.lib.dbf_status_string(3)
    assert _lib.lib.dbf_status_string(99) == b"unknown status"


@pytest.mark.parametrize("cols", [1, 7, 8, 9, 31, 32, 33, 127, 128, 129, 255, 256, 257, 4096, 5952, 11008])
def test_layout_queries(cols):
    L = _lib.lib
    assert L.dbf_row_bytes(cols) == (cols + 7) // 8  # bitcore.py:67-69
    pitch = L.dbf_canonical_pitch_words(cols)
    assert pitch % 4 == 0 and pitch * 32 >= cols and (pitch - 4) * 32 < cols
    rows = 37
    assert L.dbf_tiled_bytes(rows, cols) == -(-rows // 16) * -(-cols // 256) * 512


def test_invalid_arguments_are_rejected_without_a_gpu():
    L = _lib.lib
    assert L.dbf_pack_signs(None, 1, 4, 4, 4, None, 4, None, None) == _lib.ERR_INVALID_ARGUMENT
    assert L.dbf_forward(None, None, None, None, None, 0, 1, 1, 1, None, 0, 1, 1, None, 0, 1, None, 0, None) == _lib.ERR_INVALID_ARGUMENT
    assert L.dbf_sign_matvec(None, 1, 1, None, 0, 1, 1, None, 0, 1, None, 0, None) == _lib.ERR_INVALID_ARGUMENT
    assert L.dbf_tile_signs(None, 1, 1, 4, None, None) == _lib.ERR_INVALID_ARGUMENT
    assert L.dbf_forward_workspace_bytes(4096, 4096, 4096, 2) >= 2 * 4096 * 4
    size = ctypes.c_size_t(0)
    assert L.dbf_engine_smem_bytes(11008, 1, ctypes.byref(size)) == 0 and 200_000 < size.value <= 227 * 1024
    assert L.dbf_engine_smem_bytes(11008, 4, ctypes.byref(size)) == 0 and size.value <= 227 * 1024
    assert L.dbf_engine_smem_bytes(10**7, 1, ctypes.byref(size)) == _lib.ERR_UNSUPPORTED
    # batch 1 keeps a warp's quantized input chunks in shared memory: at most 16 x 7 chunks wide
    assert L.dbf_engine_smem_bytes(28672, 1, ctypes.byref(size)) == 0
    assert L.dbf_engine_smem_bytes(28673, 1, ctypes.byref(size)) == _lib.ERR_UNSUPPORTED
    assert L.dbf_engine_smem_bytes(29000, 2, ctypes.byref(size)) == 0
    assert L.dbf_engine_smem_bytes(4096, 5, ctypes.byref(size)) == _lib.ERR_INVALID_ARGUMENT


def test_engine_run_records_resolve_everything_on_the_host():
    from paper_2505_11076_b200.engine import SEG_DTYPE, VEC_DTYPE

    segs = np.zeros(2, dtype=SEG_DTYPE)
    # segment 0: B (k=40 rows, m=300 cols) plain vec0 -> LL vec1 ; segment 1: A (n=70, k=40) vec1 -> LL vec2
    segs[0] = (0x1000, 40, 300, 0, 1, 0x2000, 0x3000, 1, 1, 0)
    segs[1] = (0x9000, 70, 40, 1, 2, 0, 0x4000, 1, 0, 0x5000)
    vecs = np.zeros(3, dtype=VEC_DTYPE)
    vecs[0] = (0xA000, 300, 0, 0, 0)
    vecs[1] = (0xB000, 40, 1, 0, 0)
    vecs[2] = (0xC000, 70, 1, 0, 0)
    runs = np.array([[0, 0, 3], [1, 2, 3]], dtype=np.int32)
    out = np.zeros(2 * 128, dtype=np.uint8)
    ready = 0x7000
    st = _lib.lib.dbf_engine_build_runs(segs.ctypes.data, 2, vecs.ctypes.data, 3, runs.ctypes.data, 2, 1, ready, out.ctypes.data)
    assert st == 0
    q = out.view(np.uint64)
    i32 = out.view(np.int32)
    r0, r1 = q[:16], q[16:]
    assert r0[0] == 0x1000 and r0[1] == 0xA000 and r0[2] == 0x2000 and r0[3] == 0x3000
    assert r0[5] == 0xB000 and r0[6] == 0 and r0[7] == ready + 4 * 1  # plain input: no ready_in
    assert list(i32[16:27]) == [40, 300, 0, 3, 0, 0, 0, 1, 1, 0, 1]  # rows cols rb n seg kind dt sdt odt in out
    # run 1 starts at row block 2 of A: tiled offset 2 blocks x 1 chunk x 512 B
    assert r1[0] == 0x9000 + 2 * 1 * 512 and r1[4] == 0x5000 and r1[6] == ready + 4 and r1[7] == ready + 8
    assert i32[32 + 27] == 3  # in_producers of vec1 = ceil(40/16) units of segment 0
    bad = np.array([[1, 4, 2]], dtype=np.int32)  # rows 64..95 of a 70-row segment: out of range
    assert _lib.lib.dbf_engine_build_runs(segs.ctypes.data, 2, vecs.ctypes.data, 3, bad.ctypes.data, 1, 1, ready, out.ctypes.data) == _lib.ERR_SHAPE


def test_python_struct_mirrors_match_the_c_layout(tmp_path):
    """The ctypes / numpy mirrors of the engine structs (engine.py) have the C header's size and
    field offsets (gcc compiles a probe against include/dbf_b200.h; no CUDA needed)."""
    import shutil
    import subprocess

    from paper_2505_11076_b200 import engine

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    prog = [f[0] for f in engine._Program._fields_]
    probes = [("dbf_engine_program", n) for n in prog]
    probes += [("dbf_engine_segment", n) for n in engine.SEG_DTYPE.names]
    probes += [("dbf_engine_vector", n) for n in engine.VEC_DTYPE.names]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "dbf_b200.h"', "int main(void) {"]
    for t in ("dbf_engine_program", "dbf_engine_segment", "dbf_engine_vector"):
        lines.append(f'  printf("{t} size %zu\\n", sizeof({t}));')
    for t, n in probes:
        lines.append(f'  printf("{t} {n} %zu\\n", offsetof({t}, {n}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", f"-I{HEADER.parent}", str(src), "-o", str(exe)], check=True)
    c = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        t, n, v = line.split()
        c[(t, n)] = int(v)
    assert c[("dbf_engine_program", "size")] == ctypes.sizeof(engine._Program)
    for f in engine._Program._fields_:
        assert c[("dbf_engine_program", f[0])] == getattr(engine._Program, f[0]).offset, f[0]
    for t, dt in (("dbf_engine_segment", engine.SEG_DTYPE), ("dbf_engine_vector", engine.VEC_DTYPE)):
        assert c[(t, "size")] == dt.itemsize, t
        for n in dt.names:
            assert c[(t, n)] == dt.fields[n][1], (t, n)


def test_batched_entry_points_validate_without_a_gpu():
    """The single-pass batched decode entry points (csrc/batched.cu): sizes on the host, argument
    and shape errors before any launch."""
    L = _lib.lib
    # up to 32 tokens; 0 (invalid) beyond
    assert L.dbf_forward_batched_workspace_bytes(4096, 2048, 4096, 16) > 0
    assert L.dbf_forward_batched_workspace_bytes(4096, 2048, 4096, 33) == 0
    assert L.dbf_forward_batched_workspace_bytes(4096, 2048, 4096, 0) == 0
    # fragments: chunks(cols) x 8 k-blocks x (tokens/4) x 32 lanes x 8 B, plus F and T per chunk
    # and token slot, rounded to 256 B
    for cols, batch in [(4096, 16), (300, 3), (11008, 32)]:
        tpad = -(-batch // 4) * 4
        ch = -(-cols // 256)
        want = ch * 8 * (tpad // 4) * 32 * 8 + 2 * ch * tpad * 4
        assert L.dbf_batched_frag_bytes(cols, batch) == -(-want // 256) * 256
    # the full call needs more workspace than the chained one (it quantizes x itself)
    assert L.dbf_forward_batched_workspace_bytes(4096, 2048, 4096, 8) > L.dbf_forward_batched_frag_workspace_bytes(
        4096, 2048, 4096, 8)
    args = [None, None, None, None, None, 0, 64, 32, 64, None, 0, 4, 64, None, 0, 64, None, 0, None, None]
    assert L.dbf_forward_batched(*args) == _lib.ERR_INVALID_ARGUMENT
    dummy = 0x1000
    ok = [dummy, dummy, dummy, dummy, dummy, 0, 64, 32, 64, dummy, 0, 4, 64, dummy, 0, 64, None, 0, None, None]
    assert L.dbf_forward_batched(*(ok[:11] + [33] + ok[12:])) == _lib.ERR_UNSUPPORTED   # > 32 tokens
    assert L.dbf_forward_batched(*(ok[:12] + [63] + ok[13:])) == _lib.ERR_SHAPE          # ldx < m
    assert L.dbf_forward_batched(*ok) == _lib.ERR_WORKSPACE                             # no workspace
    assert L.dbf_batched_quantize(None, 0, 64, 4, 64, None, 0, None, None) == _lib.ERR_INVALID_ARGUMENT
    assert L.dbf_batched_quantize(dummy, 0, 32, 4, 64, None, 0, dummy, None) == _lib.ERR_SHAPE
    fr = [dummy, dummy, dummy, dummy, 0, 64, 32, 64, dummy, 4, dummy, 0, 64, None, 5, None, 0, None, None]
    assert L.dbf_forward_batched_frag(*fr) == _lib.ERR_INVALID_ARGUMENT                 # consumers=NULL, n=5
    assert L.dbf_forward_batched_frag(*(fr[:13] + [dummy, 5] + fr[15:])) == _lib.ERR_UNSUPPORTED  # > 4 consumers


def test_prefill_path_rule_and_workspace_without_a_gpu():
    """Host-side prefill queries: the auto path rule (no GPU: 148 SMs assumed) and the workspace,
    which covers t plus the split-K partials (T <= 256) or the one-launch tile counters (T > 256)."""
    L = _lib.lib
    assert L.dbf_prefill_layer_path(4096, 2048, 4096, 2048) == 1     # q: 16 x 8 = 128 GEMM1 tiles
    assert L.dbf_prefill_layer_path(11008, 2976, 4096, 2048) == 2    # gate: 24 x 8 = 192 > 148
    assert L.dbf_prefill_layer_path(11008, 2976, 4096, 256) == 1     # one token tile: split-K path
    assert L.dbf_prefill_layer_path(0, 2976, 4096, 2048) == 1
    t_bytes = L.dbf_prefill_workspace_bytes(2976, 2048)
    assert t_bytes == 2048 * L.dbf_prefill_ld(2976) * 2 and L.dbf_prefill_ld(2976) % 64 == 0
    assert L.dbf_prefill_workspace_bytes_nkm(11008, 2976, 4096, 2048) > t_bytes
    bad = L.dbf_forward_prefill_ex(None, 1, None, 1, None, None, None, 1, 1, 1, None, 1, 1, None, 1, None, 0, 2, None)
    assert bad == _lib.ERR_INVALID_ARGUMENT
