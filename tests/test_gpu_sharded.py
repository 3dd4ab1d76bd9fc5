"""k-sharded DBF layer on one GPU: the shards' fp32 partials (dbf_forward_partial) summed and
finalized equal the unsharded forward within the fp16 tolerance, for 70B-like shapes; plus the
NCCL path end to end with a 1-rank process group."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2505_11076_b200 as P  # noqa: E402
from paper_2505_11076_b200 import sharded  # noqa: E402
from conftest import rel_max, rel_norm  # noqa: E402


def _host_layer(rng, n, k, m):
    A = rng.integers(0, 2, (n, k)) * 2.0 - 1
    B = rng.integers(0, 2, (k, m)) * 2.0 - 1
    f16 = lambda v: v.astype(np.float16).astype(np.float64)
    return P.DbfLayer(a=f16(rng.uniform(0.5, 1.5, n) / np.sqrt(k)), A=P.SignMatrix(n, k, np.packbits(A > 0, axis=1, bitorder="little")),
                      mid=f16(rng.uniform(0.5, 1.5, k)), B=P.SignMatrix(k, m, np.packbits(B > 0, axis=1, bitorder="little")),
                      b=f16(rng.uniform(0.5, 1.5, m) / np.sqrt(m)))


@pytest.mark.parametrize("world,n,k,m,batch", [(2, 1024, 1792, 8192, 1), (4, 2048, 3000, 4096, 3), (8, 1024, 1792, 8192, 16)])
def test_simulated_shards_sum_to_the_full_forward(world, n, k, m, batch):
    import torch

    rng = np.random.default_rng(world * 7 + batch)
    layer = _host_layer(rng, n, k, m)
    X = rng.standard_normal((batch, m)).astype(np.float16)
    Xd = torch.from_numpy(X).cuda()
    total = None
    for r in range(world):
        ds = sharded.DeviceShard(sharded.shard_layer(layer, r, world), scale_dtype=torch.float16)
        p = ds.partial(Xd)
        total = p if total is None else total + p
    y = ds.finalize(total, out_dtype=torch.float32).cpu().numpy()
    ref = oracle.c_forward(X.astype(np.float64), layer.a, layer.A.bits, layer.mid, layer.B.bits, layer.b)
    assert rel_max(y, ref) <= 1e-2 and rel_norm(y, ref) <= 1e-2


@pytest.mark.parametrize("world,n,k,m,batch", [(2, 1024, 1792, 8192, 1), (4, 2048, 3000, 4096, 3), (2, 1000, 600, 777, 4)])
def test_engine_partials_sum_to_the_full_forward(world, n, k, m, batch):
    """partial_engine (one decode-engine launch per shard, launch-time I/O buffers): the shards'
    fp32 partials summed and finalized match the oracle forward within the fp16 tolerance, and a
    second call on other buffers gives the same bits."""
    import torch

    rng = np.random.default_rng(world * 11 + batch)
    layer = _host_layer(rng, n, k, m)
    X = rng.standard_normal((batch, m)).astype(np.float16)
    Xd = torch.from_numpy(X).cuda()
    total = None
    for r in range(world):
        ds = sharded.DeviceShard(sharded.shard_layer(layer, r, world), scale_dtype=torch.float16)
        p = ds.partial_engine(Xd)
        assert torch.equal(ds.partial_engine(Xd.clone()), p)
        q = ds.partial(Xd)
        assert rel_max(p.cpu().numpy(), q.cpu().numpy()) <= 1e-2
        total = p if total is None else total + p
    y = ds.finalize(total, out_dtype=torch.float32).cpu().numpy()
    ref = oracle.c_forward(X.astype(np.float64), layer.a, layer.A.bits, layer.mid, layer.B.bits, layer.b)
    assert rel_max(y, ref) <= 1e-2 and rel_norm(y, ref) <= 1e-2


def test_nccl_single_rank_group():
    import torch
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(3)
        layer = _host_layer(rng, 512, 640, 1024)
        ds = sharded.DeviceShard(sharded.shard_layer(layer, 0, 1), scale_dtype=torch.float16)
        X = rng.standard_normal((2, 1024)).astype(np.float16)
        y = ds.forward(torch.from_numpy(X).cuda()).float().cpu().numpy()
        ref = oracle.c_forward(X.astype(np.float64), layer.a, layer.A.bits, layer.mid, layer.B.bits, layer.b)
        assert rel_max(y, ref) <= 1e-2
    finally:
        dist.destroy_process_group()


# ---- all-reduce fused into GEMV2 (dbf_forward_allreduce) -----------------------------------------

def _ptrs(ts):
    import torch

    return torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device="cuda")


@pytest.mark.parametrize("batch", [1, 3, 16])
def test_fused_allreduce_single_rank_equals_partial_path(batch):
    """world = 1: the fused kernel's in-place combine (no push, fence or flags: nothing to exchange)
    gives the same bits as dbf_forward_partial + dbf_finalize_partial, over several epochs."""
    import torch

    from paper_2505_11076_b200 import _lib

    rng = np.random.default_rng(20 + batch)
    layer = _host_layer(rng, 1000, 640, 1024)
    ds = sharded.DeviceShard(sharded.shard_layer(layer, 0, 1), scale_dtype=torch.float16)
    recv = torch.empty(_lib.lib.dbf_allreduce_recv_bytes(1000, batch, 1) // 4, dtype=torch.float32, device="cuda")
    flags = torch.zeros(_lib.lib.dbf_allreduce_flag_bytes(1000, 1) // 4, dtype=torch.int32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    for epoch in range(1, 5):
        X = torch.from_numpy(rng.standard_normal((batch, 1024)).astype(np.float16)).cuda()
        ref = ds.finalize(ds.partial(X), out_dtype=torch.float16)
        y = ds.forward_allreduce(X, _ptrs([recv]), _ptrs([flags]), counter)
        torch.cuda.synchronize()
        assert torch.equal(y, ref), epoch
        assert int(counter.item()) == epoch
        # world 1 takes the in-place combine: no flags are raised (nothing waits on them)
        assert int(flags.abs().max()) == 0
    out = oracle.c_forward(X.double().cpu().numpy(), layer.a, layer.A.bits, layer.mid, layer.B.bits, layer.b)
    assert rel_max(y.float().cpu().numpy(), out) <= 1e-2


@pytest.mark.parametrize("world,rank,batch", [(4, 1, 2), (2, 0, 1), (8, 7, 16)])
def test_fused_allreduce_combines_pushed_peer_partials(world, rank, batch):
    """One rank of a `world`-GPU group on one GPU, the other ranks' pushes staged beforehand (their
    partials written into this rank's receive slots and their flags raised), so nothing waits on
    another kernel: the result is a * (sum of all ranks' partials in rank order) bit for bit, and
    this rank's own partial lands in slot `rank` of every peer buffer."""
    import torch

    from paper_2505_11076_b200 import _lib

    rng = np.random.default_rng(world * 10 + rank)
    n, k, m = 1000, 1792, 2048
    layer = _host_layer(rng, n, k, m)
    X = torch.from_numpy(rng.standard_normal((batch, m)).astype(np.float16)).cuda()
    shards = [sharded.DeviceShard(sharded.shard_layer(layer, g, world), scale_dtype=torch.float16) for g in range(world)]
    parts = [s.partial(X) for s in shards]
    nrb = -(-n // 16)
    rbytes = _lib.lib.dbf_allreduce_recv_bytes(n, batch, world)
    recvs = [torch.zeros(rbytes // 4, dtype=torch.float32, device="cuda") for _ in range(world)]
    flags = [torch.zeros(_lib.lib.dbf_allreduce_flag_bytes(n, world) // 4, dtype=torch.int32, device="cuda")
             for _ in range(world)]
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    for epoch in (1, 2):
        mine = recvs[rank].view(2, world, batch, n)[epoch & 1]
        for g in range(world):
            if g != rank:
                mine[g].copy_(parts[g])
        fl = flags[rank].view(16, world, nrb)
        for g in range(world):
            if g != rank:
                fl[:, g, :] = epoch
        torch.cuda.synchronize()
        y = shards[rank].forward_allreduce(X, _ptrs(recvs), _ptrs(flags), counter, out_dtype=torch.float32)
        torch.cuda.synchronize()
        acc = np.zeros((batch, n))
        for g in range(world):
            acc += parts[g].double().cpu().numpy()
        a = shards[rank].a.double().cpu().numpy()
        want = (acc.astype(np.float32).astype(np.float64) * a[None, :]).astype(np.float32)
        np.testing.assert_array_equal(y.cpu().numpy(), want)
        for g in range(world):  # the push: our partial in slot `rank` of every buffer, our flag raised
            assert torch.equal(recvs[g].view(2, world, batch, n)[epoch & 1][rank], parts[rank])
            assert int(flags[g].view(16, world, nrb)[0, rank].min()) == epoch
    ref = oracle.c_forward(X.double().cpu().numpy(), layer.a, layer.A.bits, layer.mid, layer.B.bits, layer.b)
    assert rel_max(y.cpu().numpy(), ref) <= 1e-2 and rel_norm(y.cpu().numpy(), ref) <= 1e-2


def test_fused_allreduce_symmetric_memory_single_rank():
    """FusedAllReduce over a 1-rank NCCL group: buffers from torch symmetric memory."""
    import torch
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(9)
        layer = _host_layer(rng, 512, 640, 1024)
        ds = sharded.DeviceShard(sharded.shard_layer(layer, 0, 1), scale_dtype=torch.float16)
        try:
            ar = sharded.FusedAllReduce(512, 4)
        except Exception as e:  # noqa: BLE001 - symmetric memory needs driver/fabric support
            pytest.skip(f"torch symmetric memory unavailable: {e}")
        for _ in range(3):
            X = torch.from_numpy(rng.standard_normal((4, 1024)).astype(np.float16)).cuda()
            y = ar.forward(ds, X)
            assert torch.equal(y, ds.forward(X))
        # graph replay: the device-side call counter gives every replay a fresh epoch
        X = torch.from_numpy(rng.standard_normal((4, 1024)).astype(np.float16)).cuda()
        ref = ds.forward(X)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            ar.forward(ds, X)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            yg = ar.forward(ds, X)
        for _ in range(4):
            yg.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(yg, ref)
        assert int(ar.counter.item()) == 3 + 1 + 4  # eager calls, warm-up call, replays (capture runs nothing)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [1, 3, 4])
def test_engine_fused_allreduce_single_rank_equals_engine_partial(batch):
    """world = 1 through the decode engine: the fused last stage (in-place combine at world 1) gives
    the same bits as partial_engine + dbf_finalize_partial, over several calls; the call counter
    advances once per call."""
    import torch

    from paper_2505_11076_b200 import _lib

    rng = np.random.default_rng(30 + batch)
    n, k, m = 1000, 640, 1024
    layer = _host_layer(rng, n, k, m)
    ds = sharded.DeviceShard(sharded.shard_layer(layer, 0, 1), scale_dtype=torch.float16)
    recv = torch.empty(_lib.lib.dbf_allreduce_recv_bytes(n, batch, 1) // 4, dtype=torch.float32, device="cuda")
    flags = torch.zeros(_lib.lib.dbf_allreduce_flag_bytes(n, 1) // 4, dtype=torch.int32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    for epoch in range(1, 5):
        X = torch.from_numpy(rng.standard_normal((batch, m)).astype(np.float16)).cuda()
        ref = ds.finalize(ds.partial_engine(X), out_dtype=torch.float16)
        y = ds.forward_allreduce_engine(X, _ptrs([recv]), _ptrs([flags]), counter)
        torch.cuda.synchronize()
        assert torch.equal(y, ref), epoch
        assert int(counter.item()) == epoch
        # world 1 takes the in-place combine: no flags are raised (nothing waits on them)
        assert int(flags.abs().max()) == 0
    # the per-layer fused path shares the counter / flags / buffers: calls of both paths interleave
    y2 = ds.forward_allreduce(X, _ptrs([recv]), _ptrs([flags]), counter)
    y3 = ds.forward_allreduce_engine(X, _ptrs([recv]), _ptrs([flags]), counter)
    torch.cuda.synchronize()
    assert int(counter.item()) == 6 and torch.equal(y3, ref)
    out = oracle.c_forward(X.double().cpu().numpy(), layer.a, layer.A.bits, layer.mid, layer.B.bits, layer.b)
    for v in (y, y2, y3):
        assert rel_max(v.float().cpu().numpy(), out) <= 1e-2 and rel_norm(v.float().cpu().numpy(), out) <= 1e-2


@pytest.mark.parametrize("world,rank,batch", [(2, 1, 1), (4, 0, 4), (8, 5, 2)])
def test_engine_fused_allreduce_combines_pushed_peer_partials(world, rank, batch):
    """One rank of a `world`-GPU group through the engine, the other ranks' pushes staged
    beforehand (no kernel waits on another): y = a * (sum of all ranks' engine partials in rank
    order) bit for bit, and this rank's partial lands in slot `rank` of every peer buffer."""
    import torch

    from paper_2505_11076_b200 import _lib

    rng = np.random.default_rng(world * 100 + rank)
    n, k, m = 1000, 1792, 2048
    layer = _host_layer(rng, n, k, m)
    X = torch.from_numpy(rng.standard_normal((batch, m)).astype(np.float16)).cuda()
    shards = [sharded.DeviceShard(sharded.shard_layer(layer, g, world), scale_dtype=torch.float16) for g in range(world)]
    parts = [s.partial_engine(X) for s in shards]
    nrb = -(-n // 16)
    recvs = [torch.zeros(_lib.lib.dbf_allreduce_recv_bytes(n, batch, world) // 4, dtype=torch.float32, device="cuda")
             for _ in range(world)]
    flags = [torch.zeros(_lib.lib.dbf_allreduce_flag_bytes(n, world) // 4, dtype=torch.int32, device="cuda")
             for _ in range(world)]
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    for epoch in (1, 2, 3):
        mine = recvs[rank].view(2, world, batch, n)[epoch & 1]
        fl = flags[rank].view(16, world, nrb)
        for g in range(world):
            if g != rank:
                mine[g].copy_(parts[g])
                fl[0, g, :] = epoch
        torch.cuda.synchronize()
        y = shards[rank].forward_allreduce_engine(X, _ptrs(recvs), _ptrs(flags), counter, out_dtype=torch.float32)
        torch.cuda.synchronize()
        acc = np.zeros((batch, n))
        for g in range(world):
            acc += parts[g].double().cpu().numpy()
        a = shards[rank].a.double().cpu().numpy()
        want = (acc.astype(np.float32).astype(np.float64) * a[None, :]).astype(np.float32)
        np.testing.assert_array_equal(y.cpu().numpy(), want)
        for g in range(world):
            assert torch.equal(recvs[g].view(2, world, batch, n)[epoch & 1][rank], parts[rank])
            assert int(flags[g].view(16, world, nrb)[0, rank].min()) == epoch
    ref = oracle.c_forward(X.double().cpu().numpy(), layer.a, layer.A.bits, layer.mid, layer.B.bits, layer.b)
    assert rel_max(y.cpu().numpy(), ref) <= 1e-2 and rel_norm(y.cpu().numpy(), ref) <= 1e-2


def test_engine_fused_allreduce_symmetric_memory_single_rank():
    """FusedAllReduce.forward(engine=True) over a 1-rank NCCL group (symmetric-memory buffers):
    equal to the engine partial + NCCL all-reduce path, eager and graph-replayed."""
    import torch
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(19)
        layer = _host_layer(rng, 512, 640, 1024)
        ds = sharded.DeviceShard(sharded.shard_layer(layer, 0, 1), scale_dtype=torch.float16)
        try:
            ar = sharded.FusedAllReduce(512, 4)
        except Exception as e:  # noqa: BLE001 - symmetric memory needs driver/fabric support
            pytest.skip(f"torch symmetric memory unavailable: {e}")
        for _ in range(3):
            X = torch.from_numpy(rng.standard_normal((4, 1024)).astype(np.float16)).cuda()
            assert torch.equal(ar.forward(ds, X, engine=True), ds.forward(X, engine=True))
        X = torch.from_numpy(rng.standard_normal((4, 1024)).astype(np.float16)).cuda()
        ref = ds.forward(X, engine=True)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            ar.forward(ds, X, engine=True)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            yg = ar.forward(ds, X, engine=True)
        for _ in range(4):
            yg.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(yg, ref)
        assert int(ar.counter.item()) == 3 + 1 + 4
    finally:
        dist.destroy_process_group()
