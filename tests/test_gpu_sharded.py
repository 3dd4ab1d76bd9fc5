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
