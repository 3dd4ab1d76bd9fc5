"""World-size-2 k-sharded forward on CPU (gloo): each rank cuts its shard with the product's
host logic, computes its partial with the ORACLE (the checker -- no GPU here), the partials are
SUM all-reduced over gloo, and a * sum must equal the oracle's unsharded forward."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_q):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from oracle import dbf_oracle as npo
        from paper_2505_11076_b200 import sharded

        rng = np.random.default_rng(42)
        n, k, m, batch = 96, 1100, 130, 3
        A = rng.integers(0, 2, (n, k)) * 2.0 - 1
        B = rng.integers(0, 2, (k, m)) * 2.0 - 1
        a, mid, b = rng.standard_normal(n), rng.standard_normal(k), rng.standard_normal(m)
        X = rng.standard_normal((batch, m))
        bitsA, bitsB = npo.pack_bits(A), npo.pack_bits(B)

        class L:  # duck-typed reference layer
            pass

        layer = L()
        layer.a, layer.mid, layer.b = a, mid, b
        layer.A = type("S", (), {"rows": n, "cols": k, "bits": bitsA})()
        layer.B = type("S", (), {"rows": k, "cols": m, "bits": bitsB})()
        sh = sharded.shard_layer(layer, rank, world)
        part = np.stack([
            oracle.c_sign_matvec(sh.A.bits, sh.k_shard, oracle.c_sign_matvec(sh.B.bits, m, X[i] * b) * sh.mid)
            for i in range(batch)
        ])
        t = torch.from_numpy(part)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        y = t.numpy() * a[None, :]
        ref = npo.forward(X, a, bitsA, mid, bitsB, b)
        result_q.put((rank, float(np.max(np.abs(y - ref)) / np.max(np.abs(ref))), sh.k0, sh.k1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_k_sharded_forward_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[2:] for r in res] == [(0, 544), (544, 1100)]
    for _, err, _, _ in res:
        assert err < 1e-12
