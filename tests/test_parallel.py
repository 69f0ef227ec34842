"""World-size-2 gloo tests (CPU) of the row-sharded driver: shard ranges, CSR gather, and
that the sharded result equals the single-process result (rows are independent, §8(e)).
The per-shard compute is injected (the fp64 oracle) so the host logic runs without a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_19892_b200.parallel import gather_topk_csr, shard_rows, sharded_sparse_precision


def test_shard_rows_partition():
    for n in (1, 7, 100, 1_000_000, 30_001):
        for w in (1, 2, 3, 8):
            ranges = [shard_rows(n, w, r) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(V, lam, b, e, t):
    import oracle as O
    rp, col, val = O.sparse_precision(V.numpy(), lam.numpy(), b, e, mode=0, t=t)
    return (torch.from_numpy(rp), torch.from_numpy(col.astype(np.int32)),
            torch.from_numpy(val.astype(np.float32)))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from synth import gen
        axes = []
        for (n, k, seed) in [(203, 7, 1), (64, 5, 2)]:
            V, lam = gen.small_factor(seed, n, k)
            Vt, lt = torch.from_numpy(V), torch.from_numpy(lam)
            if rank != 0:          # factors arrive by broadcast
                Vt.zero_()
                lt.zero_()
            from paper_2407_19892_b200.parallel import broadcast_factors
            broadcast_factors(Vt, lt, 0)
            axes.append((Vt, lt))
        res = sharded_sparse_precision(axes, 6, compute=_oracle_compute)
        if rank == 0:
            q.put([(r.numpy(), c.numpy(), v.numpy()) for r, c, v in res])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_single(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle as O
    from synth import gen
    for (n, k, seed), (rp, c, v) in zip([(203, 7, 1), (64, 5, 2)], got):
        V, lam = gen.small_factor(seed, n, k)
        rp1, c1, v1 = O.sparse_precision(V, lam, 0, n, mode=0, t=6)
        np.testing.assert_array_equal(rp, rp1)
        np.testing.assert_array_equal(c, c1)
        np.testing.assert_allclose(v, v1, rtol=1e-6)


def test_gather_single_process_passthrough():
    col = torch.arange(12, dtype=torch.int32)
    val = torch.ones(12)
    rp, c, v = gather_topk_csr(col, val, 3, 4)
    assert rp.tolist() == [0, 3, 6, 9, 12]
    assert torch.equal(c, col)
