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


# ---------------------------------------------------------------- distributed symmetric scheme
# Host logic of parallel.sharded_symmetric_precision (all-to-all of candidate buckets, merge
# of the received rows, all-gather + scatter by original row id) with oracle-backed injected
# shard / merge functions standing in for libggm's ggm_sparse_precision_sym_shard / ggm_sym_merge.

def _sym_fns(n, world, t):
    import oracle as O
    rng = np.random.default_rng(12)
    perm = rng.permutation(n).astype(np.int32)          # bound order -> original id
    bounds = [shard_rows(n, world, r)[0] for r in range(world)] + [n]

    def rows_begin(r):
        return bounds[r]

    def shard(V, lam, tt, rank, w):
        Vp = V.numpy()[perm]                            # rows in bound order
        P = O.psi_rows(Vp, lam.numpy(), np.arange(n))
        A = np.abs(P)
        np.fill_diagonal(A, -1.0)
        thr = -np.partition(-A, min(tt + 3, n - 2), axis=1)[:, min(tt + 3, n - 2)]
        keys, src, vals = [], [], []
        for i in range(bounds[rank], bounds[rank + 1]):  # this rank's pairs (i, j), j >= i
            for j in range(i, n):
                if j == i:
                    continue
                if A[i, j] >= thr[i]:
                    keys.append(i); src.append(j); vals.append(P[i, j])
                if A[j, i] >= thr[j]:               # the transposed direction
                    keys.append(j); src.append(i); vals.append(P[j, i])
        order = np.argsort(np.asarray(keys, np.int64), kind="stable")
        keys = np.asarray(keys, np.int32)[order]
        v2 = np.stack([np.asarray(src, np.int32)[order],
                       np.asarray(vals, np.float32)[order].view(np.int32)], 1)
        counts = [int(np.sum((keys >= bounds[d]) & (keys < bounds[d + 1]))) for d in range(w)]
        return torch.from_numpy(keys), torch.from_numpy(v2), counts, torch.from_numpy(perm)

    def merge(nn, tt, key, val, pm, b, e):
        key, val, pm = key.numpy(), val.numpy(), pm.numpy()
        te = min(tt, nn - 1)
        rid, cols, vs = [], [], []
        for j in range(b, e):
            sel = key == j
            src = pm[val[sel, 0]]
            v = val[sel, 1].copy().view(np.float32)
            order = np.lexsort((src, -np.abs(v)))[:te]
            keep = np.argsort(src[order], kind="stable")
            rid.append(pm[j]); cols.append(src[order][keep]); vs.append(v[order][keep])
        return (torch.tensor(rid, dtype=torch.int64),
                torch.from_numpy(np.concatenate(cols).astype(np.int32)) if cols else torch.empty(0, dtype=torch.int32),
                torch.from_numpy(np.concatenate(vs).astype(np.float32)) if vs else torch.empty(0))

    return shard, merge, rows_begin


def _sym_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from synth import gen
        from paper_2407_19892_b200.parallel import sharded_symmetric_precision
        n, k, t = 150, 6, 5
        V, lam = gen.small_factor(31, n, k)
        shard, merge, rows_begin = _sym_fns(n, world, t)
        rp, c, v = sharded_symmetric_precision(torch.from_numpy(V), torch.from_numpy(lam), t,
                                               shard=shard, merge=merge, rows_begin=rows_begin)
        q.put((rank, rp.numpy(), c.numpy(), v.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_symmetric_equals_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sym_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle as O
    from synth import gen
    n, k, t = 150, 6, 5
    V, lam = gen.small_factor(31, n, k)
    rp1, c1, v1 = O.sparse_precision(V, lam, 0, n, mode=0, t=t)
    for _, rp, c, v in got:                      # every rank holds the full CSR
        np.testing.assert_array_equal(rp, rp1)
        np.testing.assert_array_equal(c, c1)
        np.testing.assert_allclose(v, v1, rtol=1e-6)


# ------------------------------------------------------------ sharded spectrum (one all-reduce)

def _np_csr_fns():
    """NumPy stand-ins of the three CUDA steps (dense from CSR; host logic under test)."""
    def dense(rp, c, v, m):
        rp, c, v = rp.numpy(), c.numpy(), v.numpy().astype(np.float64)
        A = np.zeros((len(rp) - 1, m))
        for i in range(len(rp) - 1):
            A[i, c[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
        return A

    def acc(rp, c, v, m, npn):
        A = dense(rp, c, v, m)
        return torch.from_numpy(A.T @ A)

    def eig(Gm, k):
        w, Z = np.linalg.eigh(Gm.numpy())
        W = Z[:, ::-1][:, :k].copy()
        E = w[::-1][:k].copy()
        return torch.from_numpy(W.astype(np.float32)), torch.from_numpy(E), torch.from_numpy(W)

    def proj(rp, c, v, m, W, E, npn):
        A = dense(rp, c, v, m)
        return torch.from_numpy((A @ W.numpy()) / np.sqrt(E.numpy()))
    return acc, eig, proj


def _spectrum_matrix():
    rng = np.random.default_rng(21)
    X = rng.standard_normal((157, 23)) * (rng.random((157, 23)) < 0.3)
    return X.astype(np.float32)


def _spec_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_19892_b200.parallel import sharded_csr_spectrum
        X = _spectrum_matrix()
        b, e = shard_rows(X.shape[0], world, rank)
        Xr = X[b:e]
        rows, cols = np.nonzero(Xr)
        rp = np.zeros(e - b + 1, np.int64)
        np.add.at(rp, rows + 1, 1)
        rp = np.cumsum(rp)
        acc, eig, proj = _np_csr_fns()
        Vs, E, Vl = sharded_csr_spectrum(torch.from_numpy(rp), torch.from_numpy(cols.astype(np.int32)),
                                         torch.from_numpy(Xr[rows, cols]), X.shape[1], 6,
                                         accumulate=acc, eig=eig, project=proj)
        q.put((rank, Vs.numpy(), E.numpy(), Vl.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_spectrum_equals_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spec_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle as O
    X = _spectrum_matrix()
    Vg, Eg = O.gram_eig(X, 1, 6)      # short axis (columns)
    Vc, Ec = O.gram_eig(X, 0, 6)      # long axis (rows), same spectrum for a matrix
    for _, Vs, E, _ in got:
        np.testing.assert_allclose(E, Eg, rtol=1e-10)
        np.testing.assert_allclose(np.abs(np.sum(Vs * Vg, axis=0)), 1.0, atol=1e-6)
    Vl = np.concatenate([g[3] for g in got], axis=0)
    np.testing.assert_allclose(np.abs(np.sum(Vl * Vc, axis=0)), 1.0, atol=1e-9)
    np.testing.assert_allclose(Ec, Eg, rtol=1e-10)
