"""Multi-GPU drivers for ggm_sparse_precision.

Plain scheme (row shards): rows of Ψ_l = V_l diag(λ_l) V_l^T are independent units (each
row's top-t needs all n columns but no other row), so rank r owns rows [begin_r, end_r) of
every axis and sweeps all n columns locally.  V_l and λ_l are replicated (one NCCL broadcast
from rank 0); the only data-path collective is the gather of the per-rank CSR shards.

Symmetric scheme (Ψ = Ψᵀ, each unordered block pair once): every rank runs the replicated
seed/ordering phases and its share of the symmetric units, which emit candidates for rows
owned by any rank; one all-to-all moves each candidate bucket to the owner of its target
row, which merges its rows; the CSR rows (in bound order, with their original ids) are then
all-gathered and scattered.

One process per GPU, torch.distributed over NCCL (NVLink/NVSwitch) on the GPU box; the same
code runs on gloo for the CPU tests (tests/test_parallel.py) with injected compute functions.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_rows(n: int, world: int, rank: int):
    """Contiguous balanced row range of rank `rank` (first n % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(int(n), int(world))
    begin = rank * base + min(rank, rem)
    end = begin + base + (1 if rank < rem else 0)
    return begin, end


def broadcast_factors(V: torch.Tensor, lam: torch.Tensor, src: int = 0, group=None):
    """Replicate (V, λ) from `src` to every rank (NCCL broadcast over NVLink)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(V, src, group=group)
        dist.broadcast(lam, src, group=group)
    return V, lam


def gather_topk_csr(col: torch.Tensor, val: torch.Tensor, t_eff: int, n_rows: int,
                    group=None, dst: int = 0):
    """Gather equal-degree (mode 0) CSR shards: every rank holds rows_r x t_eff entries of its
    contiguous row range.  Shards are padded to the largest shard for all_gather_into_tensor;
    returns (row_ptr, col, val) of all n_rows on every rank (callers may use rank dst only)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        rp = torch.arange(0, (n_rows + 1) * t_eff, t_eff, dtype=torch.int64, device=col.device)
        return rp, col, val
    rank = dist.get_rank(group)
    sizes = [shard_rows(n_rows, world, r) for r in range(world)]
    max_rows = max(e - b for b, e in sizes)
    pad = max_rows * t_eff
    c = torch.full((pad,), -1, dtype=col.dtype, device=col.device)
    v = torch.zeros((pad,), dtype=val.dtype, device=val.device)
    c[:col.numel()] = col
    v[:val.numel()] = val
    call = torch.empty((world * pad,), dtype=col.dtype, device=col.device)
    vall = torch.empty((world * pad,), dtype=val.dtype, device=val.device)
    dist.all_gather_into_tensor(call, c, group=group)
    dist.all_gather_into_tensor(vall, v, group=group)
    parts_c, parts_v = [], []
    for r, (b, e) in enumerate(sizes):
        m = (e - b) * t_eff
        parts_c.append(call[r * pad:r * pad + m])
        parts_v.append(vall[r * pad:r * pad + m])
    rp = torch.arange(0, (n_rows + 1) * t_eff, t_eff, dtype=torch.int64, device=col.device)
    del rank
    return rp, torch.cat(parts_c), torch.cat(parts_v)


def sharded_sparse_precision(axes, t: int, compute: Callable | None = None, group=None,
                             gather: bool = True):
    """Per-axis sparse precision graphs with rows sharded over the process group.

    axes    : list of (V, λ) replicated on every rank (device tensors on the GPU path).
    compute : (V, λ, begin, end, t) -> (row_ptr, col, val) local CSR; default is the CUDA
              path (ggm_sparse_precision).  Injected in the CPU tests.
    Returns a list of (row_ptr, col, val) per axis — global if gather else the local shard.
    """
    if compute is None:
        from ._ggm import ggm_sparse_precision

        def compute(V, lam, b, e, tt):
            return ggm_sparse_precision(V, lam, b, e, mode=0, topk=tt)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    out = []
    for V, lam in axes:
        n = V.shape[0]
        b, e = shard_rows(n, world, rank)
        rp, col, val = compute(V, lam, b, e, t)
        if gather:
            out.append(gather_topk_csr(col, val, min(t, n - 1), n, group=group))
        else:
            out.append((rp, col, val))
    return out


def exchange_candidates(key: torch.Tensor, val: torch.Tensor, counts, group=None):
    """All-to-all of key-sorted candidate buckets (bucket r -> rank r).  key: [m], val: [m, 2]
    (int32 views of (source, ψ bits)); counts: per-destination sizes, in rank order.
    Returns the (key, val) this rank received."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return key, val
    send = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=key.device)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    rc = [int(x) for x in recv.tolist()]
    sc = [int(c) for c in counts]
    rkey = torch.empty(sum(rc), dtype=key.dtype, device=key.device)
    rval = torch.empty((sum(rc), 2), dtype=val.dtype, device=val.device)
    dist.all_to_all_single(rkey, key.contiguous(), output_split_sizes=rc, input_split_sizes=sc,
                           group=group)
    dist.all_to_all_single(rval, val.contiguous(), output_split_sizes=rc, input_split_sizes=sc,
                           group=group)
    return rkey, rval


def assemble_rows(row_id: torch.Tensor, col: torch.Tensor, val: torch.Tensor, n: int,
                  t_eff: int, group=None):
    """All-gather the (original row id, t_eff columns, t_eff values) rows every rank merged
    and scatter them into one full CSR (row_ptr = i * t_eff) on every rank."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = col.device
    if world > 1:
        m = torch.tensor([row_id.numel()], dtype=torch.int64, device=dev)
        ms = [torch.empty_like(m) for _ in range(world)]
        dist.all_gather(ms, m, group=group)
        sizes = [int(x.item()) for x in ms]
        mx = max(sizes)
        rid = torch.full((mx,), -1, dtype=torch.int64, device=dev)
        c = torch.zeros((mx * t_eff,), dtype=col.dtype, device=dev)
        v = torch.zeros((mx * t_eff,), dtype=val.dtype, device=dev)
        rid[:row_id.numel()] = row_id
        c[:col.numel()] = col
        v[:val.numel()] = val
        rid_all = [torch.empty_like(rid) for _ in range(world)]
        c_all = [torch.empty_like(c) for _ in range(world)]
        v_all = [torch.empty_like(v) for _ in range(world)]
        dist.all_gather(rid_all, rid, group=group)
        dist.all_gather(c_all, c, group=group)
        dist.all_gather(v_all, v, group=group)
        row_id = torch.cat([r[:sz] for r, sz in zip(rid_all, sizes)])
        col = torch.cat([x[:sz * t_eff] for x, sz in zip(c_all, sizes)])
        val = torch.cat([x[:sz * t_eff] for x, sz in zip(v_all, sizes)])
    if row_id.numel() != n:
        raise RuntimeError(f"assembled {row_id.numel()} rows, expected {n}")
    full_c = torch.empty((n, t_eff), dtype=col.dtype, device=dev)
    full_v = torch.empty((n, t_eff), dtype=val.dtype, device=dev)
    full_c[row_id] = col.view(-1, t_eff)
    full_v[row_id] = val.view(-1, t_eff)
    rp = torch.arange(0, (n + 1) * t_eff, t_eff, dtype=torch.int64, device=dev)
    return rp, full_c.view(-1), full_v.view(-1)


def sharded_symmetric_precision(V, lam, t: int, group=None, shard=None, merge=None,
                                rows_begin=None, gather: bool = True):
    """Distributed symmetric scheme for one axis (include/ggm.h (3b)).

    shard      : (V, λ, t, rank, world) -> (key, val, counts, perm); default libggm:
                 this rank's share of the seed pass (ggm_sym_seed_shard), one all-reduce(MIN)
                 of the n seed values, then ggm_sparse_precision_sym_shard_seeded.
    merge      : (n, t, key, val, perm, row_begin, row_end) -> (row_id, col, val); default
                 libggm ggm_sym_merge.
    rows_begin : (rank) -> first bound-order row owned by rank (default ggm_sym_rows_begin).
    Returns the full CSR (gather) or this rank's (row_id, col, val)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n, k = V.shape
    if shard is None or merge is None or rows_begin is None:
        from . import _ggm as G
        if shard is None:
            def shard(V_, lam_, tt, r, w):
                plan = G.SymShardPlan(n, k, tt, r, w, device=V_.device)
                thr_all = None
                if w > 1:  # sharded seed pass, combined by one all-reduce(MIN) of n floats
                    thr_all = plan.seed(V_, lam_)
                    dist.all_reduce(thr_all, op=dist.ReduceOp.MIN, group=group)
                return plan.run(V_, lam_, thr_all=thr_all)
        if merge is None:
            merge = G.sym_merge
        if rows_begin is None:
            def rows_begin(r):
                return G.sym_rows_begin(n, k, t, r, world)
    key, val, counts, perm = shard(V, lam, t, rank, world)
    rkey, rval = exchange_candidates(key, val, counts, group=group)
    b, e = rows_begin(rank), rows_begin(rank + 1)
    row_id, col, vals = merge(n, t, rkey, rval, perm, b, e)
    if not gather:
        return row_id, col, vals
    return assemble_rows(row_id, col, vals, n, min(t, n - 1), group=group)


def sharded_csr_spectrum(row_ptr, col, val, m: int, k: int, nonparanormal: bool = False,
                         group=None, accumulate: Callable | None = None,
                         eig: Callable | None = None, project: Callable | None = None):
    """Spectrum of a matrix whose rows (the long axis, e.g. 1.25M cells) are sharded over the
    process group, m <= 32768 columns (e.g. genes) — §8(f) row 1, "sharded Gram with one
    all-reduce" (include/ggm.h (1f)).  Every rank passes its own CSR rows.

    G_r = A_r^T A_r (m x m) -> ONE all_reduce(SUM) -> every rank eigensolves G (short-axis V,
    E, W) -> local long-axis rows V_r = A_r W diag(E^-1/2).  For a matrix both axes share E
    (Thm 1).  Returns (V_short replicated, E, V_long local rows).

    accumulate(rp, col, val, m, nonparanormal) -> G, eig(G, k) -> (V, E, W),
    project(rp, col, val, m, W, E, nonparanormal) -> V_r default to the CUDA path; the CPU
    tests inject NumPy versions."""
    if accumulate is None or eig is None or project is None:
        from . import _ggm as G_
        accumulate = accumulate or (lambda rp, c, v, mm, npn: G_.gram_accumulate_csr(
            rp, c, v, mm, npn)[0])
        eig = eig or (lambda Gm, kk: G_.eig_gram(Gm, kk))
        project = project or (lambda rp, c, v, mm, W, E, npn: G_.project_csr(
            rp, c, v, mm, W, E, npn))
    Gm = accumulate(row_ptr, col, val, m, nonparanormal)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(Gm, op=dist.ReduceOp.SUM, group=group)
    V_short, E, W = eig(Gm, k)
    V_long = project(row_ptr, col, val, m, W, E, nonparanormal)
    return V_short, E, V_long
