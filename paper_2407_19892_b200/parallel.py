"""Row-sharded multi-GPU driver for ggm_sparse_precision.

Rows of Ψ_l = V_l diag(λ_l) V_l^T are independent units (each row's top-t needs all n
columns but no other row), so rank r owns rows [begin_r, end_r) of every axis and sweeps all
n columns locally.  V_l and λ_l are replicated (one NCCL broadcast from rank 0); the only
data-path collective is the gather of the per-rank CSR shards.  One process per GPU,
torch.distributed over NCCL (NVLink/NVSwitch) on the GPU box; the same code runs on gloo for
the CPU tests (tests/test_parallel.py) with an injected compute function.
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
