"""B200-native (sm_100a) hot path of the scalable multi-axis GGM (arXiv 2407.19892).

Public API (thin bindings of libggm.so, include/ggm.h):
  ggm_gram_eig         per-axis Gram spectrum          (Alg. 1 lines 1-4)
  ggm_gram_eig_rsi     at-scale spectrum: randomized subspace iteration (automatic in
                       ggm_gram_eig above 32768 x 32768 Grams)
  ggm_solve_eigvals    Kronecker-sum eigenvalue MLE    (Thm 2, Alg. 1 lines 5-17)
  ggm_grid_marginals   the Thm 2 trace term alone
  ggm_sparse_precision fused V diag(λ) V^T + per-row top-t / threshold (Alg. 1 line 19)
  SymShardPlan / sym_merge / sym_rows_begin  distributed symmetric scheme (one rank's share)
  parallel.sharded_sparse_precision  multi-GPU driver (torch.distributed/NCCL): row shards
                       (plain scheme) or the distributed symmetric scheme with an all-to-all
"""
from ._ggm import (GGMError, SparsePlan, device_supported, ggm_gram_eig, ggm_gram_eig_rsi,
                   ggm_gram_eig_multi, ggm_gram_eig_matrix, ggm_gram_eig_axes, ggm_solve_eigvals_multi, ggm_gram_eig_csr, ggm_nonparanormal,
                   gram_accumulate_csr, eig_gram, project_csr,
                   ggm_grid_marginals,
                   ggm_solve_eigvals, ggm_sparse_precision, ggm_sparse_precision_overall, overall_last_path, overall_last_timing, last_launches, last_stats, last_timing, lib,
                   set_timing, SymShardPlan, sym_merge, sym_rows_begin, wald_edge, wald_threshold,
                   version, EXPORTED, MAX_TOPK)

__all__ = ["GGMError", "SparsePlan", "device_supported", "ggm_gram_eig", "ggm_gram_eig_rsi",
           "ggm_gram_eig_multi", "ggm_gram_eig_matrix", "ggm_gram_eig_axes", "ggm_solve_eigvals_multi", "ggm_gram_eig_csr", "ggm_nonparanormal",
           "gram_accumulate_csr", "eig_gram", "project_csr",
           "ggm_grid_marginals",
           "ggm_solve_eigvals", "ggm_sparse_precision", "ggm_sparse_precision_overall", "overall_last_path", "overall_last_timing", "last_launches", "last_stats", "last_timing", "lib", "set_timing",
           "SymShardPlan", "sym_merge", "sym_rows_begin", "wald_edge", "wald_threshold", "version",
           "EXPORTED", "MAX_TOPK"]
