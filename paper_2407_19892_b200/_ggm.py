"""ctypes binding of libggm.so (include/ggm.h).  Argument marshalling only: every step of
the hot path runs in the library's CUDA kernels.  PyTorch supplies device memory (tensors),
the current CUDA stream and, in ``parallel``, the process groups.

There is no CPU fallback: if libggm.so is missing or the device is not sm_100a the calls
raise.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# GGM_LIB_PATH: alternative build of the same library (same-session A/B experiments, tools/)
_LIB_PATH = os.environ.get("GGM_LIB_PATH") or os.path.join(_PKG, "libggm.so")

GGM_OK = 0
STATUS_NAMES = {
    0: "GGM_OK", 1: "GGM_ERR_INVALID_ARGUMENT", 2: "GGM_ERR_RANK", 3: "GGM_ERR_DOMAIN",
    4: "GGM_ERR_NO_CONVERGENCE", 5: "GGM_ERR_CAPACITY", 6: "GGM_ERR_CUDA",
    7: "GGM_ERR_UNSUPPORTED",
}
MAX_TOPK = 32

# symbols declared in include/ggm.h (checked by tests/test_abi.py)
EXPORTED = [
    "ggm_last_error", "ggm_version", "ggm_device_supported",
    "ggm_gram_eig_workspace", "ggm_gram_eig", "ggm_gram_eig_rsi_workspace", "ggm_gram_eig_rsi",
    "ggm_solve_opts_default", "ggm_solve_eigvals", "ggm_grid_marginals",
    "ggm_sparse_precision_workspace", "ggm_sparse_precision",
    "ggm_set_timing", "ggm_last_timing", "ggm_last_launches", "ggm_last_stats",
    "ggm_sym_rows_begin", "ggm_sparse_precision_sym_shard_workspace",
    "ggm_sparse_precision_sym_shard", "ggm_sym_merge_workspace", "ggm_sym_merge",
    "ggm_wald_edge", "ggm_wald_threshold",
    "ggm_sparse_precision_overall_workspace", "ggm_sparse_precision_overall",
    "ggm_overall_last_path",
    "ggm_gram_eig_multi_workspace", "ggm_gram_eig_multi", "ggm_solve_eigvals_multi",
    "ggm_sym_seed_shard", "ggm_sparse_precision_sym_shard_seeded",
    "ggm_gram_eig_matrix_workspace", "ggm_gram_eig_matrix",
    "ggm_gram_eig_axes_workspace", "ggm_gram_eig_axes",
    "ggm_gram_eig_csr_workspace", "ggm_gram_eig_csr", "ggm_nonparanormal_workspace",
    "ggm_nonparanormal", "ggm_gram_accumulate_csr_workspace", "ggm_gram_accumulate_csr",
    "ggm_eig_gram_workspace", "ggm_eig_gram", "ggm_project_csr_workspace", "ggm_project_csr",
]


class GGMError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        self.status_name = STATUS_NAMES.get(status, str(status))
        super().__init__(f"{self.status_name}: {message}")


class SolveOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("eps_scale", C.c_double),
                ("method", C.c_int), ("gauge", C.c_int), ("trace_tol", C.c_double)]


class SolveInfo(C.Structure):
    _fields_ = [("iterations", C.c_int), ("stationarity", C.c_double), ("nll", C.c_double),
                ("grid_min", C.c_double), ("trace_inconsistency", C.c_double),
                ("floor_active", C.c_int), ("passes", C.c_int), ("kernel_ms", C.c_double)]


class SparsifyOpts(C.Structure):
    _fields_ = [("mode", C.c_int), ("topk", C.c_int), ("tau", C.c_float),
                ("col_chunks", C.c_int), ("symmetric", C.c_int)]


class OverallOpts(C.Structure):
    _fields_ = [("n_edges", C.c_int64), ("downweight", C.c_int), ("min_edges", C.c_int)]


_lib = None


def lib() -> C.CDLL:
    """Load libggm.so (built in-tree by ``paper_2407_19892_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} missing: run `python -m paper_2407_19892_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(_LIB_PATH)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    L.ggm_last_error.restype = C.c_char_p
    L.ggm_version.restype = i32
    L.ggm_device_supported.restype = i32
    L.ggm_gram_eig_workspace.argtypes = [i32, C.POINTER(i64), i32, i32, C.POINTER(C.c_size_t)]
    L.ggm_gram_eig.argtypes = [vp, i32, C.POINTER(i64), i32, i32, vp, vp, C.POINTER(C.c_double),
                               vp, C.c_size_t, vp]
    L.ggm_gram_eig_rsi_workspace.argtypes = [i32, C.POINTER(i64), i32, i32, i32,
                                             C.POINTER(C.c_size_t)]
    L.ggm_gram_eig_rsi.argtypes = [vp, i32, C.POINTER(i64), i32, i32, i32, i32, C.c_double,
                                   C.c_uint64, vp, vp, C.POINTER(C.c_double), C.POINTER(i32),
                                   C.POINTER(C.c_double), vp, C.c_size_t, vp]
    L.ggm_solve_opts_default.argtypes = [C.POINTER(SolveOpts)]
    L.ggm_solve_opts_default.restype = None
    L.ggm_solve_eigvals.argtypes = [i32, C.POINTER(i32), vp, C.POINTER(SolveOpts), vp,
                                    C.POINTER(SolveInfo), vp]
    L.ggm_grid_marginals.argtypes = [i32, C.POINTER(i32), vp, vp, C.POINTER(C.c_double), vp]
    L.ggm_sparse_precision_workspace.argtypes = [i64, i32, i64, i64, C.POINTER(SparsifyOpts), i64,
                                                 C.POINTER(C.c_size_t)]
    L.ggm_sparse_precision.argtypes = [i64, i32, vp, vp, i64, i64, C.POINTER(SparsifyOpts), vp, vp,
                                       vp, i64, C.POINTER(i64), vp, C.c_size_t, vp]
    L.ggm_set_timing.argtypes = [i32]
    L.ggm_set_timing.restype = None
    L.ggm_last_timing.argtypes = [C.POINTER(C.c_float)]
    L.ggm_last_timing.restype = None
    L.ggm_last_launches.restype = i32
    L.ggm_last_stats.argtypes = [C.POINTER(C.c_double)]
    L.ggm_last_stats.restype = None
    L.ggm_wald_edge.argtypes = [C.c_double, i64, C.c_double, i64, C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.ggm_wald_edge.restype = i32
    L.ggm_wald_threshold.argtypes = [i64, C.c_double, C.c_double, i64, C.POINTER(C.c_double)]
    L.ggm_wald_threshold.restype = i32
    L.ggm_sym_rows_begin.argtypes = [i64, i32, C.POINTER(SparsifyOpts), i32, i32]
    L.ggm_sym_rows_begin.restype = i64
    L.ggm_sparse_precision_sym_shard_workspace.argtypes = [i64, i32, C.POINTER(SparsifyOpts),
                                                           C.POINTER(C.c_size_t)]
    L.ggm_sparse_precision_sym_shard.argtypes = [i64, i32, vp, vp, C.POINTER(SparsifyOpts), i32,
                                                 i32, vp, vp, i64, C.POINTER(i64), vp, vp,
                                                 C.c_size_t, vp]
    L.ggm_gram_eig_matrix_workspace.argtypes = [i64, i64, i32, i32, C.POINTER(C.c_size_t)]
    L.ggm_gram_eig_matrix.argtypes = [vp, i64, i64, i32, i32, vp, vp, vp, vp,
                                      C.POINTER(C.c_double), vp, C.c_size_t, vp]
    L.ggm_gram_eig_axes_workspace.argtypes = [i32, C.POINTER(i64), C.POINTER(i32),
                                              C.POINTER(C.c_size_t)]
    L.ggm_gram_eig_axes.argtypes = [vp, i32, C.POINTER(i64), C.POINTER(i32), C.POINTER(vp),
                                    C.POINTER(vp), C.POINTER(C.c_double), vp, C.c_size_t, vp]
    L.ggm_gram_eig_axes_workspace.restype = i32
    L.ggm_gram_eig_axes.restype = i32
    L.ggm_gram_eig_matrix_workspace.restype = i32
    L.ggm_gram_eig_matrix.restype = i32
    L.ggm_sym_seed_shard.argtypes = [i64, i32, vp, vp, C.POINTER(SparsifyOpts), i32, i32, vp, vp,
                                     C.c_size_t, vp]
    L.ggm_sparse_precision_sym_shard_seeded.argtypes = [i64, i32, vp, vp, C.POINTER(SparsifyOpts),
                                                        i32, i32, vp, vp, vp, i64, C.POINTER(i64),
                                                        vp, vp, C.c_size_t, vp]
    L.ggm_sym_merge_workspace.argtypes = [i64, C.POINTER(C.c_size_t)]
    L.ggm_sym_merge.argtypes = [i64, i32, vp, vp, i64, vp, i64, i64, vp, vp, vp, vp, C.c_size_t, vp]
    L.ggm_sparse_precision_overall_workspace.argtypes = [i64, i32, C.POINTER(OverallOpts), i64,
                                                         C.POINTER(C.c_size_t)]
    L.ggm_sparse_precision_overall.argtypes = [i64, i32, vp, vp, C.POINTER(OverallOpts), i64, vp,
                                               vp, vp, i64, C.POINTER(i64), vp, C.c_size_t, vp]
    L.ggm_overall_last_path.argtypes = [C.POINTER(i64), C.POINTER(C.c_float)]
    L.ggm_gram_eig_multi_workspace.argtypes = [i32, C.POINTER(i32), C.POINTER(i64), C.POINTER(i32),
                                               i32, C.POINTER(C.c_size_t)]
    L.ggm_gram_eig_multi.argtypes = [i32, C.POINTER(vp), C.POINTER(i32), C.POINTER(i64),
                                     C.POINTER(i32), i32, vp, vp, C.POINTER(C.c_double), vp,
                                     C.c_size_t, vp]
    L.ggm_solve_eigvals_multi.argtypes = [i32, C.POINTER(i32), vp, i32, C.POINTER(i32),
                                          C.POINTER(i32), C.POINTER(SolveOpts), vp,
                                          C.POINTER(SolveInfo), vp]
    L.ggm_overall_last_path.restype = i32
    L.ggm_gram_eig_csr_workspace.argtypes = [i64, i64, i64, i32, i32, C.POINTER(C.c_size_t)]
    L.ggm_gram_eig_csr.argtypes = [i64, i64, i64, vp, vp, vp, i32, i32, i32, i32, C.c_double,
                                   C.c_uint64, vp, vp, C.POINTER(C.c_double), C.POINTER(i32),
                                   C.POINTER(C.c_double), vp, C.c_size_t, vp]
    L.ggm_nonparanormal_workspace.argtypes = [i32, C.POINTER(i64), i32, C.POINTER(C.c_size_t)]
    L.ggm_nonparanormal.argtypes = [vp, i32, C.POINTER(i64), i32, vp, vp, C.c_size_t, vp]
    L.ggm_gram_accumulate_csr_workspace.argtypes = [i64, i64, i64, C.POINTER(C.c_size_t)]
    L.ggm_gram_accumulate_csr.argtypes = [i64, i64, i64, vp, vp, vp, i32, vp, i32,
                                          C.POINTER(C.c_double), vp, C.c_size_t, vp]
    L.ggm_eig_gram_workspace.argtypes = [i64, i32, C.POINTER(C.c_size_t)]
    L.ggm_eig_gram.argtypes = [i64, vp, i32, vp, vp, vp, vp, C.c_size_t, vp]
    L.ggm_project_csr_workspace.argtypes = [i64, i64, i64, i32, C.POINTER(C.c_size_t)]
    L.ggm_project_csr.argtypes = [i64, i64, i64, vp, vp, vp, i32, i32, vp, vp, vp, vp,
                                  C.c_size_t, vp]
    for name in ("ggm_gram_accumulate_csr_workspace", "ggm_gram_accumulate_csr",
                 "ggm_eig_gram_workspace", "ggm_eig_gram", "ggm_project_csr_workspace",
                 "ggm_project_csr", "ggm_gram_eig_csr_workspace", "ggm_gram_eig_csr", "ggm_nonparanormal_workspace",
                 "ggm_nonparanormal", "ggm_gram_eig_multi_workspace", "ggm_gram_eig_multi", "ggm_solve_eigvals_multi",
                 "ggm_sparse_precision_overall_workspace", "ggm_sparse_precision_overall",
                 "ggm_gram_eig_workspace", "ggm_gram_eig", "ggm_solve_eigvals",
                 "ggm_gram_eig_rsi_workspace", "ggm_gram_eig_rsi",
                 "ggm_grid_marginals", "ggm_sparse_precision_workspace", "ggm_sparse_precision",
                 "ggm_sparse_precision_sym_shard_workspace", "ggm_sparse_precision_sym_shard",
                 "ggm_sym_merge_workspace", "ggm_sym_merge", "ggm_sym_seed_shard",
                 "ggm_sparse_precision_sym_shard_seeded"):
        getattr(L, name).restype = i32
    _lib = L
    return L


def _check(status: int):
    if status != GGM_OK:
        msg = lib().ggm_last_error()
        raise GGMError(status, msg.decode() if msg else "")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def _require_cuda(t: torch.Tensor, dtype, name):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def device_supported() -> bool:
    return bool(lib().ggm_device_supported())


def version() -> int:
    return int(lib().ggm_version())


# --------------------------------------------------------------------------- (1) gram_eig

def ggm_gram_eig(X: torch.Tensor, axis: int, k: int, stream=None):
    """Top-k eigenpairs of S_axis = mat_axis(X) mat_axis(X)^T (Alg. 1 lines 1-4).
    Returns (V float32 d x k, E float64 k descending, trace_S float)."""
    _require_cuda(X, torch.float32, "X")
    shape = (C.c_int64 * X.dim())(*X.shape)
    nbytes = C.c_size_t(0)
    _check(lib().ggm_gram_eig_workspace(X.dim(), shape, axis, k, C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=X.device)
    d = X.shape[axis]
    V = torch.empty((d, k), dtype=torch.float32, device=X.device)
    E = torch.empty((k,), dtype=torch.float64, device=X.device)
    tr = C.c_double(0.0)
    _check(lib().ggm_gram_eig(_ptr(X), X.dim(), shape, axis, k, _ptr(V), _ptr(E), C.byref(tr),
                              _ptr(ws), nbytes.value, _stream(stream)))
    return V, E, tr.value


def ggm_gram_eig_axes(X: torch.Tensor, ks, stream=None):
    """Every axis of X at once (include/ggm.h (1h)): [(V_a, E_a)], trace."""
    _require_cuda(X, torch.float32, "X")
    nd = X.dim()
    if len(ks) != nd:
        raise ValueError("one k per axis")
    shp = (C.c_int64 * nd)(*X.shape)
    kk = (C.c_int32 * nd)(*[int(k) for k in ks])
    nbytes = C.c_size_t(0)
    _check(lib().ggm_gram_eig_axes_workspace(nd, shp, kk, C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=X.device)
    Vs = [torch.empty((X.shape[a], int(ks[a])), dtype=torch.float32, device=X.device)
          for a in range(nd)]
    Es = [torch.empty((int(ks[a]),), dtype=torch.float64, device=X.device) for a in range(nd)]
    vp_arr = (C.c_void_p * nd)(*[_ptr(v) for v in Vs])
    ep_arr = (C.c_void_p * nd)(*[_ptr(e) for e in Es])
    tr = C.c_double(0.0)
    _check(lib().ggm_gram_eig_axes(_ptr(X), nd, shp, kk, vp_arr, ep_arr, C.byref(tr), _ptr(ws),
                                   nbytes.value, _stream(stream)))
    return list(zip(Vs, Es)), tr.value


def ggm_gram_eig_matrix(X: torch.Tensor, k0: int, k1: int, stream=None):
    """Both axes of a matrix from one Gram + one eigensolve (include/ggm.h (1g)).
    Returns (V0, E0, V1, E1, trace)."""
    _require_cuda(X, torch.float32, "X")
    if X.dim() != 2:
        raise ValueError("X must be a matrix")
    d0, d1 = X.shape
    nbytes = C.c_size_t(0)
    _check(lib().ggm_gram_eig_matrix_workspace(d0, d1, int(k0), int(k1), C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=X.device)
    V0 = torch.empty((d0, k0), dtype=torch.float32, device=X.device)
    V1 = torch.empty((d1, k1), dtype=torch.float32, device=X.device)
    E0 = torch.empty((k0,), dtype=torch.float64, device=X.device)
    E1 = torch.empty((k1,), dtype=torch.float64, device=X.device)
    tr = C.c_double(0.0)
    _check(lib().ggm_gram_eig_matrix(_ptr(X), d0, d1, int(k0), int(k1), _ptr(V0), _ptr(E0),
                                     _ptr(V1), _ptr(E1), C.byref(tr), _ptr(ws), nbytes.value,
                                     _stream(stream)))
    return V0, E0, V1, E1, tr.value


def ggm_gram_eig_rsi(X: torch.Tensor, axis: int, k: int, oversample: int = 0,
                     max_iter: int = 200, tol: float = 1e-13, seed: int = 0x2407198920240728,
                     stream=None):
    """At-scale top-k eigenpairs of S_axis by randomized subspace iteration (include/ggm.h
    (1b)).  Returns (V, E, trace_S, iterations, last relative change of the Ritz values)."""
    _require_cuda(X, torch.float32, "X")
    shape = (C.c_int64 * X.dim())(*X.shape)
    nbytes = C.c_size_t(0)
    _check(lib().ggm_gram_eig_rsi_workspace(X.dim(), shape, axis, k, oversample, C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=X.device)
    d = X.shape[axis]
    V = torch.empty((d, k), dtype=torch.float32, device=X.device)
    E = torch.empty((k,), dtype=torch.float64, device=X.device)
    tr, it, ch = C.c_double(0.0), C.c_int(0), C.c_double(0.0)
    _check(lib().ggm_gram_eig_rsi(_ptr(X), X.dim(), shape, axis, k, oversample, max_iter, tol,
                                  C.c_uint64(seed), _ptr(V), _ptr(E), C.byref(tr), C.byref(it),
                                  C.byref(ch), _ptr(ws), nbytes.value, _stream(stream)))
    return V, E, tr.value, it.value, ch.value


def ggm_gram_eig_multi(tensors, axis_pos, k: int, stream=None):
    """Shared-axis spectrum (Alg. 1 line 2): tensors = per-modality fp32 CUDA tensors
    (None where the axis is absent), axis_pos[g] = the axis' position in modality g or -1.
    Returns (V float32 d x k, E float64 k descending, ||D_l||_F^2)."""
    M = len(tensors)
    if len(axis_pos) != M:
        raise ValueError("axis_pos length != number of modalities")
    dev = None
    for X, p in zip(tensors, axis_pos):
        if p >= 0:
            _require_cuda(X, torch.float32, "X")
            dev = X.device
    if dev is None:
        raise ValueError("the axis occurs in no modality")
    nd = [X.dim() if X is not None else 1 for X in tensors]
    flat = []
    for X in tensors:
        flat.extend(list(X.shape) if X is not None else [1])
    ndim = (C.c_int * M)(*nd)
    shapes = (C.c_int64 * len(flat))(*flat)
    pos = (C.c_int * M)(*[int(p) for p in axis_pos])
    ptrs = (C.c_void_p * M)(*[X.data_ptr() if X is not None else None for X in tensors])
    nbytes = C.c_size_t(0)
    _check(lib().ggm_gram_eig_multi_workspace(M, ndim, shapes, pos, int(k), C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=dev)
    d = next(X.shape[p] for X, p in zip(tensors, axis_pos) if p >= 0)
    V = torch.empty((d, k), dtype=torch.float32, device=dev)
    E = torch.empty((k,), dtype=torch.float64, device=dev)
    tr = C.c_double(0.0)
    _check(lib().ggm_gram_eig_multi(M, ptrs, ndim, shapes, pos, int(k), _ptr(V), _ptr(E),
                                    C.byref(tr), _ptr(ws), nbytes.value, _stream(stream)))
    return V, E, tr.value


def ggm_gram_eig_csr(row_ptr: torch.Tensor, col: torch.Tensor, val: torch.Tensor, m: int, k: int,
                     nonparanormal: bool = False, oversample: int = 0, max_iter: int = 200,
                     tol: float = 1e-13, seed: int = 0x2407198920240728, stream=None):
    """Spectrum of a sparse unfolding given as CSR (d = len(row_ptr) - 1 rows, m columns),
    optionally COCA-transformed in its sparse + rank-one form (include/ggm.h (1d)).
    Returns (V, E, trace, iterations, last Ritz change)."""
    _require_cuda(row_ptr, torch.int64, "row_ptr")
    _require_cuda(col, torch.int32, "col")
    _require_cuda(val, torch.float32, "val")
    d = row_ptr.numel() - 1
    nnz = val.numel()
    nbytes = C.c_size_t(0)
    _check(lib().ggm_gram_eig_csr_workspace(d, int(m), nnz, int(k), int(oversample),
                                            C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=val.device)
    V = torch.empty((d, k), dtype=torch.float32, device=val.device)
    E = torch.empty((k,), dtype=torch.float64, device=val.device)
    tr, it, ch = C.c_double(0.0), C.c_int(0), C.c_double(0.0)
    _check(lib().ggm_gram_eig_csr(d, int(m), nnz, _ptr(row_ptr), _ptr(col), _ptr(val), int(k),
                                  int(bool(nonparanormal)), int(oversample), int(max_iter),
                                  float(tol), C.c_uint64(seed), _ptr(V), _ptr(E), C.byref(tr),
                                  C.byref(it), C.byref(ch), _ptr(ws), nbytes.value,
                                  _stream(stream)))
    return V, E, tr.value, it.value, ch.value


def gram_accumulate_csr(row_ptr, col, val, m: int, nonparanormal: bool = False, G=None,
                        stream=None):
    """G (+)= A_r^T A_r for this rank's CSR rows (include/ggm.h (1f)); returns (G, ||A_r||^2).
    G is fp64 m x m column-major with the LOWER triangle filled."""
    _require_cuda(row_ptr, torch.int64, "row_ptr")
    _require_cuda(col, torch.int32, "col")
    _require_cuda(val, torch.float32, "val")
    d, nnz = row_ptr.numel() - 1, val.numel()
    acc = G is not None
    if G is None:
        G = torch.zeros((m, m), dtype=torch.float64, device=val.device)
    nbytes = C.c_size_t(0)
    _check(lib().ggm_gram_accumulate_csr_workspace(d, int(m), nnz, C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=val.device)
    fro = C.c_double(0.0)
    _check(lib().ggm_gram_accumulate_csr(d, int(m), nnz, _ptr(row_ptr), _ptr(col), _ptr(val),
                                         int(bool(nonparanormal)), _ptr(G), int(acc),
                                         C.byref(fro), _ptr(ws), nbytes.value, _stream(stream)))
    return G, fro.value


def eig_gram(G: torch.Tensor, k: int, stream=None):
    """Top-k eigenpairs of an (all-reduced) Gram; G is overwritten.  Returns (V fp32 m x k,
    E fp64 k descending, W fp64 for ggm_project_csr)."""
    _require_cuda(G, torch.float64, "G")
    m = G.shape[0]
    nbytes = C.c_size_t(0)
    _check(lib().ggm_eig_gram_workspace(m, int(k), C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=G.device)
    V = torch.empty((m, k), dtype=torch.float32, device=G.device)
    E = torch.empty((k,), dtype=torch.float64, device=G.device)
    W = torch.empty((k, m), dtype=torch.float64, device=G.device)   # column-major m x k
    _check(lib().ggm_eig_gram(m, _ptr(G), int(k), _ptr(V), _ptr(E), _ptr(W), _ptr(ws),
                              nbytes.value, _stream(stream)))
    return V, E, W


def project_csr(row_ptr, col, val, m: int, W: torch.Tensor, E: torch.Tensor,
                nonparanormal: bool = False, stream=None) -> torch.Tensor:
    """This rank's rows of the long-axis factor A_r W diag(E^-1/2) (fp32 d x k)."""
    _require_cuda(row_ptr, torch.int64, "row_ptr")
    _require_cuda(col, torch.int32, "col")
    _require_cuda(val, torch.float32, "val")
    _require_cuda(W, torch.float64, "W")
    _require_cuda(E, torch.float64, "E")
    d, nnz, k = row_ptr.numel() - 1, val.numel(), E.numel()
    if col.numel() != nnz:
        raise ValueError("col and val must have the same length")
    if W.numel() != k * int(m):
        raise ValueError(f"W must hold k x m = {k} x {m} values (as returned by eig_gram)")
    nbytes = C.c_size_t(0)
    _check(lib().ggm_project_csr_workspace(d, int(m), nnz, int(k), C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=val.device)
    V = torch.empty((d, k), dtype=torch.float32, device=val.device)
    _check(lib().ggm_project_csr(d, int(m), nnz, _ptr(row_ptr), _ptr(col), _ptr(val),
                                 int(bool(nonparanormal)), int(k), _ptr(W), _ptr(E), _ptr(V),
                                 _ptr(ws), nbytes.value, _stream(stream)))
    return V


def ggm_nonparanormal(X: torch.Tensor, axis: int, stream=None) -> torch.Tensor:
    """COCA transform of X for `axis` (include/ggm.h (1e)); same shape as X."""
    _require_cuda(X, torch.float32, "X")
    shape = (C.c_int64 * X.dim())(*X.shape)
    nbytes = C.c_size_t(0)
    _check(lib().ggm_nonparanormal_workspace(X.dim(), shape, int(axis), C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=X.device)
    out = torch.empty_like(X)
    _check(lib().ggm_nonparanormal(_ptr(X), X.dim(), shape, int(axis), _ptr(out), _ptr(ws),
                                   nbytes.value, _stream(stream)))
    return out


# --------------------------------------------------------------------------- (2) solve

def ggm_solve_eigvals(E: torch.Tensor, ks, tol: float = 1e-7, max_iter: int = 20000,
                      gauge: int = 0, eps_scale: float = 1e-10, method: int = 0,
                      trace_tol: float = 1e-8, stream=None, out=None):
    """Eigenvalue MLE of Thm 2 on the k-grid (Alg. 1 lines 5-17) over Lemma 6's domain
    λ >= ε (include/ggm.h (2), reading T).  E: float64 CUDA tensor, axis-concatenated
    (sum(ks)).  Returns (lambda float64 sum(ks), info dict).  With out=(tensor,) the last
    iterate is written there even when GGM_ERR_NO_CONVERGENCE is raised."""
    _require_cuda(E, torch.float64, "E")
    ks = [int(k) for k in ks]
    if E.numel() != sum(ks):
        raise ValueError("E length != sum(ks)")
    karr = (C.c_int * len(ks))(*ks)
    o = SolveOpts()
    lib().ggm_solve_opts_default(C.byref(o))
    o.tol, o.max_iter, o.gauge, o.eps_scale, o.method = tol, max_iter, gauge, eps_scale, method
    o.trace_tol = trace_tol
    lam = out[0] if out is not None else torch.empty_like(E)
    info = SolveInfo()
    _check(lib().ggm_solve_eigvals(len(ks), karr, _ptr(E), C.byref(o), _ptr(lam), C.byref(info),
                                   _stream(stream)))
    return lam, {f: getattr(info, f) for f, _ in SolveInfo._fields_}


def ggm_solve_eigvals_multi(E: torch.Tensor, ks, modalities, tol: float = 1e-7,
                            max_iter: int = 20000, gauge: int = 0, method: int = 0,
                            eps_scale: float = 1e-10, trace_tol: float = 1e-8, stream=None):
    """Multi-modal eigenvalue MLE (Thm 2 with Σ_γ): E axis-concatenated over the global
    axes (ranks ks), modalities = lists of global axis ids.  Returns (lambda, info)."""
    _require_cuda(E, torch.float64, "E")
    ks = [int(k) for k in ks]
    if E.numel() != sum(ks):
        raise ValueError("E length != sum(ks)")
    ptr = [0]
    axes = []
    for mod in modalities:
        axes.extend(int(a) for a in mod)
        ptr.append(len(axes))
    o = SolveOpts()
    lib().ggm_solve_opts_default(C.byref(o))
    o.tol, o.max_iter, o.gauge, o.method = tol, max_iter, gauge, method
    o.eps_scale, o.trace_tol = eps_scale, trace_tol
    lam = torch.empty_like(E)
    info = SolveInfo()
    _check(lib().ggm_solve_eigvals_multi(len(ks), (C.c_int * len(ks))(*ks), _ptr(E),
                                         len(modalities), (C.c_int * len(ptr))(*ptr),
                                         (C.c_int * max(len(axes), 1))(*axes), C.byref(o),
                                         _ptr(lam), C.byref(info), _stream(stream)))
    return lam, {f: getattr(info, f) for f, _ in SolveInfo._fields_}


def ggm_grid_marginals(lam: torch.Tensor, ks, with_logsum: bool = False, stream=None):
    """g_l[i] = Σ_{j: j_l = i} 1/s_j (the Thm 2 trace term); optional Σ log s."""
    _require_cuda(lam, torch.float64, "lam")
    ks = [int(k) for k in ks]
    karr = (C.c_int * len(ks))(*ks)
    g = torch.empty_like(lam)
    ls = C.c_double(0.0)
    _check(lib().ggm_grid_marginals(len(ks), karr, _ptr(lam), _ptr(g),
                                    C.byref(ls) if with_logsum else None, _stream(stream)))
    return (g, ls.value) if with_logsum else g


# --------------------------------------------------------------------------- (3) sparse

class SparsePlan:
    """Workspace + output buffers for repeated ggm_sparse_precision calls (bench loop)."""

    def __init__(self, n, k, row_begin, row_end, mode=0, topk=10, tau=0.0, col_chunks=0,
                 capacity=None, device="cuda", symmetric=0):
        self.n, self.k, self.row_begin, self.row_end = int(n), int(k), int(row_begin), int(row_end)
        self.opts = SparsifyOpts(int(mode), int(topk), float(tau), int(col_chunks),
                                 int(symmetric))
        rows = self.row_end - self.row_begin
        self.t_eff = min(int(topk), self.n - 1)
        if capacity is None:
            capacity = rows * self.t_eff if mode == 0 else max(rows * 16, 1024)
        self.capacity = int(capacity)
        nbytes = C.c_size_t(0)
        _check(lib().ggm_sparse_precision_workspace(self.n, self.k, self.row_begin, self.row_end,
                                                    C.byref(self.opts), self.capacity,
                                                    C.byref(nbytes)))
        self.ws_bytes = nbytes.value
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=device)
        self.row_ptr = torch.empty(rows + 1, dtype=torch.int64, device=device)
        self.col = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=device)
        self.val = torch.empty(max(self.capacity, 1), dtype=torch.float32, device=device)

    def run(self, V: torch.Tensor, lam: torch.Tensor, stream=None) -> int:
        _require_cuda(V, torch.float32, "V")
        _require_cuda(lam, torch.float64, "lam")
        if V.shape != (self.n, self.k) or lam.numel() != self.k:
            raise ValueError("V/lam shape mismatch with plan")
        nnz = C.c_int64(0)
        st = lib().ggm_sparse_precision(self.n, self.k, _ptr(V), _ptr(lam), self.row_begin,
                                        self.row_end, C.byref(self.opts), _ptr(self.row_ptr),
                                        _ptr(self.col), _ptr(self.val), self.capacity,
                                        C.byref(nnz), _ptr(self.ws), self.ws_bytes,
                                        _stream(stream))
        if st != GGM_OK:
            try:
                _check(st)
            except GGMError as e:
                e.required = int(nnz.value)
                raise
        return int(nnz.value)


def ggm_sparse_precision(V: torch.Tensor, lam: torch.Tensor, row_begin: int = 0,
                         row_end: int | None = None, mode: int = 0, topk: int = 10,
                         tau: float = 0.0, col_chunks: int = 0, capacity: int | None = None,
                         stream=None, symmetric: int = 0):
    """Fused thresh[V diag(λ) V^T] for rows [row_begin,row_end) (Alg. 1 line 19).
    Returns CSR (row_ptr int64, col int32, val float32) on the device.  Mode 1 retries once
    with the required capacity (two-call protocol)."""
    n, k = V.shape
    if row_end is None:
        row_end = n
    plan = SparsePlan(n, k, row_begin, row_end, mode, topk, tau, col_chunks, capacity,
                      device=V.device, symmetric=symmetric)
    for attempt in range(3):
        try:
            nnz = plan.run(V, lam, stream)
            break
        except GGMError as e:
            if e.status != 5 or attempt == 2:
                raise
            # two-call protocol; the slack covers entries within rounding of tau whose side of
            # the threshold depends on the scheme the larger workspace selects
            plan = SparsePlan(n, k, row_begin, row_end, mode, topk, tau, col_chunks,
                              max(int(e.required * 1.01) + 4096, 1), device=V.device,
                              symmetric=symmetric)
    return plan.row_ptr, plan.col[:nnz], plan.val[:nnz]


def ggm_sparse_precision_overall(V: torch.Tensor, lam: torch.Tensor, n_edges: int,
                                 downweight: bool = False, min_edges: int = 0,
                                 cand_capacity: int | None = None, capacity: int | None = None,
                                 stream=None, return_caps: bool = False):
    """Whole-graph edge rules (include/ggm.h (3c)): the n_edges best undirected
    edges by |psi| (or |psi|/sqrt(w_i w_j), downweight) plus each vertex's min_edges best.
    Returns the symmetric CSR (row_ptr, col, val) (+ the (cand_capacity, capacity) that
    succeeded when return_caps).  Retries on either capacity error."""
    _require_cuda(V, torch.float32, "V")
    _require_cuda(lam, torch.float64, "lam")
    n, k = V.shape
    o = OverallOpts(int(n_edges), int(bool(downweight)), int(min_edges))
    if cand_capacity is None:
        cand_capacity = 4 * int(n_edges) + 2 * n * int(min_edges) + 1024
    if capacity is None:
        capacity = 2 * int(n_edges) + 2 * n * int(min_edges)
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=V.device)
    for _ in range(4):
        nbytes = C.c_size_t(0)
        _check(lib().ggm_sparse_precision_overall_workspace(n, k, C.byref(o), int(cand_capacity),
                                                            C.byref(nbytes)))
        ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=V.device)
        col = torch.empty(max(capacity, 1), dtype=torch.int32, device=V.device)
        val = torch.empty(max(capacity, 1), dtype=torch.float32, device=V.device)
        nnz = C.c_int64(0)
        st = lib().ggm_sparse_precision_overall(n, k, _ptr(V), _ptr(lam), C.byref(o),
                                                int(cand_capacity), _ptr(row_ptr), _ptr(col),
                                                _ptr(val), int(capacity), C.byref(nnz), _ptr(ws),
                                                nbytes.value, _stream(stream))
        if st == 5 and nnz.value < 0:
            cand_capacity = -int(nnz.value)
            continue
        if st == 5:
            capacity = int(nnz.value)
            continue
        _check(st)
        out = (row_ptr, col[:nnz.value], val[:nnz.value])
        return out + ((int(cand_capacity), int(capacity)),) if return_caps else out
    raise GGMError(5, "capacity retries exhausted")


def overall_last_path():
    """(path, saturated rows) of the last ggm_sparse_precision_overall call on this thread:
    0 lists only, 2 lists + saturated block, 1 histogram + threshold pass."""
    sat = C.c_int64(0)
    ms = (C.c_float * 5)()
    p = lib().ggm_overall_last_path(C.byref(sat), ms)
    return int(p), int(sat.value)


def overall_last_timing():
    """Phase times (ms) of the last overall call when set_timing(True): row masses,
    top-t1 lists, bound + saturation, candidate pass, ranking + CSR."""
    sat = C.c_int64(0)
    ms = (C.c_float * 5)()
    lib().ggm_overall_last_path(C.byref(sat), ms)
    return dict(zip(("mass", "lists", "bound", "candidates", "rank_csr"), [float(x) for x in ms]))


def wald_edge(psi: float, d_rest: int, sigma2: float, n_tests: int):
    """(z, p_raw, p_bonferroni) of one edge under the empty-graph null (Thm 5 / Cor. 10)."""
    z, pr, pb = C.c_double(), C.c_double(), C.c_double()
    _check(lib().ggm_wald_edge(float(psi), int(d_rest), float(sigma2), int(n_tests), C.byref(z),
                               C.byref(pr), C.byref(pb)))
    return z.value, pr.value, pb.value


def wald_threshold(d_rest: int, sigma2: float = 1.0, alpha: float = 0.05, n_tests: int = 1) -> float:
    """Critical magnitude: |psi| > tau <=> Bonferroni-corrected p < alpha."""
    tau = C.c_double()
    _check(lib().ggm_wald_threshold(int(d_rest), float(sigma2), float(alpha), int(n_tests),
                                    C.byref(tau)))
    return tau.value


def sym_rows_begin(n: int, k: int, topk: int, rank: int, nranks: int) -> int:
    """First bound-order row owned by `rank` in the distributed symmetric scheme."""
    o = SparsifyOpts(0, int(topk), 0.0, 0, 1)
    r = lib().ggm_sym_rows_begin(int(n), int(k), C.byref(o), int(rank), int(nranks))
    if r < 0:
        raise GGMError(1, "ggm_sym_rows_begin: invalid arguments")
    return int(r)


class SymShardPlan:
    """Workspace for repeated ggm_sparse_precision_sym_shard calls (one rank's share of the
    distributed symmetric scheme, include/ggm.h (3b))."""

    def __init__(self, n, k, topk, rank, nranks, cand_capacity=None, device="cuda"):
        self.n, self.k, self.t = int(n), int(k), int(topk)
        self.rank, self.nranks = int(rank), int(nranks)
        self.opts = SparsifyOpts(0, self.t, 0.0, 0, 1)
        nb = C.c_size_t(0)
        _check(lib().ggm_sparse_precision_sym_shard_workspace(self.n, self.k, C.byref(self.opts),
                                                              C.byref(nb)))
        self.ws = torch.empty(max(nb.value, 256), dtype=torch.uint8, device=device)
        cap = cand_capacity if cand_capacity is not None else self.n * max(8 * self.t, 64)
        self.cap = int(cap)
        self.key = torch.empty(self.cap, dtype=torch.int32, device=device)
        self.val = torch.empty((self.cap, 2), dtype=torch.int32, device=device)
        self.perm = torch.empty(self.n, dtype=torch.int32, device=device)
        self.counts = (C.c_int64 * self.nranks)()

    def seed(self, V: torch.Tensor, lam: torch.Tensor, stream=None) -> torch.Tensor:
        """This rank's share of the sharded seed pass: raw seed values of its row blocks,
        +inf elsewhere (combine the ranks' arrays with an element-wise minimum)."""
        _require_cuda(V, torch.float32, "V")
        _require_cuda(lam, torch.float64, "lam")
        thr = torch.empty(self.n, dtype=torch.float32, device=V.device)
        _check(lib().ggm_sym_seed_shard(self.n, self.k, _ptr(V), _ptr(lam), C.byref(self.opts),
                                        self.rank, self.nranks, _ptr(thr), _ptr(self.ws),
                                        self.ws.numel(), _stream(stream)))
        return thr

    def run(self, V: torch.Tensor, lam: torch.Tensor, stream=None, thr_all=None):
        """Returns (key, val, counts, perm): this rank's candidates sorted by target row,
        counts per destination rank (list), bound order -> original id.  thr_all: the
        combined sharded seed (skips this rank's own full seed pass)."""
        _require_cuda(V, torch.float32, "V")
        _require_cuda(lam, torch.float64, "lam")
        if thr_all is None:
            st = lib().ggm_sparse_precision_sym_shard(
                self.n, self.k, _ptr(V), _ptr(lam), C.byref(self.opts), self.rank, self.nranks,
                _ptr(self.key), _ptr(self.val), self.cap, self.counts, _ptr(self.perm),
                _ptr(self.ws), self.ws.numel(), _stream(stream))
        else:
            _require_cuda(thr_all, torch.float32, "thr_all")
            st = lib().ggm_sparse_precision_sym_shard_seeded(
                self.n, self.k, _ptr(V), _ptr(lam), C.byref(self.opts), self.rank, self.nranks,
                _ptr(thr_all), _ptr(self.key), _ptr(self.val), self.cap, self.counts,
                _ptr(self.perm), _ptr(self.ws), self.ws.numel(), _stream(stream))
        _check(st)
        counts = [int(c) for c in self.counts]
        tot = sum(counts)
        return self.key[:tot], self.val[:tot], counts, self.perm


def sym_merge(n: int, t: int, key: torch.Tensor, val: torch.Tensor, perm: torch.Tensor,
              row_begin: int, row_end: int, stream=None):
    """Merge received candidates of bound-order rows [row_begin, row_end): returns
    (row_id int64 [rows], col int32 [rows*t_eff], val float32 [rows*t_eff])."""
    _require_cuda(key, torch.int32, "key")
    _require_cuda(val, torch.int32, "val")
    _require_cuda(perm, torch.int32, "perm")
    ncand = int(key.numel())
    if val.numel() != 2 * ncand:
        raise ValueError("val must hold two int32 words per candidate key")
    if perm.numel() != int(n) or not (0 <= int(row_begin) <= int(row_end) <= int(n)):
        raise ValueError("perm length != n or row range outside [0, n]")
    dev = perm.device
    te = min(int(t), int(n) - 1)
    rows = int(row_end) - int(row_begin)
    nb = C.c_size_t(0)
    _check(lib().ggm_sym_merge_workspace(ncand, C.byref(nb)))
    ws = torch.empty(max(nb.value, 256), dtype=torch.uint8, device=dev)
    row_id = torch.empty(max(rows, 1), dtype=torch.int64, device=dev)
    col = torch.empty(max(rows * te, 1), dtype=torch.int32, device=dev)
    out = torch.empty(max(rows * te, 1), dtype=torch.float32, device=dev)
    kp = _ptr(key) if ncand else C.c_void_p(0)
    vp_ = _ptr(val) if ncand else C.c_void_p(0)
    _check(lib().ggm_sym_merge(int(n), int(t), kp, vp_, ncand, _ptr(perm), int(row_begin),
                               int(row_end), _ptr(row_id), _ptr(col), _ptr(out), _ptr(ws),
                               ws.numel(), _stream(stream)))
    return row_id[:rows], col[:rows * te], out[:rows * te]


def set_timing(enabled: bool):
    lib().ggm_set_timing(1 if enabled else 0)


def last_stats() -> dict:
    arr = (C.c_double * 6)()
    lib().ggm_last_stats(arr)
    return {"scheme": "symmetric" if arr[0] == 2 else "plain", "entries_main": arr[1],
            "candidates": int(arr[2]), "recomputed": int(arr[3]),
            "mma_k_per_entry": int(arr[4]), "cta_pair": bool(arr[5])}


def last_launches() -> int:
    return int(lib().ggm_last_launches())


def last_timing():
    arr = (C.c_float * 3)()
    lib().ggm_last_timing(arr)
    return list(arr)
