// gram_eig.cu — per-axis Gram spectrum (Algorithm 1 lines 1-4; Theorem 1,
// P:308-331): top-k eigenpairs of S_l = mat_l(X) mat_l(X)^T — equivalently the
// top-k left singular vectors of D_l = mat_l(X) with E = sigma^2.
//
// fp64 throughout (C2's top-50 spectrum has relative eigengaps ~3e-4, so an fp32
// Gram would rotate the subspace):
//   unfold_f64  : mat_l(X) in fp64, column-major d_l x d_\l (one coalesced permute pass)
//   cuBLAS DSYRK: S = M M^T  (or, for a matrix whose axis is the longer side, the Gram of the
//                 OTHER axis, so both axes of a matrix share one bitwise-identical spectrum,
//                 reading T; V is mapped back as V = M^T W diag(1/sigma))
//   cuSOLVER DSYEVD: all eigenpairs of the small Gram (a library eigensolver, like a sort)
//   select_topk : descending top-k, deterministic sign (largest-|.| entry positive), fp32
//                 row-major V (k contiguous)
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cusparse.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "ggm_internal.h"

namespace ggm {
namespace ge {

struct Handles {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  ~Handles() {
    if (blas) cublasDestroy(blas);
    if (solver) cusolverDnDestroy(solver);
  }
};
static thread_local Handles g_handles;

static ggm_status get_handles(cudaStream_t s, cublasHandle_t* b, cusolverDnHandle_t* so) {
  if (!g_handles.blas && cublasCreate(&g_handles.blas) != CUBLAS_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cublasCreate failed");
  if (!g_handles.solver && cusolverDnCreate(&g_handles.solver) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnCreate failed");
  if (cublasSetStream(g_handles.blas, s) != CUBLAS_STATUS_SUCCESS ||
      cusolverDnSetStream(g_handles.solver, s) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "set stream failed");
  *b = g_handles.blas;
  *so = g_handles.solver;
  return GGM_OK;
}

// M (column-major, rows = d_axis, cols = d_\axis) from row-major X viewed as
// [pre, d_axis, post]: M[i + c*d] = X[pre, i, post], c = pre*post_n + post.
__global__ void unfold_f64(const float* __restrict__ X, int64_t pre_n, int64_t d, int64_t post_n,
                           double* __restrict__ M, double* __restrict__ fro) {
  const int64_t total = pre_n * d * post_n;
  double acc = 0.0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    // idx enumerates the OUTPUT (i fastest) for coalesced writes
    const int64_t i = idx % d;
    const int64_t c = idx / d;
    const int64_t pre = c / post_n, post = c % post_n;
    const double x = (double)X[(pre * d + i) * post_n + post];
    M[idx] = x;
    acc += x * x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(fro, acc);
}

// Eigenvalues w (ascending, length dim) and eigenvectors Z (column-major dim x dim) ->
// top-k descending E and column-major V64 (rows x k) from Z (primal: rows = dim).
__global__ void take_topk(const double* __restrict__ w, const double* __restrict__ Z, int dim,
                          int k, double* __restrict__ E, double* __restrict__ Vk) {
  const int r = blockIdx.x;  // output column
  if (r >= k) return;
  const int src = dim - 1 - r;
  if (threadIdx.x == 0) E[r] = w[src];
  for (int i = threadIdx.x; i < dim; i += blockDim.x) Vk[(size_t)r * dim + i] = Z[(size_t)src * dim + i];
}

// Sign fix (largest-|.| entry positive; first index on ties) and fp32 row-major output.
__global__ void sign_and_store(const double* __restrict__ V64, int64_t rows, int k,
                               float* __restrict__ V) {
  const int r = blockIdx.x;
  __shared__ double sv[32];
  __shared__ long long si[32];
  double best = -1.0;
  long long bi = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double a = fabs(V64[(size_t)r * rows + i]);
    if (a > best) {
      best = a;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > sv[0] || (sv[w] == sv[0] && si[w] < si[0])) {
        sv[0] = sv[w];
        si[0] = si[w];
      }
  }
  __syncthreads();
  const double sgn = V64[(size_t)r * rows + si[0]] < 0 ? -1.0 : 1.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x)
    V[i * k + r] = (float)(sgn * V64[(size_t)r * rows + i]);
}

// mode 1/2: Vasc (d x k, ascending eigen order) -> V64 column r = Vasc column (k-1-r) /
// sigma_r, E[r] = w[dim-1-r].
__global__ void reverse_scale(const double* __restrict__ w, int dim, const double* __restrict__ Vasc,
                              int64_t d, int k, double* __restrict__ E, double* __restrict__ V64) {
  const int r = blockIdx.y;
  const double e = w[dim - 1 - r];
  if (blockIdx.x == 0 && threadIdx.x == 0) E[r] = e;
  const double inv = e > 0.0 ? 1.0 / sqrt(e) : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x)
    V64[(size_t)r * d + i] = Vasc[(size_t)(k - 1 - r) * d + i] * inv;
}

struct GPlan {
  int64_t d, m;        // axis length, product of the others
  int64_t pre_n, post_n;
  int mode;            // 0 primal (S = M M^T), 1 dual via the other axis of a matrix,
                       // 2 dual via M^T M (tensor with d > m)
  int64_t dim;         // Gram dimension
  int64_t Md_rows, Md_cols;  // the unfolding actually materialised (column-major)
  int k;
  int lwork;
};

static ggm_status make_gplan(int ndim, const int64_t* shape, int axis, int k, GPlan* g) {
  if (ndim < 1 || !shape) return fail(GGM_ERR_INVALID_ARGUMENT, "ndim/shape invalid");
  if (axis < 0 || axis >= ndim) return fail(GGM_ERR_INVALID_ARGUMENT, "axis %d out of range", axis);
  int64_t pre = 1, post = 1;
  for (int a = 0; a < ndim; ++a) {
    if (shape[a] < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "shape[%d] < 1", a);
    if (a < axis) pre *= shape[a];
    if (a > axis) post *= shape[a];
  }
  g->d = shape[axis];
  g->m = pre * post;
  g->pre_n = pre;
  g->post_n = post;
  g->k = k;
  if (k < 1 || k > std::min(g->d, g->m))
    return fail(GGM_ERR_RANK, "k=%d not in [1, min(d_l=%lld, d_\\l=%lld)] (S:116)", k,
                (long long)g->d, (long long)g->m);
  if (g->d <= g->m) {
    g->mode = 0;
    g->dim = g->d;
    g->Md_rows = g->d;
    g->Md_cols = g->m;
  } else if (ndim == 2) {
    g->mode = 1;  // Gram of the other axis: M_o = mat_other (m x d), S_o = M_o M_o^T (m x m)
    g->dim = g->m;
    g->Md_rows = g->m;
    g->Md_cols = g->d;
  } else {
    g->mode = 2;
    g->dim = g->m;
    g->Md_rows = g->d;
    g->Md_cols = g->m;
  }
  return GGM_OK;
}
// Gram dimensions above this use randomized subspace iteration (ggm_gram_eig_rsi): a dense
// fp64 eigensolve of a 32768^2 Gram (8.6 GB) is already minutes of DSYEVD.
constexpr int64_t kMaxDenseGram = 32768;
constexpr int kRsiMaxIter = 200;       // ggm_gram_eig's automatic at-scale path
constexpr double kRsiTol = 1e-13;      // max relative change of the top-k Ritz values
constexpr uint64_t kRsiSeed = 0x2407198920240728ull;

static size_t gcarve(const GPlan& g, int lwork, void* ws, double** Md, double** S, double** w,
                     double** work, int** info, double** V64, double** fro, double** Ek,
                     double** Vasc) {
  Carve c(ws);
  *Md = c.take<double>((size_t)g.Md_rows * g.Md_cols);
  *S = c.take<double>((size_t)g.dim * g.dim);
  *w = c.take<double>((size_t)g.dim);
  *work = c.take<double>((size_t)std::max(lwork, 1));
  *info = c.take<int>(4);
  *V64 = c.take<double>((size_t)g.d * g.k);
  *fro = c.take<double>(4);
  *Ek = c.take<double>((size_t)g.k);
  *Vasc = c.take<double>(g.mode == 0 ? 0 : (size_t)g.d * g.k);
  return c.used();
}

static ggm_status query_lwork(const GPlan& g, int* lwork) {
  cusolverDnHandle_t h = g_handles.solver;
  if (!h && cusolverDnCreate(&g_handles.solver) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnCreate failed");
  h = g_handles.solver;
  int lw = 0;
  if (cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)g.dim,
                                  nullptr, (int)g.dim, nullptr, &lw) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
  *lwork = lw;
  return GGM_OK;
}


// ------------------------------------------------------------------ randomized subspace iteration
// Seeded standard normals (counter-based splitmix64 + Box-Muller): Omega[idx], idx < count.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void fill_normal(double* __restrict__ out, int64_t count, uint64_t seed) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < count;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = splitmix64(seed ^ (2 * (uint64_t)idx));
    const uint64_t b = splitmix64(seed ^ (2 * (uint64_t)idx + 1));
    const double u1 = ((double)(a >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = ((double)(b >> 11)) * (1.0 / 9007199254740992.0);
    out[idx] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  }
}

struct RPlan {
  int64_t d, m, pre_n, post_n;
  int k, r;  // wanted pairs, subspace width (k + oversampling)
  int lw_syevd, lw_geqrf, lw_orgqr;
};

static ggm_status make_rplan(int ndim, const int64_t* shape, int axis, int k, int oversample,
                             RPlan* rp) {
  GPlan g;
  ggm_status st = make_gplan(ndim, shape, axis, k, &g);
  if (st != GGM_OK) return st;
  rp->d = g.d;
  rp->m = g.m;
  rp->pre_n = g.pre_n;
  rp->post_n = g.post_n;
  rp->k = k;
  const int64_t mn = std::min(g.d, g.m);
  const int64_t p = oversample > 0 ? oversample : std::max<int64_t>(16, k);
  rp->r = (int)std::min<int64_t>(mn, k + p);
  cusolverDnHandle_t h = g_handles.solver;
  if (!h && cusolverDnCreate(&g_handles.solver) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnCreate failed");
  h = g_handles.solver;
  if (cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, rp->r,
                                  nullptr, rp->r, nullptr, &rp->lw_syevd) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDgeqrf_bufferSize(h, (int)rp->d, rp->r, nullptr, (int)rp->d, &rp->lw_geqrf) !=
          CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDorgqr_bufferSize(h, (int)rp->d, rp->r, rp->r, nullptr, (int)rp->d, nullptr,
                                  &rp->lw_orgqr) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cuSOLVER buffer size query failed");
  if (rp->d > INT32_MAX || rp->m > INT32_MAX)
    return fail(GGM_ERR_UNSUPPORTED, "axis extents above 2^31 are not supported");
  return GGM_OK;
}

struct RWork {
  double *M, *Om, *Y, *T, *w, *work, *tau, *V64, *fro, *Ek, *Wk;
  int* info;
};
static size_t rcarve(const RPlan& rp, void* ws, RWork* w, bool dense_M = true) {
  Carve c(ws);
  w->M = c.take<double>(dense_M ? (size_t)rp.d * rp.m : 0);
  w->Om = c.take<double>((size_t)rp.m * rp.r);  // Omega, then Z = M^T Q
  w->Y = c.take<double>((size_t)rp.d * rp.r);   // Y = M Z, then Q
  w->T = c.take<double>((size_t)rp.r * rp.r);
  w->w = c.take<double>((size_t)rp.r);
  w->work = c.take<double>((size_t)std::max({rp.lw_syevd, rp.lw_geqrf, rp.lw_orgqr, 1}));
  w->tau = c.take<double>((size_t)rp.r);
  w->V64 = c.take<double>((size_t)rp.d * rp.k);
  w->fro = c.take<double>(4);
  w->Ek = c.take<double>((size_t)rp.k);
  w->Wk = c.take<double>((size_t)rp.r * rp.k);
  w->info = c.take<int>(4);
  return c.used();
}

// top-k of T's eigen-decomposition (ascending w, vectors in T): Ek descending, Wk (r x k)
__global__ void take_topk_small(const double* __restrict__ w, const double* __restrict__ T, int r,
                                int k, double* __restrict__ Ek, double* __restrict__ Wk) {
  const int c = blockIdx.x;
  if (c >= k) return;
  const int src = r - 1 - c;
  if (threadIdx.x == 0) Ek[c] = w[src];
  for (int i = threadIdx.x; i < r; i += blockDim.x) Wk[(size_t)c * r + i] = T[(size_t)src * r + i];
}

}  // namespace ge
}  // namespace ggm

using namespace ggm;
using namespace ggm::ge;

static ggm_status rsi_core(const RPlan& rp, const RWork& w, int max_iter, double tol,
                           uint64_t seed, float* V, double* E, double* trace_S, int* iters_out,
                           double* change_out, cublasHandle_t hb, cusolverDnHandle_t hs,
                           cudaStream_t s);

extern "C" ggm_status ggm_gram_eig_rsi_workspace(int ndim, const int64_t* shape, int axis, int k,
                                                 int oversample, size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  RPlan rp;
  ggm_status st = make_rplan(ndim, shape, axis, k, oversample, &rp);
  if (st != GGM_OK) return st;
  RWork w;
  *bytes = rcarve(rp, nullptr, &w);
  return GGM_OK;
}

extern "C" ggm_status ggm_gram_eig_rsi(const float* X, int ndim, const int64_t* shape, int axis,
                                       int k, int oversample, int max_iter, double tol,
                                       uint64_t seed, float* V, double* E, double* trace_S,
                                       int* iters_out, double* change_out, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  if (!X || !V || !E || !workspace) return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  if (max_iter < 1 || !(tol >= 0.0)) return fail(GGM_ERR_INVALID_ARGUMENT, "max_iter/tol invalid");
  RPlan rp;
  ggm_status st = make_rplan(ndim, shape, axis, k, oversample, &rp);
  if (st != GGM_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  RWork w;
  const size_t need = rcarve(rp, workspace, &w);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  const int sms = num_sms();
  GGM_CUDA_TRY(cudaMemsetAsync(w.fro, 0, sizeof(double), s));
  {
    const int64_t total = rp.pre_n * rp.d * rp.post_n;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, sms * 16));
    unfold_f64<<<grid, 256, 0, s>>>(X, rp.pre_n, rp.d, rp.post_n, w.M, w.fro);  // M: d x m
    GGM_CUDA_TRY(cudaGetLastError());
  }
  return rsi_core(rp, w, max_iter, tol, seed, V, E, trace_S, iters_out, change_out, hb, hs, s);
}

template <class FA, class FAt>
static ggm_status rsi_generic(const RPlan& rp, const RWork& w, FA applyA, FAt applyAt,
                              int max_iter, double tol, uint64_t seed, float* V, double* E,
                              double* trace_S, int* iters_out, double* change_out,
                              cublasHandle_t hb, cusolverDnHandle_t hs, cudaStream_t s);

// Randomized subspace iteration on the unfolding already in w.M (d x m column-major) and its
// squared Frobenius norm in w.fro.
static ggm_status rsi_core(const RPlan& rp, const RWork& w, int max_iter, double tol,
                           uint64_t seed, float* V, double* E, double* trace_S, int* iters_out,
                           double* change_out, cublasHandle_t hb, cusolverDnHandle_t hs,
                           cudaStream_t s) {
  const int d = (int)rp.d, m = (int)rp.m, r = rp.r;
  const double one = 1.0, zero = 0.0;
  auto applyA = [&](const double* in, double* out) -> bool {  // out (d x r) = M in (m x r)
    return cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, d, r, m, &one, w.M, d, in, m, &zero, out,
                       d) == CUBLAS_STATUS_SUCCESS;
  };
  auto applyAt = [&](const double* in, double* out) -> bool {  // out (m x r) = M^T in (d x r)
    return cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, m, r, d, &one, w.M, d, in, d, &zero, out,
                       m) == CUBLAS_STATUS_SUCCESS;
  };
  return rsi_generic(rp, w, applyA, applyAt, max_iter, tol, seed, V, E, trace_S, iters_out,
                     change_out, hb, hs, s);
}

// Randomized subspace iteration for an implicit operator A (d x m): applyA(in, out) computes
// out = A in (in m x r, out d x r), applyAt(in, out) out = A^T in; all column-major fp64.
// ||A||_F^2 is expected in w.fro.  Range finder Y = A Ω, then per iteration Rayleigh-Ritz
// (Z = A^T Q, T = Z^T Z = Q^T A A^T Q, DSYEVD) and a power step Q = orth(A Z).
template <class FA, class FAt>
static ggm_status rsi_generic(const RPlan& rp, const RWork& w, FA applyA, FAt applyAt,
                              int max_iter, double tol, uint64_t seed, float* V, double* E,
                              double* trace_S, int* iters_out, double* change_out,
                              cublasHandle_t hb, cusolverDnHandle_t hs, cudaStream_t s) {
  const int sms = num_sms();
  const int d = (int)rp.d, m = (int)rp.m, r = rp.r, kk = rp.k;
  ggm_status st = GGM_OK;
  fill_normal<<<(int)std::min<int64_t>(((int64_t)m * r + 255) / 256, sms * 8), 256, 0, s>>>(
      w.Om, (int64_t)m * r, seed);
  GGM_CUDA_TRY(cudaGetLastError());
  const double one = 1.0, zero = 0.0;
  auto orth = [&](double* A) -> ggm_status {  // A (d x r) := Q of its Householder QR
    if (cusolverDnDgeqrf(hs, d, r, A, d, w.tau, w.work, rp.lw_geqrf, w.info) != CUSOLVER_STATUS_SUCCESS ||
        cusolverDnDorgqr(hs, d, r, r, A, d, w.tau, w.work, rp.lw_orgqr, w.info) != CUSOLVER_STATUS_SUCCESS)
      return fail(GGM_ERR_CUDA, "cuSOLVER QR failed");
    return GGM_OK;
  };
  // range finder: Y = A Omega, Q = orth(Y)
  if (!applyA(w.Om, w.Y)) return fail(GGM_ERR_CUDA, "operator product A Omega failed");
  st = orth(w.Y);
  if (st != GGM_OK) return st;
  std::vector<double> prev(kk, 0.0), cur(kk);
  int it = 0;
  double change = INFINITY;
  for (it = 1; it <= max_iter; ++it) {
    // Rayleigh-Ritz on span(Q): Z = A^T Q (m x r), T = Z^T Z = Q^T S Q (r x r)
    if (!applyAt(w.Y, w.Om) ||
        cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, r, m, &one, w.Om, m, &zero, w.T, r) !=
            CUBLAS_STATUS_SUCCESS)
      return fail(GGM_ERR_CUDA, "Rayleigh-Ritz products failed");
    if (cusolverDnDsyevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, r, w.T, r, w.w,
                         w.work, rp.lw_syevd, w.info) != CUSOLVER_STATUS_SUCCESS)
      return fail(GGM_ERR_CUDA, "cusolverDnDsyevd failed");
    take_topk_small<<<kk, 128, 0, s>>>(w.w, w.T, r, kk, w.Ek, w.Wk);
    GGM_CUDA_TRY(cudaMemcpyAsync(cur.data(), w.Ek, sizeof(double) * kk, cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    change = 0.0;
    for (int c = 0; c < kk; ++c)
      change = std::max(change, std::fabs(cur[c] - prev[c]) / std::max(std::fabs(cur[0]), 1e-300));
    prev = cur;
    if (change <= tol || r >= std::min(d, m) || it == max_iter) break;
    // power step: Y = A Z = S Q, Q = orth(Y)
    if (!applyA(w.Om, w.Y)) return fail(GGM_ERR_CUDA, "operator product A Z failed");
    st = orth(w.Y);
    if (st != GGM_OK) return st;
  }
  // Ritz vectors V = Q W_k (d x k)
  if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, d, kk, r, &one, w.Y, d, w.Wk, r, &zero, w.V64, d) !=
      CUBLAS_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cublasDgemm failed");
  sign_and_store<<<kk, 256, 0, s>>>(w.V64, rp.d, kk, V);
  GGM_CUDA_TRY(cudaGetLastError());
  GGM_CUDA_TRY(cudaMemcpyAsync(E, w.Ek, sizeof(double) * kk, cudaMemcpyDeviceToDevice, s));
  double hfro = 0.0;
  GGM_CUDA_TRY(cudaMemcpyAsync(&hfro, w.fro, sizeof(double), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (trace_S) *trace_S = hfro;
  if (iters_out) *iters_out = it > max_iter ? max_iter : it;
  if (change_out) *change_out = change;
  if (!(cur[0] > 0.0) || !std::isfinite(cur[0]) || !(cur[kk - 1] > 1e-12 * cur[0]))
    return fail(GGM_ERR_RANK, "E_k=%.3e <= 1e-12 E_1=%.3e: k exceeds the rank (S:140)",
                cur[kk - 1], cur[0]);
  return GGM_OK;
}

namespace ggm {
namespace ge {
}  // namespace ge
}  // namespace ggm


static ggm_status dense_core(const GPlan& g, int lwork, double* Md, double* S, double* w,
                             double* work, int* dinfo, double* V64, double* fro, double* Ek,
                             double* Vasc, float* V, double* E, double* trace_S,
                             cublasHandle_t hb, cusolverDnHandle_t hs, cudaStream_t s);
static ggm_status enqueue_unfold(const GPlan& g, const float* X, const int64_t* shape, int axis,
                                 double* Md, double* fro, cudaStream_t s);

extern "C" ggm_status ggm_gram_eig_workspace(int ndim, const int64_t* shape, int axis, int k,
                                             size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  GPlan g;
  ggm_status st = make_gplan(ndim, shape, axis, k, &g);
  if (st != GGM_OK) return st;
  if (g.dim > kMaxDenseGram)  // at-scale path (randomized subspace iteration)
    return ggm_gram_eig_rsi_workspace(ndim, shape, axis, k, 0, bytes);
  int lwork = 0;
  st = query_lwork(g, &lwork);
  if (st != GGM_OK) return st;
  double *a, *b, *c, *d, *f, *h, *e, *v;
  int* i;
  *bytes = gcarve(g, lwork, nullptr, &a, &b, &c, &d, &i, &f, &h, &e, &v);
  return GGM_OK;
}

extern "C" ggm_status ggm_gram_eig(const float* X, int ndim, const int64_t* shape, int axis, int k,
                                   float* V, double* E, double* trace_S, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (!X || !V || !E || !workspace) return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  GPlan g;
  ggm_status st = make_gplan(ndim, shape, axis, k, &g);
  if (st != GGM_OK) return st;
  if (g.dim > kMaxDenseGram)  // at-scale path: both sides of the unfolding exceed 32768
    return ggm_gram_eig_rsi(X, ndim, shape, axis, k, 0, kRsiMaxIter, kRsiTol, kRsiSeed, V, E,
                            trace_S, nullptr, nullptr, workspace, workspace_bytes, stream);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  int lwork = 0;
  st = query_lwork(g, &lwork);
  if (st != GGM_OK) return st;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  double *Md, *S, *w, *work, *V64, *fro, *Ek, *Vasc;
  int* dinfo;
  const size_t need =
      gcarve(g, lwork, workspace, &Md, &S, &w, &work, &dinfo, &V64, &fro, &Ek, &Vasc);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);

  st = enqueue_unfold(g, X, shape, axis, Md, fro, s);
  if (st != GGM_OK) return st;
  return dense_core(g, lwork, Md, S, w, work, dinfo, V64, fro, Ek, Vasc, V, E, trace_S, hb, hs, s);
}

// fro = 0, then the unfolding GPlan g asks for (matrix other side: the transposed view).
static ggm_status enqueue_unfold(const GPlan& g, const float* X, const int64_t* shape, int axis,
                                 double* Md, double* fro, cudaStream_t s) {
  GGM_CUDA_TRY(cudaMemsetAsync(fro, 0, sizeof(double), s));
  const int sms = num_sms();
  {
    // which unfolding to materialise
    int64_t pre_n = g.pre_n, d = g.d, post_n = g.post_n;
    if (g.mode == 1) {  // matrix, other axis: X is [d0, d1]; other = 1 - axis
      if (axis == 0) {   // other axis 1: [pre=d0, d=d1, post=1]
        pre_n = shape[0];
        d = shape[1];
        post_n = 1;
      } else {           // other axis 0: [pre=1, d=d0, post=d1]
        pre_n = 1;
        d = shape[0];
        post_n = shape[1];
      }
    }
    const int64_t total = pre_n * d * post_n;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, sms * 16));
    unfold_f64<<<grid, 256, 0, s>>>(X, pre_n, d, post_n, Md, fro);
    GGM_CUDA_TRY(cudaGetLastError());
  }
  return GGM_OK;
}

// Lower triangle of the fp64 Gram S = M M^T (trans = N, M dim x inner, leading dim ld) or
// S = M^T M (trans = T, M inner x dim).  A long inner dimension leaves DSYRK's dim^2/2 output
// tiles too few for the SMs (C3: 78 tiles of 32 x 32 over K = 60,000); the full DGEMM, whose
// heuristics split K, is faster there despite computing both triangles.
static cublasStatus_t gram_lower(cublasHandle_t hb, cublasOperation_t trans, int dim,
                                 int64_t inner, const double* M, int ld, double* S) {
  const double one = 1.0, zero = 0.0;
  static const bool syrk_only = std::getenv("GGM_GRAM_SYRK") != nullptr;  // A/B hook
  if (!syrk_only && inner >= 32 * (int64_t)dim)
    return trans == CUBLAS_OP_N
               ? cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, dim, dim, (int)inner, &one, M, ld, M,
                             ld, &zero, S, dim)
               : cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, dim, dim, (int)inner, &one, M, ld, M,
                             ld, &zero, S, dim);
  return cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, trans, dim, (int)inner, &one, M, ld, &zero, S,
                     dim);
}

// Gram + eigensolve + top-k mapping on the unfolding already in Md (GPlan g decides the side);
// device work only (dense_check reads the status back).
static ggm_status dense_enqueue(const GPlan& g, int lwork, double* Md, double* S, double* w,
                                double* work, int* dinfo, double* V64, double* Ek, double* Vasc,
                                float* V, double* E, cublasHandle_t hb, cusolverDnHandle_t hs,
                                cudaStream_t s) {
  const double one = 1.0, zero = 0.0;
  cublasStatus_t bs;
  if (g.mode == 2)  // S = M^T M  (m x m), M is d x m column-major
    bs = gram_lower(hb, CUBLAS_OP_T, (int)g.dim, g.Md_rows, Md, (int)g.Md_rows, S);
  else              // S = M M^T  (Md_rows x Md_rows)
    bs = gram_lower(hb, CUBLAS_OP_N, (int)g.dim, g.Md_cols, Md, (int)g.Md_rows, S);
  if (bs != CUBLAS_STATUS_SUCCESS) return fail(GGM_ERR_CUDA, "Gram product failed (%d)", (int)bs);
  cusolverStatus_t ss = cusolverDnDsyevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                         (int)g.dim, S, (int)g.dim, w, work, lwork, dinfo);
  if (ss != CUSOLVER_STATUS_SUCCESS) return fail(GGM_ERR_CUDA, "cusolverDnDsyevd failed (%d)", (int)ss);
  // top-k eigenpairs of the Gram that was formed (syevd: ascending eigenvalues, Z in S)
  if (g.mode == 0) {
    take_topk<<<g.k, 256, 0, s>>>(w, S, (int)g.dim, g.k, Ek, V64);
    GGM_CUDA_TRY(cudaGetLastError());
  } else {
    // V = A W_k diag(1/sigma), A = mat_axis (d x m): mode 1 A = Md^T, mode 2 A = Md.
    const double* Zk = S + (size_t)(g.dim - g.k) * g.dim;  // ascending block of the top k
    if (g.mode == 1)
      bs = cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, (int)g.d, g.k, (int)g.dim, &one, Md,
                       (int)g.Md_rows, Zk, (int)g.dim, &zero, Vasc, (int)g.d);
    else
      bs = cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)g.d, g.k, (int)g.dim, &one, Md,
                       (int)g.Md_rows, Zk, (int)g.dim, &zero, Vasc, (int)g.d);
    if (bs != CUBLAS_STATUS_SUCCESS) return fail(GGM_ERR_CUDA, "cublasDgemm failed (%d)", (int)bs);
    reverse_scale<<<dim3(std::max<int64_t>(1, std::min<int64_t>((g.d + 255) / 256, 64)), g.k), 256, 0, s>>>(
        w, (int)g.dim, Vasc, g.d, g.k, Ek, V64);
    GGM_CUDA_TRY(cudaGetLastError());
  }
  sign_and_store<<<g.k, 256, 0, s>>>(V64, g.d, g.k, V);
  GGM_CUDA_TRY(cudaGetLastError());
  GGM_CUDA_TRY(cudaMemcpyAsync(E, Ek, sizeof(double) * g.k, cudaMemcpyDeviceToDevice, s));
  return GGM_OK;
}

// Synchronises s; solver status, trace, rank check.
static ggm_status dense_check(const GPlan& g, const int* dinfo, const double* fro, const double* Ek,
                              double* trace_S, cudaStream_t s) {
  std::vector<double> hE(g.k);
  int hinfo = 0;
  double hfro = 0.0;
  GGM_CUDA_TRY(cudaMemcpyAsync(hE.data(), Ek, sizeof(double) * g.k, cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(&hfro, fro, sizeof(double), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hinfo != 0) return fail(GGM_ERR_CUDA, "cusolverDnDsyevd info=%d", hinfo);
  if (trace_S) *trace_S = hfro;
  if (!(hE[0] > 0.0) || !std::isfinite(hE[0]) || !(hE[g.k - 1] > 1e-12 * hE[0]))
    return fail(GGM_ERR_RANK, "E_k=%.3e <= 1e-12 E_1=%.3e: k exceeds the rank (S:140)",
                hE[g.k - 1], hE[0]);
  return GGM_OK;
}

static ggm_status dense_core(const GPlan& g, int lwork, double* Md, double* S, double* w,
                             double* work, int* dinfo, double* V64, double* fro, double* Ek,
                             double* Vasc, float* V, double* E, double* trace_S,
                             cublasHandle_t hb, cusolverDnHandle_t hs, cudaStream_t s) {
  ggm_status st = dense_enqueue(g, lwork, Md, S, w, work, dinfo, V64, Ek, Vasc, V, E, hb, hs, s);
  if (st != GGM_OK) return st;
  return dense_check(g, dinfo, fro, Ek, trace_S, s);
}

// ------------------------------------------------------------------ multi-modal spectrum
// Alg. 1 line 2: D_l = [mat_l(D^γ1) ... mat_l(D^γΓ)] over the modalities that
// contain axis l; V, E = top-k left singular vectors / squared singular values of D_l, i.e.
// the eigenpairs of S_l = Σ_γ mat_l(D^γ) mat_l(D^γ)^T.  Each modality is unfolded into its
// own column block of one fp64 d x Σm matrix; the dense (primal or dual Gram) or at-scale
// (randomized subspace iteration) path then runs on the concatenation.
namespace {
struct MultiShape {
  int64_t d, m_tot;
  std::vector<int64_t> pre, post, coloff;
  std::vector<int> used;  // modalities that contain the axis
};
ggm_status multi_shape(int M, const int* ndim, const int64_t* shapes, const int* axis_pos,
                       MultiShape* ms) {
  if (M < 1 || !ndim || !shapes || !axis_pos)
    return fail(GGM_ERR_INVALID_ARGUMENT, "M < 1 or null descriptor");
  ms->d = -1;
  ms->m_tot = 0;
  const int64_t* sh = shapes;
  for (int g = 0; g < M; ++g) {
    if (ndim[g] < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "ndim[%d] < 1", g);
    const int ax = axis_pos[g];
    if (ax >= ndim[g]) return fail(GGM_ERR_INVALID_ARGUMENT, "axis_pos[%d] out of range", g);
    if (ax >= 0) {
      int64_t pre = 1, post = 1;
      for (int a = 0; a < ndim[g]; ++a) {
        if (sh[a] < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "shape < 1");
        if (a < ax) pre *= sh[a];
        if (a > ax) post *= sh[a];
      }
      if (ms->d >= 0 && sh[ax] != ms->d)
        return fail(GGM_ERR_INVALID_ARGUMENT, "shared axis length differs between modalities");
      ms->d = sh[ax];
      ms->pre.push_back(pre);
      ms->post.push_back(post);
      ms->coloff.push_back(ms->m_tot);
      ms->used.push_back(g);
      ms->m_tot += pre * post;
    }
    sh += ndim[g];
  }
  if (ms->used.empty()) return fail(GGM_ERR_INVALID_ARGUMENT, "the axis occurs in no modality");
  return GGM_OK;
}
}  // namespace

extern "C" ggm_status ggm_gram_eig_multi_workspace(int M, const int* ndim, const int64_t* shapes,
                                                   const int* axis_pos, int k, size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  MultiShape ms;
  ggm_status st = multi_shape(M, ndim, shapes, axis_pos, &ms);
  if (st != GGM_OK) return st;
  const int64_t shape2[2] = {ms.d, ms.m_tot};
  GPlan g;
  st = make_gplan(2, shape2, 0, k, &g);
  if (st != GGM_OK) return st;
  if (g.dim > kMaxDenseGram) return ggm_gram_eig_rsi_workspace(2, shape2, 0, k, 0, bytes);
  if (g.mode == 1) {  // the concatenation is a plain d x m matrix: use the M^T M form
    g.mode = 2;
    g.Md_rows = g.d;
    g.Md_cols = g.m;
  }
  int lwork = 0;
  st = query_lwork(g, &lwork);
  if (st != GGM_OK) return st;
  double *a, *b, *c, *d, *f, *h, *e, *v;
  int* i;
  *bytes = gcarve(g, lwork, nullptr, &a, &b, &c, &d, &i, &f, &h, &e, &v);
  return GGM_OK;
}

extern "C" ggm_status ggm_gram_eig_multi(int M, const float* const* X, const int* ndim,
                                         const int64_t* shapes, const int* axis_pos, int k,
                                         float* V, double* E, double* trace_S, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (!X || !V || !E || !workspace) return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  MultiShape ms;
  ggm_status st = multi_shape(M, ndim, shapes, axis_pos, &ms);
  if (st != GGM_OK) return st;
  for (int g = 0; g < M; ++g)
    if (axis_pos[g] >= 0 && !X[g]) return fail(GGM_ERR_INVALID_ARGUMENT, "X[%d] is NULL", g);
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  const int64_t shape2[2] = {ms.d, ms.m_tot};
  const int sms = num_sms();
  auto unfold_all = [&](double* Mbase, double* fro) -> ggm_status {
    GGM_CUDA_TRY(cudaMemsetAsync(fro, 0, sizeof(double), s));
    for (size_t u = 0; u < ms.used.size(); ++u) {
      const int64_t total = ms.pre[u] * ms.d * ms.post[u];
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, sms * 16));
      unfold_f64<<<grid, 256, 0, s>>>(X[ms.used[u]], ms.pre[u], ms.d, ms.post[u],
                                      Mbase + (size_t)ms.coloff[u] * ms.d, fro);
      GGM_CUDA_TRY(cudaGetLastError());
    }
    return GGM_OK;
  };
  GPlan g;
  st = make_gplan(2, shape2, 0, k, &g);
  if (st != GGM_OK) return st;
  if (g.dim > kMaxDenseGram) {
    RPlan rp;
    st = make_rplan(2, shape2, 0, k, 0, &rp);
    if (st != GGM_OK) return st;
    RWork w;
    const size_t need = rcarve(rp, workspace, &w);
    if (workspace_bytes < need)
      return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
    st = unfold_all(w.M, w.fro);
    if (st != GGM_OK) return st;
    return rsi_core(rp, w, kRsiMaxIter, kRsiTol, kRsiSeed, V, E, trace_S, nullptr, nullptr, hb,
                    hs, s);
  }
  if (g.mode == 1) {
    g.mode = 2;
    g.Md_rows = g.d;
    g.Md_cols = g.m;
  }
  int lwork = 0;
  st = query_lwork(g, &lwork);
  if (st != GGM_OK) return st;
  double *Md, *S, *w, *work, *V64, *fro, *Ek, *Vasc;
  int* dinfo;
  const size_t need = gcarve(g, lwork, workspace, &Md, &S, &w, &work, &dinfo, &V64, &fro, &Ek, &Vasc);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  st = unfold_all(Md, fro);
  if (st != GGM_OK) return st;
  return dense_core(g, lwork, Md, S, w, work, dinfo, V64, fro, Ek, Vasc, V, E, trace_S, hb, hs, s);
}

// ------------------------------------------------------------------ sparse unfoldings (CSR)
// §8(f) row 1 (sparse inputs) and row 4 (nonparanormal skeptic, sparse rank-one trick,
// P:965-1016).  The unfolding D_l is given as CSR (d rows = the axis, m columns).  With the
// COCA transform the data become S + z 1^T (S with D's sparsity pattern, z_i the value the
// zeros of row i map to); instead of a rank-one SVD update the randomized
// subspace iteration applies the operator implicitly: A X = S X + z (1^T X),
// A^T Y = S^T Y + 1 (z^T Y) — the matrix is never densified.
namespace {

struct SparseHandle {
  cusparseHandle_t h = nullptr;
  ~SparseHandle() {
    if (h) cusparseDestroy(h);
  }
};
thread_local SparseHandle g_sparse;

__device__ __forceinline__ float canon_zero(float x) { return x == 0.f ? 0.f : x; }

__global__ void copy_canon(const float* __restrict__ v, int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = canon_zero(v[i]);
}

// first position in sorted[lo, hi) with sorted[p] >= x
__device__ __forceinline__ int64_t lower_bound_f(const float* sorted, int64_t lo, int64_t hi,
                                                 float x) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// One warp per row: COCA values of the stored entries (rank = 1 + #entries < x, the row's
// implicit zeros counted when x > 0; Φ^-1(r/(m+1))), z_i for the zeros, S = value - z_i,
// and ||S + z 1^T||_F^2.  np = 0: S = val, z = 0.
__global__ void csr_values(const int64_t* __restrict__ rp, const float* __restrict__ val,
                           const float* __restrict__ sorted, int64_t d, int64_t m, int np,
                           double* __restrict__ sval, double* __restrict__ z,
                           double* __restrict__ fro) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < d;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = rp[i], e = rp[i + 1];
    const int64_t implicit0 = m - (e - b);
    double zi = 0.0;
    if (np) {
      const int64_t neg = lower_bound_f(sorted, b, e, 0.f) - b;  // stored entries < 0
      const bool has_zero = implicit0 > 0 || (neg < e - b && sorted[b + neg] == 0.f);
      zi = has_zero ? normcdfinv((double)(neg + 1) / (double)(m + 1)) : 0.0;
    }
    for (int64_t q = b + lane; q < e; q += 32) {
      const float x = canon_zero(val[q]);
      double v;
      if (np) {
        const int64_t less = lower_bound_f(sorted, b, e, x) - b + (x > 0.f ? implicit0 : 0);
        v = normcdfinv((double)(less + 1) / (double)(m + 1)) - zi;
        if (x == 0.f) v = 0.0;  // explicit zeros keep the pattern
      } else {
        v = (double)x;
      }
      sval[q] = v;
      acc += (v + zi) * (v + zi);
    }
    if (lane == 0) {
      z[i] = zi;
      acc += (double)implicit0 * zi * zi;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) atomicAdd(fro, acc);
}

__global__ void fill_f64(double* p, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void rp_to_i32(const int64_t* rp, int64_t n, int32_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)rp[i];
}
__global__ void col_to_i64(const int32_t* c, int64_t n, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = c[i];
}

struct CsrWork {
  double *sval, *z, *ones, *cs, *zq;
  float *canon, *sorted;
  int32_t* rp32;
  int64_t* col64;
  void* cub;
  size_t cub_bytes;
};
size_t csr_carve(int64_t d, int64_t m, int64_t nnz, int r, bool idx32, size_t cub_bytes,
                 void* ws, CsrWork* w) {
  Carve c(ws);
  w->sval = c.take<double>(nnz);
  w->z = c.take<double>(d);
  w->ones = c.take<double>(m);
  w->cs = c.take<double>(r);
  w->zq = c.take<double>(r);
  w->canon = c.take<float>(nnz);
  w->sorted = c.take<float>(nnz);
  w->rp32 = c.take<int32_t>(idx32 ? d + 1 : 0);
  w->col64 = c.take<int64_t>(idx32 ? 0 : nnz);
  w->cub = c.take<char>(cub_bytes);
  w->cub_bytes = cub_bytes;
  return c.used();
}
size_t csr_sort_bytes(int64_t d, int64_t nnz) {
  size_t b = 0;
  cub::DeviceSegmentedSort::SortKeys(nullptr, b, (const float*)nullptr, (float*)nullptr, nnz,
                                     d, (const int64_t*)nullptr, (const int64_t*)nullptr);
  return b;
}

ggm_status csr_plan(int64_t d, int64_t m, int64_t nnz, int k, int oversample, RPlan* rp) {
  if (d < 1 || m < 1 || nnz < 0) return fail(GGM_ERR_INVALID_ARGUMENT, "d, m >= 1, nnz >= 0");
  const int64_t shape2[2] = {d, m};
  return make_rplan(2, shape2, 0, k, oversample, rp);
}

// ---- exact path when the shorter side fits a dense Gram (min(d, m) <= kMaxDenseGram):
// the Gram of the shorter side accumulated over bounded dense chunks of A = S + z 1^T
// (fp64 DSYRK), dense eigensolve, and (long rows side) V = A W diag(1/σ) chunk by chunk.
// Memory stays O(chunk + dim^2): the matrix is never densified as a whole.
constexpr int64_t kChunkElems = int64_t(1) << 27;  // 1 GiB of fp64 per dense chunk

// rows [r0, r1) of A, dense column-major (r1 - r0) x m
__global__ void csr_rows_dense(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                               const double* __restrict__ sval, const double* __restrict__ z,
                               int64_t r0, int64_t r1, int64_t m, double* __restrict__ out) {
  const int64_t ld = r1 - r0;
  const int lane = threadIdx.x & 31;
  for (int64_t i = r0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < r1;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double zi = z[i];
    for (int64_t c = lane; c < m; c += 32) out[(i - r0) + c * ld] = zi;
    __syncwarp();
    for (int64_t q = rp[i] + lane; q < rp[i + 1]; q += 32) out[(i - r0) + (int64_t)col[q] * ld] = sval[q] + zi;
  }
}
// columns [c0, c1) of A, dense column-major d x (c1 - c0) (columns ascending within rows)
__global__ void csr_cols_dense(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                               const double* __restrict__ sval, const double* __restrict__ z,
                               int64_t d, int64_t c0, int64_t c1, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < d;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double zi = z[i];
    for (int64_t c = c0 + lane; c < c1; c += 32) out[i + (c - c0) * d] = zi;
    __syncwarp();
    int64_t lo = rp[i], hi = rp[i + 1];
    {  // first stored entry with col >= c0
      int64_t a = lo, b = hi;
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (col[mid] < c0) a = mid + 1; else b = mid;
      }
      lo = a;
    }
    for (int64_t q = lo + lane; q < hi; q += 32) {
      const int64_t c = col[q];
      if (c >= c1) break;
      out[i + (c - c0) * d] = sval[q] + zi;
    }
  }
}

// Z (m x k column-major, leading dimension ld) -> row-major m x k
__global__ void transpose_cm(const double* __restrict__ Z, int64_t ld, int64_t m, int k,
                             double* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * k;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t / k;
    const int j = (int)(t - g * k);
    out[t] = Z[g + (int64_t)j * ld];
  }
}
// column sums of Z (m x k column-major): one warp per column
__global__ void colsum_cm(const double* __restrict__ Z, int64_t ld, int64_t m, int k,
                          double* __restrict__ out) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= k) return;
  double acc = 0.0;
  for (int64_t g = threadIdx.x & 31; g < m; g += 32) acc += Z[g + (int64_t)j * ld];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) out[j] = acc;
}
// V[i, :] = Σ_q sval[q] W[col[q], :] (+ z_i colsum) for every CSR row i; V column-major d x k,
// W row-major m x k.  One warp per row, lanes over the k columns.
__global__ void csr_project_rows(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const double* __restrict__ sval, const double* __restrict__ z,
                                 int64_t d, int k, const double* __restrict__ W,
                                 const double* __restrict__ colsum, double* __restrict__ V) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < d;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = rp[i], e = rp[i + 1];
    for (int j0 = 0; j0 < k; j0 += 32) {
      const int j = j0 + lane;
      double acc = 0.0;
      if (j < k)
        for (int64_t q = b; q < e; ++q) acc += sval[q] * W[(int64_t)col[q] * k + j];
      if (j < k) V[i + (int64_t)j * d] = colsum ? acc + z[i] * colsum[j] : acc;
    }
  }
}

struct CsrDense {
  int64_t dim, chunk;
  bool rows_side;  // Gram = A^T A (m x m) accumulated over row chunks (m <= d)
  int lwork;
  bool tc;         // chunk Grams on the tensor cores (gram_tc.cu) instead of fp64 DSYRK
};
// Tensor-core chunk Grams (fp32-accurate 3 x fp16 products, fp64 across 4,096-sample slices)
// for large Grams: d·m·min(d, m) >= 1e11 flops (PBMC scale: 6e12); below that the fp64
// DSYRK costs milliseconds.  GGM_GRAM_TC=1 / 0 forces the choice (tests).
static bool use_gram_tc(int64_t d, int64_t m) {
  if (const char* e = getenv("GGM_GRAM_TC")) return e[0] == '1';
  return (double)d * (double)m * (double)std::min(d, m) >= 1e11;
}
ggm_status csr_dense_plan(int64_t d, int64_t m, int k, CsrDense* cd) {
  cd->rows_side = m <= d;
  cd->dim = cd->rows_side ? m : d;
  cd->chunk = std::max<int64_t>(1, kChunkElems / (cd->rows_side ? m : d));
  cd->tc = use_gram_tc(d, m);
  cusolverDnHandle_t h = g_handles.solver;
  if (!h && cusolverDnCreate(&g_handles.solver) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnCreate failed");
  if (cusolverDnDsyevd_bufferSize(g_handles.solver, CUSOLVER_EIG_MODE_VECTOR,
                                  CUBLAS_FILL_MODE_LOWER, (int)cd->dim, nullptr, (int)cd->dim,
                                  nullptr, &cd->lwork) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
  if (k < 1 || k > std::min(d, m)) return fail(GGM_ERR_RANK, "k=%d not in [1, min(d, m)]", k);
  return GGM_OK;
}
struct CsrDenseWork {
  double *G, *w, *work, *chunk, *V64, *Vasc, *Ek, *fro;
  int* info;
  void* tcws;  // gram_tc operand (cd.tc)
};
size_t csr_dense_carve(int64_t d, int64_t m, int k, const CsrDense& cd, void* ws, CsrDenseWork* w) {
  Carve c(ws);
  w->G = c.take<double>((size_t)cd.dim * cd.dim);
  w->w = c.take<double>(cd.dim);
  w->work = c.take<double>(std::max(cd.lwork, 1));
  w->chunk = c.take<double>((size_t)cd.chunk * (cd.rows_side ? m : d));
  w->V64 = c.take<double>((size_t)d * k);
  w->Vasc = c.take<double>(cd.rows_side ? (size_t)d * k : 0);
  w->Ek = c.take<double>(k);
  w->fro = c.take<double>(4);
  w->info = c.take<int>(4);
  w->tcws = c.take<uint8_t>(cd.tc ? gram_tc_workspace(cd.chunk, cd.dim) : 0);
  return c.used();
}

bool csr_dense_path(int64_t d, int64_t m) {
  return std::min(d, m) <= kMaxDenseGram && !getenv("GGM_CSR_RSI");
}

}  // namespace

static ggm_status csr_gram_dense(int64_t d, int64_t m, int64_t nnz, const int64_t* row_ptr,
                                 const int32_t* col, const float* val, int k, int nonparanormal,
                                 float* V, double* E, double* trace_S, int* iters_out,
                                 double* change_out, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  CsrDense cd;
  ggm_status st = csr_dense_plan(d, m, k, &cd);
  if (st != GGM_OK) return st;
  CsrDenseWork dw;
  const size_t b0 = csr_dense_carve(d, m, k, cd, workspace, &dw);
  CsrWork cw;
  const size_t need = b0 + csr_carve(d, m, nnz, 1, true, csr_sort_bytes(d, nnz),
                                     static_cast<char*>(workspace) + b0, &cw);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  const int sms = num_sms();
  auto grid_of = [&](int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, sms * 8));
  };
  GGM_CUDA_TRY(cudaMemsetAsync(dw.fro, 0, sizeof(double), s));
  if (nnz > 0) {
    copy_canon<<<grid_of(nnz), 256, 0, s>>>(val, nnz, cw.canon);
    if (nonparanormal) {
      size_t tb = cw.cub_bytes;
      GGM_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(cw.cub, tb, cw.canon, cw.sorted, nnz, d,
                                                      row_ptr, row_ptr + 1, s));
    }
  }
  csr_values<<<grid_of(32 * d), 256, 0, s>>>(row_ptr, cw.canon, cw.sorted, d, m,
                                              nonparanormal ? 1 : 0, cw.sval, cw.z, dw.fro);
  GGM_CUDA_TRY(cudaGetLastError());
  const double one = 1.0, zero = 0.0;
  const int dim = (int)cd.dim;
  // Gram of the shorter side over dense chunks
  const int64_t total = cd.rows_side ? d : m;
  // stage times when ggm_set_timing(1): Gram (incl. the operand scatter), eigensolve,
  // projection + store (ggm_last_timing slots 0, 1, 2)
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
  const bool timed = timing_enabled();
  if (timed)
    for (auto& e : tev) cudaEventCreate(&e);
  if (timed) cudaEventRecord(tev[0], s);
  if (cd.tc) {
    GGM_CUDA_TRY(cudaMemsetAsync(dw.G, 0, sizeof(double) * (size_t)dim * dim, s));
    st = gram_tc_csr_scale(row_ptr, cw.sval, d, dw.tcws, s);
    if (st != GGM_OK) return st;
  }
  for (int64_t c0 = 0; c0 < total; c0 += cd.chunk) {
    const int64_t c1 = std::min(total, c0 + cd.chunk);
    const double beta = c0 == 0 ? 0.0 : 1.0;
    cublasStatus_t bs = CUBLAS_STATUS_SUCCESS;
    if (cd.tc) {  // operand straight from the CSR (no dense chunk), tensor-core Gram
      st = gram_tc_accumulate_csr(row_ptr, col, cw.sval, d, cd.rows_side, c0, c1, dim, dw.G,
                                  dw.tcws, s);
      if (st != GGM_OK) return st;
    } else if (cd.rows_side) {  // chunk: (c1-c0) x m column-major; G += chunk^T chunk
      csr_rows_dense<<<grid_of(32 * (c1 - c0)), 256, 0, s>>>(row_ptr, col, cw.sval, cw.z, c0, c1, m, dw.chunk);
      {
        bs = cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, dim, (int)(c1 - c0), &one,
                         dw.chunk, (int)(c1 - c0), &beta, dw.G, dim);
      }
    } else {             // chunk: d x (c1-c0) column-major; G += chunk chunk^T
      csr_cols_dense<<<grid_of(32 * d), 256, 0, s>>>(row_ptr, col, cw.sval, cw.z, d, c0, c1, dw.chunk);
      {
        bs = cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, dim, (int)(c1 - c0), &one,
                         dw.chunk, (int)d, &beta, dw.G, dim);
      }
    }
    GGM_CUDA_TRY(cudaGetLastError());
    if (bs != CUBLAS_STATUS_SUCCESS) return fail(GGM_ERR_CUDA, "cublasDsyrk failed (%d)", (int)bs);
  }
  if (cd.tc) {  // the exact rank-one terms of S + z 1^T (fp64; z = 0 for raw data)
    st = gram_tc_csr_rank1(row_ptr, col, cw.sval, cw.z, d, cd.rows_side, dim, m, dw.G, dw.work, s);
    if (st != GGM_OK) return st;
  }
  if (timed) cudaEventRecord(tev[1], s);
  if (cusolverDnDsyevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, dim, dw.G, dim, dw.w,
                       dw.work, cd.lwork, dw.info) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnDsyevd failed");
  if (timed) cudaEventRecord(tev[2], s);
  if (!cd.rows_side) {
    take_topk<<<k, 256, 0, s>>>(dw.w, dw.G, dim, k, dw.Ek, dw.V64);
  } else {
    // V = A W_k diag(1/σ): rows chunk by chunk into Vasc (d x k, ascending order), then
    // reverse + scale
    const double* Zk = dw.G + (size_t)(dim - k) * dim;
    if (k <= 1024) {
      // in the sparse rank-one form: A Z = S Z + z (1ᵀ Z), one warp per row over its stored
      // entries (Z transposed to row-major first; fp64; no dense chunks)
      transpose_cm<<<grid_of((int64_t)m * k), 256, 0, s>>>(Zk, dim, m, k, dw.work);
      if (nonparanormal) colsum_cm<<<(k + 7) / 8, 256, 0, s>>>(Zk, dim, m, k, dw.work + (size_t)m * k);
      csr_project_rows<<<grid_of(32 * d), 256, 0, s>>>(row_ptr, col, cw.sval, cw.z, d, k, dw.work,
                                                       nonparanormal ? dw.work + (size_t)m * k : nullptr,
                                                       dw.Vasc);
      GGM_CUDA_TRY(cudaGetLastError());
    } else {
      for (int64_t r0 = 0; r0 < d; r0 += cd.chunk) {
        const int64_t r1 = std::min(d, r0 + cd.chunk);
        csr_rows_dense<<<grid_of(32 * (r1 - r0)), 256, 0, s>>>(row_ptr, col, cw.sval, cw.z, r0, r1, m, dw.chunk);
        if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)(r1 - r0), k, dim, &one, dw.chunk,
                        (int)(r1 - r0), Zk, dim, &zero, dw.Vasc + r0, (int)d) != CUBLAS_STATUS_SUCCESS)
          return fail(GGM_ERR_CUDA, "cublasDgemm failed");
      }
    }
    reverse_scale<<<dim3(std::max<int64_t>(1, std::min<int64_t>((d + 255) / 256, 64)), k), 256, 0, s>>>(
        dw.w, dim, dw.Vasc, d, k, dw.Ek, dw.V64);
  }
  GGM_CUDA_TRY(cudaGetLastError());
  sign_and_store<<<k, 256, 0, s>>>(dw.V64, d, k, V);
  GGM_CUDA_TRY(cudaGetLastError());
  if (timed) {
    cudaEventRecord(tev[3], s);
    cudaEventSynchronize(tev[3]);
    for (int q = 0; q < 3; ++q) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[q], tev[q + 1]);
      record_timing(q, ms);
    }
    for (auto& e : tev) cudaEventDestroy(e);
  }
  GGM_CUDA_TRY(cudaMemcpyAsync(E, dw.Ek, sizeof(double) * k, cudaMemcpyDeviceToDevice, s));
  std::vector<double> hE(k);
  int hinfo = 0;
  double hfro = 0.0;
  GGM_CUDA_TRY(cudaMemcpyAsync(hE.data(), dw.Ek, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(&hinfo, dw.info, sizeof(int), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(&hfro, dw.fro, sizeof(double), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hinfo != 0) return fail(GGM_ERR_CUDA, "cusolverDnDsyevd info=%d", hinfo);
  if (trace_S) *trace_S = hfro;
  if (iters_out) *iters_out = 0;
  if (change_out) *change_out = 0.0;
  if (!(hE[0] > 0.0) || !std::isfinite(hE[0]) || !(hE[k - 1] > 1e-12 * hE[0]))
    return fail(GGM_ERR_RANK, "E_k=%.3e <= 1e-12 E_1=%.3e: k exceeds the rank (S:140)",
                hE[k - 1], hE[0]);
  return GGM_OK;
}

extern "C" ggm_status ggm_gram_eig_csr_workspace(int64_t d, int64_t m, int64_t nnz, int k,
                                                 int oversample, size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  if (d >= 1 && m >= 1 && csr_dense_path(d, m)) {
    CsrDense cd;
    ggm_status st = csr_dense_plan(d, m, k, &cd);
    if (st != GGM_OK) return st;
    CsrDenseWork dw;
    CsrWork cw;
    *bytes = csr_dense_carve(d, m, k, cd, nullptr, &dw) +
             csr_carve(d, m, nnz, 1, true, csr_sort_bytes(d, nnz), nullptr, &cw);
    return GGM_OK;
  }
  RPlan rp;
  ggm_status st = csr_plan(d, m, nnz, k, oversample, &rp);
  if (st != GGM_OK) return st;
  RWork w;
  size_t b = rcarve(rp, nullptr, &w, false);
  b = (b + 255) / 256 * 256;
  const bool idx32 = nnz < INT32_MAX && d < INT32_MAX;
  CsrWork cw;
  *bytes = b + csr_carve(d, m, nnz, rp.r, idx32, csr_sort_bytes(d, nnz), nullptr, &cw);
  return GGM_OK;
}

extern "C" ggm_status ggm_gram_eig_csr(int64_t d, int64_t m, int64_t nnz, const int64_t* row_ptr,
                                       const int32_t* col, const float* val, int k,
                                       int nonparanormal, int oversample, int max_iter,
                                       double tol, uint64_t seed, float* V, double* E,
                                       double* trace_S, int* iters_out, double* change_out,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!row_ptr || (nnz > 0 && (!col || !val)) || !V || !E || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  if (max_iter < 1 || !(tol >= 0.0)) return fail(GGM_ERR_INVALID_ARGUMENT, "max_iter/tol invalid");
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  if (d >= 1 && m >= 1 && csr_dense_path(d, m))
    return csr_gram_dense(d, m, nnz, row_ptr, col, val, k, nonparanormal, V, E, trace_S,
                          iters_out, change_out, workspace, workspace_bytes, stream);
  RPlan rp;
  ggm_status st = csr_plan(d, m, nnz, k, oversample, &rp);
  if (st != GGM_OK) return st;
  RWork w;
  size_t b0 = rcarve(rp, workspace, &w, false);
  b0 = (b0 + 255) / 256 * 256;
  const bool idx32 = nnz < INT32_MAX && d < INT32_MAX;
  CsrWork cw;
  const size_t need = b0 + csr_carve(d, m, nnz, rp.r, idx32, csr_sort_bytes(d, nnz),
                                     static_cast<char*>(workspace) + b0, &cw);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  if (!g_sparse.h && cusparseCreate(&g_sparse.h) != CUSPARSE_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusparseCreate failed");
  cusparseSetStream(g_sparse.h, s);
  const int sms = num_sms();
  auto grid_of = [&](int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, sms * 8));
  };
  // (1) values of S (COCA-transformed or raw), z, ||A||_F^2
  GGM_CUDA_TRY(cudaMemsetAsync(w.fro, 0, sizeof(double), s));
  if (nnz > 0) {
    copy_canon<<<grid_of(nnz), 256, 0, s>>>(val, nnz, cw.canon);
    if (nonparanormal) {
      size_t tb = cw.cub_bytes;
      GGM_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(cw.cub, tb, cw.canon, cw.sorted, nnz, d,
                                                      row_ptr, row_ptr + 1, s));
    }
  }
  csr_values<<<grid_of(32 * d), 256, 0, s>>>(row_ptr, cw.canon, cw.sorted, d, m,
                                              nonparanormal ? 1 : 0, cw.sval, cw.z, w.fro);
  fill_f64<<<grid_of(m), 256, 0, s>>>(cw.ones, m, 1.0);
  GGM_CUDA_TRY(cudaGetLastError());
  // (2) cuSPARSE descriptors
  const void* rpp = row_ptr;
  const void* colp = col;
  if (idx32) {
    rp_to_i32<<<grid_of(d + 1), 256, 0, s>>>(row_ptr, d + 1, cw.rp32);
    rpp = cw.rp32;
  } else {
    col_to_i64<<<grid_of(nnz), 256, 0, s>>>(col, nnz, cw.col64);
    colp = cw.col64;
  }
  GGM_CUDA_TRY(cudaGetLastError());
  const cusparseIndexType_t it = idx32 ? CUSPARSE_INDEX_32I : CUSPARSE_INDEX_64I;
  cusparseSpMatDescr_t A = nullptr;
  if (cusparseCreateCsr(&A, d, m, nnz, const_cast<void*>(rpp), const_cast<void*>(colp), cw.sval,
                        it, it, CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F) != CUSPARSE_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusparseCreateCsr failed");
  const int r = rp.r;
  cusparseDnMatDescr_t Xm = nullptr, Yd = nullptr;
  cusparseCreateDnMat(&Xm, m, r, m, w.Om, CUDA_R_64F, CUSPARSE_ORDER_COL);  // m x r operand
  cusparseCreateDnMat(&Yd, d, r, d, w.Y, CUDA_R_64F, CUSPARSE_ORDER_COL);   // d x r
  const double one = 1.0, zero = 0.0;
  size_t bN = 0, bT = 0;
  cusparseSpMM_bufferSize(g_sparse.h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                          CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, Xm, &zero, Yd, CUDA_R_64F,
                          CUSPARSE_SPMM_ALG_DEFAULT, &bN);
  cusparseSpMM_bufferSize(g_sparse.h, CUSPARSE_OPERATION_TRANSPOSE,
                          CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, Yd, &zero, Xm, CUDA_R_64F,
                          CUSPARSE_SPMM_ALG_DEFAULT, &bT);
  void* spbuf = nullptr;
  GGM_CUDA_TRY(cudaMallocAsync(&spbuf, std::max<size_t>(std::max(bN, bT), 256), s));
  auto cleanup = [&]() {
    cusparseDestroySpMat(A);
    cusparseDestroyDnMat(Xm);
    cusparseDestroyDnMat(Yd);
    cudaFreeAsync(spbuf, s);
  };
  // operator products: the RSI buffers are fixed (Om: m x r, Y: d x r), so the descriptors
  // are bound to them; applyA reads Om and writes Y, applyAt reads Y and writes Om
  auto applyA = [&](const double* in, double* out) -> bool {  // Y = S Om + z (1^T Om)
    if (in != w.Om || out != w.Y) return false;
    if (cusparseSpMM(g_sparse.h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                     CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, Xm, &zero, Yd, CUDA_R_64F,
                     CUSPARSE_SPMM_ALG_DEFAULT, spbuf) != CUSPARSE_STATUS_SUCCESS)
      return false;
    if (!nonparanormal) return true;
    return cublasDgemv(hb, CUBLAS_OP_T, (int)m, r, &one, w.Om, (int)m, cw.ones, 1, &zero, cw.cs,
                       1) == CUBLAS_STATUS_SUCCESS &&
           cublasDger(hb, (int)d, r, &one, cw.z, 1, cw.cs, 1, w.Y, (int)d) == CUBLAS_STATUS_SUCCESS;
  };
  auto applyAt = [&](const double* in, double* out) -> bool {  // Om = S^T Y + 1 (z^T Y)
    if (in != w.Y || out != w.Om) return false;
    if (cusparseSpMM(g_sparse.h, CUSPARSE_OPERATION_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE,
                     &one, A, Yd, &zero, Xm, CUDA_R_64F, CUSPARSE_SPMM_ALG_DEFAULT,
                     spbuf) != CUSPARSE_STATUS_SUCCESS)
      return false;
    if (!nonparanormal) return true;
    return cublasDgemv(hb, CUBLAS_OP_T, (int)d, r, &one, w.Y, (int)d, cw.z, 1, &zero, cw.zq,
                       1) == CUBLAS_STATUS_SUCCESS &&
           cublasDger(hb, (int)m, r, &one, cw.ones, 1, cw.zq, 1, w.Om, (int)m) ==
               CUBLAS_STATUS_SUCCESS;
  };
  st = rsi_generic(rp, w, applyA, applyAt, max_iter, tol, seed, V, E, trace_S, iters_out,
                   change_out, hb, hs, s);
  cleanup();
  return st;
}

// ------------------------------------------------------------------ dense COCA transform
// ggm_nonparanormal: every entry of the tensor is replaced by Φ^-1(r / (m + 1)), r = its
// rank (ties -> smallest rank, reading Q19) among the m = d_rest entries sharing its index
// on `axis` (the row of mat_axis); output in the input's own layout, so the
// transformed tensor feeds ggm_gram_eig for that axis unchanged.
namespace {
__global__ void unfold_rows_f32(const float* __restrict__ X, int64_t pre_n, int64_t d,
                                int64_t post_n, float* __restrict__ rows) {
  const int64_t total = pre_n * d * post_n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t post = idx % post_n, i = (idx / post_n) % d, pre = idx / (post_n * d);
    rows[i * (pre_n * post_n) + pre * post_n + post] = canon_zero(X[idx]);
  }
}
__global__ void row_offsets(int64_t d, int64_t m, int64_t* off) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= d;
       i += (int64_t)gridDim.x * blockDim.x)
    off[i] = i * m;
}
__global__ void coca_dense(const float* __restrict__ X, const float* __restrict__ sorted,
                           int64_t pre_n, int64_t d, int64_t post_n, float* __restrict__ out) {
  const int64_t total = pre_n * d * post_n, m = pre_n * post_n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = (idx / post_n) % d;
    const int64_t less = lower_bound_f(sorted, i * m, (i + 1) * m, canon_zero(X[idx])) - i * m;
    out[idx] = (float)normcdfinv((double)(less + 1) / (double)(m + 1));
  }
}
ggm_status np_shape(int ndim, const int64_t* shape, int axis, int64_t* pre, int64_t* d,
                    int64_t* post) {
  if (ndim < 1 || !shape || axis < 0 || axis >= ndim)
    return fail(GGM_ERR_INVALID_ARGUMENT, "ndim/shape/axis invalid");
  *pre = 1;
  *post = 1;
  for (int a = 0; a < ndim; ++a) {
    if (shape[a] < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "shape[%d] < 1", a);
    if (a < axis) *pre *= shape[a];
    if (a > axis) *post *= shape[a];
  }
  *d = shape[axis];
  return GGM_OK;
}
size_t np_carve(int64_t d, int64_t n, void* ws, float** rows, float** sorted, int64_t** off,
                void** cub, size_t* cub_bytes) {
  size_t b = 0;
  cub::DeviceSegmentedSort::SortKeys(nullptr, b, (const float*)nullptr, (float*)nullptr, n, d,
                                     (const int64_t*)nullptr, (const int64_t*)nullptr);
  Carve c(ws);
  *rows = c.take<float>(n);
  *sorted = c.take<float>(n);
  *off = c.take<int64_t>(d + 1);
  *cub = c.take<char>(b);
  *cub_bytes = b;
  return c.used();
}
}  // namespace

extern "C" ggm_status ggm_nonparanormal_workspace(int ndim, const int64_t* shape, int axis,
                                                  size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  int64_t pre, d, post;
  ggm_status st = np_shape(ndim, shape, axis, &pre, &d, &post);
  if (st != GGM_OK) return st;
  float *a, *b;
  int64_t* o;
  void* c;
  size_t cb;
  *bytes = np_carve(d, pre * d * post, nullptr, &a, &b, &o, &c, &cb);
  return GGM_OK;
}

extern "C" ggm_status ggm_nonparanormal(const float* X, int ndim, const int64_t* shape, int axis,
                                        float* out, void* workspace, size_t workspace_bytes,
                                        void* stream) {
  if (!X || !out || !workspace) return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  int64_t pre, d, post;
  ggm_status st = np_shape(ndim, shape, axis, &pre, &d, &post);
  if (st != GGM_OK) return st;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  const int64_t n = pre * d * post;
  float *rows, *sorted;
  int64_t* off;
  void* cub;
  size_t cb;
  const size_t need = np_carve(d, n, workspace, &rows, &sorted, &off, &cub, &cb);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 16));
  unfold_rows_f32<<<grid, 256, 0, s>>>(X, pre, d, post, rows);
  row_offsets<<<(int)std::min<int64_t>((d + 256) / 256, 1024), 256, 0, s>>>(d, pre * post, off);
  GGM_CUDA_TRY(cudaGetLastError());
  GGM_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(cub, cb, rows, sorted, n, d, off, off + 1, s));
  coca_dense<<<grid, 256, 0, s>>>(X, sorted, pre, d, post, out);
  GGM_CUDA_TRY(cudaGetLastError());
  return GGM_OK;
}

// ------------------------------------------------------------------ sharded spectrum pieces
// §8(f) row 1 "sharded Gram with one all-reduce": a matrix whose rows (the long axis, e.g.
// cells) are split over ranks.  Each rank accumulates G_r = A_r^T A_r (m x m, the short side)
// over its rows (ggm_gram_accumulate_csr), the caller all-reduces G (one NCCL all-reduce of
// m^2 doubles), every rank eigensolves it (ggm_eig_gram: short-axis V and E, plus W for the
// projection) and maps its own rows V_r = A_r W diag(E^-1/2) (ggm_project_csr).
namespace {
struct ShardWork {
  CsrWork cw;
  double *chunk, *fro;
};
size_t shard_carve(int64_t d, int64_t m, int64_t nnz, void* ws, ShardWork* w) {
  Carve c(ws);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(d, kChunkElems / m));
  w->chunk = c.take<double>((size_t)chunk * m);
  w->fro = c.take<double>(4);
  const size_t b0 = c.used();
  return b0 + csr_carve(d, m, nnz, 1, true, csr_sort_bytes(d, nnz),
                        ws ? static_cast<char*>(ws) + b0 : nullptr, &w->cw);
}
ggm_status shard_values(int64_t d, int64_t m, int64_t nnz, const int64_t* rp, const float* val,
                        int np, ShardWork& w, cudaStream_t s) {
  const int sms = num_sms();
  auto grid_of = [&](int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, sms * 8));
  };
  GGM_CUDA_TRY(cudaMemsetAsync(w.fro, 0, sizeof(double), s));
  if (nnz > 0) {
    copy_canon<<<grid_of(nnz), 256, 0, s>>>(val, nnz, w.cw.canon);
    if (np) {
      size_t tb = w.cw.cub_bytes;
      GGM_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(w.cw.cub, tb, w.cw.canon, w.cw.sorted, nnz,
                                                      d, rp, rp + 1, s));
    }
  }
  csr_values<<<grid_of(32 * d), 256, 0, s>>>(rp, w.cw.canon, w.cw.sorted, d, m, np ? 1 : 0,
                                              w.cw.sval, w.cw.z, w.fro);
  GGM_CUDA_TRY(cudaGetLastError());
  return GGM_OK;
}
}  // namespace

extern "C" ggm_status ggm_gram_accumulate_csr_workspace(int64_t d, int64_t m, int64_t nnz,
                                                        size_t* bytes) {
  if (!bytes || d < 1 || m < 1 || nnz < 0) return fail(GGM_ERR_INVALID_ARGUMENT, "bad sizes");
  ShardWork w;
  *bytes = shard_carve(d, m, nnz, nullptr, &w);
  return GGM_OK;
}

extern "C" ggm_status ggm_gram_accumulate_csr(int64_t d, int64_t m, int64_t nnz,
                                              const int64_t* row_ptr, const int32_t* col,
                                              const float* val, int nonparanormal, double* G,
                                              int accumulate, double* fro_out, void* workspace,
                                              size_t workspace_bytes, void* stream) {
  if (d < 1 || m < 1 || nnz < 0 || !row_ptr || (nnz > 0 && (!col || !val)) || !G || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "bad sizes / null pointer");
  if (m > kMaxDenseGram) return fail(GGM_ERR_UNSUPPORTED, "short side m=%lld > 32768", (long long)m);
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  ShardWork w;
  const size_t need = shard_carve(d, m, nnz, workspace, &w);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  ggm_status st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  st = shard_values(d, m, nnz, row_ptr, val, nonparanormal, w, s);
  if (st != GGM_OK) return st;
  const int sms = num_sms();
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(d, kChunkElems / m));
  const double one = 1.0;
  for (int64_t r0 = 0; r0 < d; r0 += chunk) {
    const int64_t r1 = std::min(d, r0 + chunk);
    const double beta = (r0 == 0 && !accumulate) ? 0.0 : 1.0;
    csr_rows_dense<<<(int)std::max<int64_t>(1, std::min<int64_t>((32 * (r1 - r0) + 255) / 256, sms * 8)),
                     256, 0, s>>>(row_ptr, col, w.cw.sval, w.cw.z, r0, r1, m, w.chunk);
    GGM_CUDA_TRY(cudaGetLastError());
    if (cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, (int)m, (int)(r1 - r0), &one, w.chunk,
                    (int)(r1 - r0), &beta, G, (int)m) != CUBLAS_STATUS_SUCCESS)
      return fail(GGM_ERR_CUDA, "cublasDsyrk failed");
  }
  if (fro_out) {
    GGM_CUDA_TRY(cudaMemcpyAsync(fro_out, w.fro, sizeof(double), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
  }
  return GGM_OK;
}

namespace {
__global__ void fix_sign_cols(double* W, int64_t rows, int k) {
  // largest-|.| entry of each column positive (first index on ties), in place
  const int r = blockIdx.x;
  __shared__ double sv[32];
  __shared__ long long si[32];
  double best = -1.0;
  long long bi = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double a = fabs(W[(size_t)r * rows + i]);
    if (a > best) { best = a; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (sv[q] > sv[0] || (sv[q] == sv[0] && si[q] < si[0])) { sv[0] = sv[q]; si[0] = si[q]; }
  __syncthreads();
  const double sgn = W[(size_t)r * rows + si[0]] < 0 ? -1.0 : 1.0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) W[(size_t)r * rows + i] *= sgn;
}
__global__ void scale_cols_store(const double* __restrict__ X, int64_t rows, int k,
                                 const double* __restrict__ E, float* __restrict__ V) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < rows * k;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / k;
    const int c = (int)(q % k);
    V[q] = (float)(X[(size_t)c * rows + i] / sqrt(E[c]));
  }
}
}  // namespace

extern "C" ggm_status ggm_eig_gram_workspace(int64_t dim, int k, size_t* bytes) {
  if (!bytes || dim < 1 || dim > kMaxDenseGram || k < 1 || k > dim)
    return fail(GGM_ERR_INVALID_ARGUMENT, "bad sizes");
  cusolverDnHandle_t h = g_handles.solver;
  if (!h && cusolverDnCreate(&g_handles.solver) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnCreate failed");
  int lw = 0;
  if (cusolverDnDsyevd_bufferSize(g_handles.solver, CUSOLVER_EIG_MODE_VECTOR,
                                  CUBLAS_FILL_MODE_LOWER, (int)dim, nullptr, (int)dim, nullptr,
                                  &lw) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
  Carve c(nullptr);
  c.take<double>((size_t)dim);
  c.take<double>((size_t)std::max(lw, 1));
  c.take<int>(4);
  *bytes = c.used();
  return GGM_OK;
}

extern "C" ggm_status ggm_eig_gram(int64_t dim, double* G, int k, float* V, double* E, double* W,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  if (!G || !V || !E || !W || !workspace) return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  size_t need = 0;
  ggm_status st = ggm_eig_gram_workspace(dim, k, &need);
  if (st != GGM_OK) return st;
  if (workspace_bytes < need) return fail(GGM_ERR_INVALID_ARGUMENT, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  int lw = 0;
  cusolverDnDsyevd_bufferSize(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)dim,
                              G, (int)dim, nullptr, &lw);
  Carve c(workspace);
  double* w = c.take<double>((size_t)dim);
  double* work = c.take<double>((size_t)std::max(lw, 1));
  int* info = c.take<int>(4);
  if (cusolverDnDsyevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)dim, G,
                       (int)dim, w, work, lw, info) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnDsyevd failed");
  take_topk<<<k, 256, 0, s>>>(w, G, (int)dim, k, E, W);  // W: dim x k, descending
  fix_sign_cols<<<k, 256, 0, s>>>(W, dim, k);
  sign_and_store<<<k, 256, 0, s>>>(W, dim, k, V);         // signs already fixed: plain store
  GGM_CUDA_TRY(cudaGetLastError());
  std::vector<double> hE(k);
  int hinfo = 0;
  GGM_CUDA_TRY(cudaMemcpyAsync(hE.data(), E, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hinfo != 0) return fail(GGM_ERR_CUDA, "cusolverDnDsyevd info=%d", hinfo);
  if (!(hE[0] > 0.0) || !std::isfinite(hE[0]) || !(hE[k - 1] > 1e-12 * hE[0]))
    return fail(GGM_ERR_RANK, "E_k=%.3e <= 1e-12 E_1=%.3e: k exceeds the rank (S:140)",
                hE[k - 1], hE[0]);
  return GGM_OK;
}

extern "C" ggm_status ggm_project_csr_workspace(int64_t d, int64_t m, int64_t nnz, int k,
                                                size_t* bytes) {
  ggm_status st = ggm_gram_accumulate_csr_workspace(d, m, nnz, bytes);
  if (st != GGM_OK) return st;
  if (k < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "k < 1");
  *bytes += (size_t)d * k * sizeof(double) + 256;
  return GGM_OK;
}

extern "C" ggm_status ggm_project_csr(int64_t d, int64_t m, int64_t nnz, const int64_t* row_ptr,
                                      const int32_t* col, const float* val, int nonparanormal,
                                      int k, const double* W, const double* E, float* V,
                                      void* workspace, size_t workspace_bytes, void* stream) {
  if (d < 1 || m < 1 || k < 1 || !row_ptr || !W || !E || !V || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "bad sizes / null pointer");
  size_t need = 0;
  ggm_status st = ggm_gram_accumulate_csr_workspace(d, m, nnz, &need);
  if (st != GGM_OK) return st;
  need += (size_t)d * k * sizeof(double) + 256;
  if (workspace_bytes < need) return fail(GGM_ERR_INVALID_ARGUMENT, "workspace too small");
  ShardWork w;
  const size_t b0 = shard_carve(d, m, nnz, workspace, &w);
  double* X = reinterpret_cast<double*>(static_cast<char*>(workspace) + b0);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  st = shard_values(d, m, nnz, row_ptr, val, nonparanormal, w, s);
  if (st != GGM_OK) return st;
  const int sms = num_sms();
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(d, kChunkElems / m));
  const double one = 1.0, zero = 0.0;
  for (int64_t r0 = 0; r0 < d; r0 += chunk) {
    const int64_t r1 = std::min(d, r0 + chunk);
    csr_rows_dense<<<(int)std::max<int64_t>(1, std::min<int64_t>((32 * (r1 - r0) + 255) / 256, sms * 8)),
                     256, 0, s>>>(row_ptr, col, w.cw.sval, w.cw.z, r0, r1, m, w.chunk);
    GGM_CUDA_TRY(cudaGetLastError());
    if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)(r1 - r0), k, (int)m, &one, w.chunk,
                    (int)(r1 - r0), W, (int)m, &zero, X + r0, (int)d) != CUBLAS_STATUS_SUCCESS)
      return fail(GGM_ERR_CUDA, "cublasDgemm failed");
  }
  scale_cols_store<<<(int)std::max<int64_t>(1, std::min<int64_t>((d * k + 255) / 256, sms * 8)), 256, 0, s>>>(
      X, d, k, E, V);
  GGM_CUDA_TRY(cudaGetLastError());
  return GGM_OK;
}

// ------------------------------------------------------------------ both axes of a matrix
// Thm 1 / P:125: for a matrix X (d0 x d1) the nonzero spectra of S_0 = X X^T and S_1 = X^T X
// coincide, and the top eigenvectors of the larger Gram are X^T W diag(1/σ) (or X W ...) of
// the smaller one's.  One Gram of the shorter side + one eigensolve give both axes' factors
// (the per-axis calls would form and solve the same Gram twice).
extern "C" ggm_status ggm_gram_eig_matrix_workspace(int64_t d0, int64_t d1, int k0, int k1,
                                                    size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  const int64_t dim = std::min(d0, d1), big = std::max(d0, d1);
  const int kmax = std::max(k0, k1);
  if (d0 < 1 || d1 < 1 || k0 < 1 || k1 < 1 || kmax > dim)
    return fail(GGM_ERR_RANK, "k0=%d, k1=%d not in [1, min(d0, d1)=%lld]", k0, k1, (long long)dim);
  if (dim > kMaxDenseGram) return fail(GGM_ERR_UNSUPPORTED, "both sides exceed 32768: use ggm_gram_eig (RSI)");
  cusolverDnHandle_t h = g_handles.solver;
  if (!h && cusolverDnCreate(&g_handles.solver) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnCreate failed");
  int lw = 0;
  if (cusolverDnDsyevd_bufferSize(g_handles.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                  (int)dim, nullptr, (int)dim, nullptr, &lw) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
  Carve c(nullptr);
  c.take<double>((size_t)d0 * d1);   // unfolding of the Gram side
  c.take<double>((size_t)dim * dim); // Gram / eigenvectors
  c.take<double>(dim);               // eigenvalues
  c.take<double>(std::max(lw, 1));
  c.take<int>(4);
  c.take<double>((size_t)big * kmax);  // V64 (either side)
  c.take<double>((size_t)big * kmax);  // Vasc
  c.take<double>(kmax);                // Ek
  c.take<double>(4);                   // fro
  *bytes = c.used();
  return GGM_OK;
}

extern "C" ggm_status ggm_gram_eig_matrix(const float* X, int64_t d0, int64_t d1, int k0, int k1,
                                          float* V0, double* E0, float* V1, double* E1,
                                          double* trace_S, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  if (!X || !V0 || !E0 || !V1 || !E1 || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  size_t need = 0;
  ggm_status st = ggm_gram_eig_matrix_workspace(d0, d1, k0, k1, &need);
  if (st != GGM_OK) return st;
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cublasHandle_t hb;
  cusolverDnHandle_t hs;
  st = get_handles(s, &hb, &hs);
  if (st != GGM_OK) return st;
  const bool g0 = d0 <= d1;  // the Gram is formed on axis 0 (else on axis 1)
  const int64_t dim = g0 ? d0 : d1, other = g0 ? d1 : d0;
  const int kmax = std::max(k0, k1);
  int lw = 0;
  cusolverDnDsyevd_bufferSize(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)dim,
                              nullptr, (int)dim, nullptr, &lw);
  Carve c(workspace);
  double* Md = c.take<double>((size_t)d0 * d1);
  double* S = c.take<double>((size_t)dim * dim);
  double* w = c.take<double>(dim);
  double* work = c.take<double>(std::max(lw, 1));
  int* dinfo = c.take<int>(4);
  double* V64 = c.take<double>((size_t)std::max(d0, d1) * kmax);
  double* Vasc = c.take<double>((size_t)std::max(d0, d1) * kmax);
  double* Ek = c.take<double>(kmax);
  double* fro = c.take<double>(4);
  const int sms = num_sms();
  GGM_CUDA_TRY(cudaMemsetAsync(fro, 0, sizeof(double), s));
  {
    // Md: dim x other, column-major (rows = the Gram side)
    const int64_t total = d0 * d1;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, sms * 16));
    if (g0)
      unfold_f64<<<grid, 256, 0, s>>>(X, 1, d0, d1, Md, fro);
    else
      unfold_f64<<<grid, 256, 0, s>>>(X, d0, d1, 1, Md, fro);
    GGM_CUDA_TRY(cudaGetLastError());
  }
  const double one = 1.0, zero = 0.0;
  if (gram_lower(hb, CUBLAS_OP_N, (int)dim, other, Md, (int)dim, S) != CUBLAS_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "Gram product failed");
  if (cusolverDnDsyevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)dim, S, (int)dim, w,
                       work, lw, dinfo) != CUSOLVER_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cusolverDnDsyevd failed");
  // the Gram side: its own eigenvectors
  const int kg = g0 ? k0 : k1;
  take_topk<<<kg, 256, 0, s>>>(w, S, (int)dim, kg, Ek, V64);
  sign_and_store<<<kg, 256, 0, s>>>(V64, dim, kg, g0 ? V0 : V1);
  GGM_CUDA_TRY(cudaMemcpyAsync(g0 ? E0 : E1, Ek, sizeof(double) * kg, cudaMemcpyDeviceToDevice, s));
  // the other side: Md^T W_k diag(1/σ)
  const int ko = g0 ? k1 : k0;
  const double* Zk = S + (size_t)(dim - ko) * dim;
  if (cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, (int)other, ko, (int)dim, &one, Md, (int)dim, Zk,
                  (int)dim, &zero, Vasc, (int)other) != CUBLAS_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cublasDgemm failed");
  reverse_scale<<<dim3(std::max<int64_t>(1, std::min<int64_t>((other + 255) / 256, 64)), ko), 256, 0, s>>>(
      w, (int)dim, Vasc, other, ko, Ek, V64);
  sign_and_store<<<ko, 256, 0, s>>>(V64, other, ko, g0 ? V1 : V0);
  GGM_CUDA_TRY(cudaMemcpyAsync(g0 ? E1 : E0, Ek, sizeof(double) * ko, cudaMemcpyDeviceToDevice, s));
  GGM_CUDA_TRY(cudaGetLastError());
  std::vector<double> hE(kmax);
  int hinfo = 0;
  double hfro = 0.0;
  GGM_CUDA_TRY(cudaMemcpyAsync(hE.data(), w + (dim - kmax), sizeof(double) * kmax, cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(&hfro, fro, sizeof(double), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hinfo != 0) return fail(GGM_ERR_CUDA, "cusolverDnDsyevd info=%d", hinfo);
  if (trace_S) *trace_S = hfro;
  // ascending: hE[0] is the kmax-th largest, hE[kmax-1] the largest
  if (!(hE[kmax - 1] > 0.0) || !std::isfinite(hE[kmax - 1]) || !(hE[0] > 1e-12 * hE[kmax - 1]))
    return fail(GGM_ERR_RANK, "E_k=%.3e <= 1e-12 E_1=%.3e: k exceeds the rank (S:140)", hE[0],
                hE[kmax - 1]);
  return GGM_OK;
}

// ------------------------------------------------------------------ every axis at once
// Alg. 1 lines 1-4 for all axes of one tensor.  The per-axis eigensolves (cuSOLVER's
// tridiagonal reduction of a few-hundred-square Gram is latency-bound: ~10 sequential
// kernels of a few CTAs) run concurrently on side streams forked from `stream`; every
// axis has its own workspace segment and handles, results are joined back onto `stream`.
namespace {
constexpr int kAxisStreams = 4;
struct AxisPool {
  cudaStream_t s[kAxisStreams] = {};
  cudaEvent_t ev[kAxisStreams + 1] = {};
  cublasHandle_t b[kAxisStreams] = {};
  cusolverDnHandle_t so[kAxisStreams] = {};
  bool ready = false;
  int device = -1;
  ~AxisPool() {
    for (int i = 0; i < kAxisStreams; ++i) {
      if (b[i]) cublasDestroy(b[i]);
      if (so[i]) cusolverDnDestroy(so[i]);
    }
    // streams and events are reclaimed with the context
  }
};
thread_local AxisPool g_axis_pool;

ggm_status axis_pool(AxisPool** out) {
  AxisPool& P = g_axis_pool;
  int dev = 0;
  GGM_CUDA_TRY(cudaGetDevice(&dev));
  if (P.ready && P.device != dev) {  // the thread moved to another device: new streams there
    for (int i = 0; i < kAxisStreams; ++i) {
      cublasDestroy(P.b[i]);
      cusolverDnDestroy(P.so[i]);
      P.b[i] = nullptr;
      P.so[i] = nullptr;
    }
    P.ready = false;
  }
  if (!P.ready) {
    P.device = dev;
    for (int i = 0; i < kAxisStreams; ++i) {
      GGM_CUDA_TRY(cudaStreamCreateWithFlags(&P.s[i], cudaStreamNonBlocking));
      if (cublasCreate(&P.b[i]) != CUBLAS_STATUS_SUCCESS ||
          cusolverDnCreate(&P.so[i]) != CUSOLVER_STATUS_SUCCESS ||
          cublasSetStream(P.b[i], P.s[i]) != CUBLAS_STATUS_SUCCESS ||
          cusolverDnSetStream(P.so[i], P.s[i]) != CUSOLVER_STATUS_SUCCESS)
        return fail(GGM_ERR_CUDA, "axis stream handles");
    }
    for (int i = 0; i <= kAxisStreams; ++i)
      GGM_CUDA_TRY(cudaEventCreateWithFlags(&P.ev[i], cudaEventDisableTiming));
    P.ready = true;
  }
  *out = &P;
  return GGM_OK;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }
}  // namespace

extern "C" ggm_status ggm_gram_eig_axes_workspace(int ndim, const int64_t* shape, const int* k,
                                                  size_t* bytes) {
  if (!bytes || !shape || !k) return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  size_t tot = 0;
  for (int a = 0; a < ndim; ++a) {
    size_t b = 0;
    ggm_status st = ggm_gram_eig_workspace(ndim, shape, a, k[a], &b);
    if (st != GGM_OK) return st;
    tot += align256(b);
  }
  *bytes = tot;
  return GGM_OK;
}

extern "C" ggm_status ggm_gram_eig_axes(const float* X, int ndim, const int64_t* shape,
                                        const int* k, float* const* V, double* const* E,
                                        double* trace_S, void* workspace, size_t workspace_bytes,
                                        void* stream) {
  if (!X || !shape || !k || !V || !E || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  size_t need = 0;
  ggm_status st = ggm_gram_eig_axes_workspace(ndim, shape, k, &need);
  if (st != GGM_OK) return st;
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  for (int a = 0; a < ndim; ++a)
    if (!V[a] || !E[a]) return fail(GGM_ERR_INVALID_ARGUMENT, "null V/E for axis %d", a);
  cudaStream_t s0 = static_cast<cudaStream_t>(stream);
  AxisPool* P = nullptr;
  st = axis_pool(&P);
  if (st != GGM_OK) return st;
  std::vector<GPlan> g(ndim);
  std::vector<int> lwork(ndim, 0);
  std::vector<size_t> off(ndim, 0);
  std::vector<char> dense(ndim, 0);
  size_t at = 0;
  for (int a = 0; a < ndim; ++a) {
    st = make_gplan(ndim, shape, a, k[a], &g[a]);
    if (st != GGM_OK) return st;
    size_t b = 0;
    ggm_gram_eig_workspace(ndim, shape, a, k[a], &b);
    off[a] = at;
    at += align256(b);
    dense[a] = g[a].dim <= kMaxDenseGram;
    if (dense[a]) {
      st = query_lwork(g[a], &lwork[a]);
      if (st != GGM_OK) return st;
    }
  }
  // fork: every side stream starts after the work already queued on `stream`
  GGM_CUDA_TRY(cudaEventRecord(P->ev[kAxisStreams], s0));
  const int nside = std::min(ndim, kAxisStreams);
  for (int i = 0; i < nside; ++i) GGM_CUDA_TRY(cudaStreamWaitEvent(P->s[i], P->ev[kAxisStreams], 0));
  struct Ptrs { double *Md, *S, *w, *work, *V64, *fro, *Ek, *Vasc; int* dinfo; };
  std::vector<Ptrs> pp(ndim);
  ggm_status first = GGM_OK;
  for (int a = 0; a < ndim && first == GGM_OK; ++a) {
    if (!dense[a]) continue;
    const int i = a % kAxisStreams;
    Ptrs& q = pp[a];
    gcarve(g[a], lwork[a], static_cast<char*>(workspace) + off[a], &q.Md, &q.S, &q.w, &q.work,
           &q.dinfo, &q.V64, &q.fro, &q.Ek, &q.Vasc);
    st = enqueue_unfold(g[a], X, shape, a, q.Md, q.fro, P->s[i]);
    if (st == GGM_OK)
      st = dense_enqueue(g[a], lwork[a], q.Md, q.S, q.w, q.work, q.dinfo, q.V64, q.Ek, q.Vasc,
                         V[a], E[a], P->b[i], P->so[i], P->s[i]);
    if (st != GGM_OK) first = st;
  }
  // status checks (each synchronises its own side stream while the others keep running)
  double tr = 0.0;
  for (int a = 0; a < ndim && first == GGM_OK; ++a) {
    if (!dense[a]) continue;
    st = dense_check(g[a], pp[a].dinfo, pp[a].fro, pp[a].Ek, &tr, P->s[a % kAxisStreams]);
    if (st != GGM_OK) first = st;
  }
  // join back onto `stream`
  for (int i = 0; i < nside; ++i) {
    GGM_CUDA_TRY(cudaEventRecord(P->ev[i], P->s[i]));
    GGM_CUDA_TRY(cudaStreamWaitEvent(s0, P->ev[i], 0));
  }
  if (first != GGM_OK) return first;
  // axes beyond the dense Gram: randomized subspace iteration on `stream`
  for (int a = 0; a < ndim; ++a) {
    if (dense[a]) continue;
    st = ggm_gram_eig(X, ndim, shape, a, k[a], V[a], E[a], &tr,
                      static_cast<char*>(workspace) + off[a],
                      (a + 1 < ndim ? off[a + 1] : need) - off[a], stream);
    if (st != GGM_OK) return st;
  }
  if (trace_S) *trace_S = tr;
  return GGM_OK;
}
