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

#include <algorithm>
#include <cmath>
#include <cstdint>
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
static size_t rcarve(const RPlan& rp, void* ws, RWork* w) {
  Carve c(ws);
  w->M = c.take<double>((size_t)rp.d * rp.m);
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

// Randomized subspace iteration on the unfolding already in w.M (d x m column-major) and its
// squared Frobenius norm in w.fro.
static ggm_status rsi_core(const RPlan& rp, const RWork& w, int max_iter, double tol,
                           uint64_t seed, float* V, double* E, double* trace_S, int* iters_out,
                           double* change_out, cublasHandle_t hb, cusolverDnHandle_t hs,
                           cudaStream_t s) {
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
  // range finder: Y = M Omega, Q = orth(Y)
  if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, d, r, m, &one, w.M, d, w.Om, m, &zero, w.Y, d) !=
      CUBLAS_STATUS_SUCCESS)
    return fail(GGM_ERR_CUDA, "cublasDgemm failed");
  st = orth(w.Y);
  if (st != GGM_OK) return st;
  std::vector<double> prev(kk, 0.0), cur(kk);
  int it = 0;
  double change = INFINITY;
  for (it = 1; it <= max_iter; ++it) {
    // Rayleigh-Ritz on span(Q): Z = M^T Q (m x r), T = Z^T Z = Q^T S Q (r x r)
    if (cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, m, r, d, &one, w.M, d, w.Y, d, &zero, w.Om, m) !=
            CUBLAS_STATUS_SUCCESS ||
        cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, r, m, &one, w.Om, m, &zero, w.T, r) !=
            CUBLAS_STATUS_SUCCESS)
      return fail(GGM_ERR_CUDA, "cuBLAS Rayleigh-Ritz failed");
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
    // power step: Y = M Z = S Q, Q = orth(Y)
    if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, d, r, m, &one, w.M, d, w.Om, m, &zero, w.Y, d) !=
        CUBLAS_STATUS_SUCCESS)
      return fail(GGM_ERR_CUDA, "cublasDgemm failed");
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
  return dense_core(g, lwork, Md, S, w, work, dinfo, V64, fro, Ek, Vasc, V, E, trace_S, hb, hs, s);
}

// Gram + eigensolve + top-k mapping on the unfolding already in Md (GPlan g decides the side).
static ggm_status dense_core(const GPlan& g, int lwork, double* Md, double* S, double* w,
                             double* work, int* dinfo, double* V64, double* fro, double* Ek,
                             double* Vasc, float* V, double* E, double* trace_S,
                             cublasHandle_t hb, cusolverDnHandle_t hs, cudaStream_t s) {
  const double one = 1.0, zero = 0.0;
  cublasStatus_t bs;
  if (g.mode == 2)  // S = M^T M  (m x m), M is d x m column-major
    bs = cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, (int)g.dim, (int)g.Md_rows, &one, Md,
                     (int)g.Md_rows, &zero, S, (int)g.dim);
  else              // S = M M^T  (Md_rows x Md_rows)
    bs = cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, (int)g.dim, (int)g.Md_cols, &one, Md,
                     (int)g.Md_rows, &zero, S, (int)g.dim);
  if (bs != CUBLAS_STATUS_SUCCESS) return fail(GGM_ERR_CUDA, "cublasDsyrk failed (%d)", (int)bs);
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
