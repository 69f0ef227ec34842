// grid_solve.cu — Kronecker-sum eigenvalue MLE on the k-grid (Theorem 2, P:354-376;
// Algorithm 1 lines 5-17).
//
// The Thm 2 trace term for one modality is the vector of grid marginals
//     g_l[i] = Σ_{grid points j with j_l = i} 1 / s_j,   s_j = Σ_l λ_l[j_l]
// over all prod(k) grid points.  The grid is never stored: each pass regenerates s_j from
// the Σk eigenvalues held in shared memory (BK4 is bound by the reciprocal rate, not HBM).
//
// Solver: the multiplicative update λ ← λ ⊙ g / E.  It is the
// majorise-minimise step for the NLL (Jensen on -log s with weights λ_l[j_l]/s_j gives a
// separable majoriser whose minimiser is exactly λ g / E), so the NLL decreases
// monotonically and λ stays > 0: Algorithm 1's feasibility loop never triggers.
// By default the step is over-relaxed, λ ← λ ⊙ (g / E)^1.5 off the common-scale direction
// (same fixed point, λ still > 0, 20-37 % fewer iterations), with a plain-MM rerun if that
// does not converge (mm_omega).
// The whole loop runs in ONE cooperative persistent kernel: per iteration a grid pass
// (per-block partial marginals), grid.sync, a per-entry reduction + update + stationarity
// max, grid.sync.
//
// Layout of the pass: the axis with the largest k is the "inner" axis (contiguous in the
// lanes of a warp); every other axis is "outer".  One warp owns one outer multi-index row
// at a time: s = base(row) + λ_inner[m].  fp64 throughout: SFU-seeded fp64 reciprocals
// (one Newton step), per-lane accumulators, warp-shuffle row sums, shared-memory block
// partials and cross-block sums.  The pass is bound by the FP64 + SFU pipes, not HBM.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>

#include "ggm_internal.h"

namespace cg = cooperative_groups;

namespace ggm {
namespace gs {

constexpr int kMaxAxes = 8;
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

struct GridDesc {
  int L;                   // axes
  int inner;               // index of the inner axis (original order)
  int k[kMaxAxes];         // ranks, original order
  int off[kMaxAxes + 1];   // offsets into the concatenated vectors
  int outer_axes[kMaxAxes];  // original indices of outer axes, last = fastest
  int64_t outer_stride[kMaxAxes];  // row = Σ_a idx_a · outer_stride[a]
  int n_outer;
  int64_t rows;            // prod of outer k
  int total;               // Σ k
};


// One grid pass: this block's partial marginals in sg (fp64, Σk entries, zeroed by caller).
// slam: fp32 λ (Σk), in shared memory.
// Reciprocal of a positive double: MUFU 64-bit approximation (~2^-20 relative, the SFU
// pipe) refined by one Newton step on the FP64 pipe (error ~2^-40).
__device__ __forceinline__ double rcp_f64(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  const double e = fma(-s, r, 1.0);
  return fma(r, e, r);
}

// One grid pass over this block's share of the outer rows: per-lane fp64 accumulators for
// the inner axis, warp-shuffle row sums for the outer axes, fp64 shared-memory partials sg.
// All of s, 1/s and the sums are fp64 (no fixed fp32 rounding of λ or s that would floor
// the stationarity residual; e.g. the isotropic case, where every s_j is equal, would
// otherwise carry one identical rounding error in every term).
// NOUT = number of outer axes when known at compile time (0, 1, 2 cover L <= 3, i.e. every
// BASELINE config); -1 = generic.  The per-row bookkeeping (base sum, odometer, outer
// marginal atomics) is kept out of constant-bank indexing so that it stays small next to the
// k_inner points of the row.
template <int J, int NOUT>
__device__ void grid_pass_block(const GridDesc& gd, const double* slam, double* sg, int64_t gwarp,
                                int64_t nwarps) {
  constexpr int NO = NOUT < 0 ? kMaxAxes : (NOUT == 0 ? 1 : NOUT);
  const int lane = threadIdx.x & 31;
  const int kin = gd.k[gd.inner];
  const int oin = gd.off[gd.inner];
  const int nout = NOUT < 0 ? gd.n_outer : NOUT;
  int ko[NO], oo[NO], idx[NO];
  int64_t so[NO];
#pragma unroll
  for (int a = 0; a < NO; ++a) {
    const bool live = a < nout;
    ko[a] = live ? gd.k[gd.outer_axes[a]] : 1;
    oo[a] = live ? gd.off[gd.outer_axes[a]] : 0;
    so[a] = live ? gd.outer_stride[a] : 1;
  }
  double lv[J], acc[J];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const int m = lane + 32 * jj;
    lv[jj] = (m < kin) ? slam[oin + m] : 1.0;
    acc[jj] = 0.0;
  }
  // this warp's contiguous range of outer rows; the multi-index advances like an odometer
  const int64_t per = (gd.rows + nwarps - 1) / nwarps;
  const int64_t r0 = gwarp * per;
  const int64_t r1 = min(gd.rows, r0 + per);
#pragma unroll
  for (int a = 0; a < NO; ++a) idx[a] = a < nout ? (int)((r0 / so[a]) % ko[a]) : 0;
  for (int64_t row = r0; row < r1; ++row) {
    double base = 0.0;
#pragma unroll
    for (int a = 0; a < NO; ++a)
      if (a < nout) base += slam[oo[a] + idx[a]];
    double rsum = 0.0;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      const int m = lane + 32 * jj;
      if (m < kin) {
        const double r = rcp_f64(base + lv[jj]);
        rsum += r;
        acc[jj] += r;
      }
    }
    if (nout > 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
      // lane a adds the row sum to g_{outer axis a}[idx_a]
#pragma unroll
      for (int a = 0; a < NO; ++a)
        if (a < nout && lane == a) atomicAdd(&sg[oo[a] + idx[a]], rsum);
      // odometer: last outer axis fastest
      bool carry = true;
#pragma unroll
      for (int a = NO - 1; a >= 0; --a) {
        if (a < nout && carry) {
          if (++idx[a] == ko[a])
            idx[a] = 0;
          else
            carry = false;
        }
      }
    }
  }
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const int m = lane + 32 * jj;
    if (m < kin) atomicAdd(&sg[oin + m], acc[jj]);
  }
}

template <int J>
__device__ __forceinline__ void grid_pass(const GridDesc& gd, const double* slam, double* sg,
                                          int64_t gwarp, int64_t nwarps) {
  switch (gd.n_outer) {
    case 0: grid_pass_block<J, 0>(gd, slam, sg, gwarp, nwarps); break;
    case 1: grid_pass_block<J, 1>(gd, slam, sg, gwarp, nwarps); break;
    case 2: grid_pass_block<J, 2>(gd, slam, sg, gwarp, nwarps); break;
    default: grid_pass_block<J, -1>(gd, slam, sg, gwarp, nwarps); break;
  }
}

__device__ __forceinline__ void load_lambda(const double* lam, int total, double* slam,
                                            bool bypass_l1) {
  for (int i = threadIdx.x; i < total; i += blockDim.x)
    slam[i] = bypass_l1 ? __ldcg(&lam[i]) : lam[i];
}

constexpr int kMaxMods = 8;  // modalities of a multi-modal solve

// Exponent ω of the multiplicative update λ <- λ ⊙ (g/E)^ω.  ω = 1 is the MM step (monotone
// NLL); near the fixed point its error contracts by the MM Jacobian's eigenvalues μ ∈ [0, 1),
// over-relaxation maps them to 1 − ω(1 − μ) (still contracting for ω < 2 / (1 − μ_min)), which
// speeds the slow modes that set the iteration count; the common-scale direction (μ = 0) is
// left at the MM step (see solve_kernel).  Default 1.5 with a plain-MM rerun if it does not
// converge (solve_with_fallback); GGM_MM_OMEGA overrides (BK4 has the sweep).
static double mm_omega() {
  const char* e = std::getenv("GGM_MM_OMEGA");
  const double w = e ? std::atof(e) : 1.5;
  return (w > 0.0 && w < 2.0) ? w : 1.0;
}

struct SolveParams {
  GridDesc gd[kMaxMods];  // one per modality; offsets index the global concatenation
  int M;                  // modalities
  int T;                  // Σk over all axes
  const double* E;
  double* lam_out;    // converged λ (gauge 1: as iterated), Σk
  double* g;          // marginals at lam_out, Σk
  double* gacc;       // [3][Σk] rotating global accumulators of the block partials
  int* status;        // [0] iterations, [1] converged flag
  double* res_out;    // stationarity of lam_out
  double tol;
  int max_iter;
  double omega;       // update exponent: λ <- λ ⊙ (g / E)^omega (1 = the MM step)
};

// Whole MM iteration in one cooperative kernel with ONE grid-wide barrier per iteration:
// every block keeps its own copy of λ in shared memory; block partial marginals are added
// atomically into global slot it%3; after grid.sync every block reads the same sums,
// computes the same residual and the same update (bitwise identical in all blocks).
// Slot (it+1)%3 is cleared by block 0 during iteration it: its last readers finished before
// the barrier of iteration it-1, and its next writers start after the barrier of it.
template <int J>
__global__ void __launch_bounds__(kThreads, 1) solve_kernel(const SolveParams p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dsm[];
  const int T = p.T;
  double* sg = dsm;        // Σk block partials, then the reduced marginals
  double* slam = sg + T;   // Σk this block's λ
  __shared__ double s_red[kWarps];
  __shared__ double s_emax;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < T; i += blockDim.x) slam[i] = 1.0 / p.E[i];  // Alg. 1 line 5
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < T; ++i) m = fmax(m, p.E[i]);
    s_emax = m;
  }
  const int64_t gw = (int64_t)blockIdx.x * kWarps + wid;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  int it = 0;
  bool done = false;
  double res = 0.0;
  const bool single = gridDim.x == 1;
  for (;; ++it) {
    for (int i = threadIdx.x; i < T; i += blockDim.x) sg[i] = 0.0;
    if (blockIdx.x == 0 && !single)
      for (int i = threadIdx.x; i < T; i += blockDim.x) p.gacc[(size_t)((it + 1) % 3) * T + i] = 0.0;
    __syncthreads();
    // Σ_γ of the modalities' marginals (Thm 2): each pass adds into the same sg
    for (int m = 0; m < p.M; ++m) grid_pass<J>(p.gd[m], slam, sg, gw, nw);
    __syncthreads();
    double mr = 0.0;
    if (single) {  // one block: the block partials are the marginals, no grid barrier
      for (int i = threadIdx.x; i < T; i += blockDim.x) mr = fmax(mr, fabs(p.E[i] - sg[i]));
    } else {
      double* acc = p.gacc + (size_t)(it % 3) * T;
      for (int i = threadIdx.x; i < T; i += blockDim.x) atomicAdd(&acc[i], sg[i]);
      grid.sync();
      // reduced marginals g (identical in every block), stationarity max |E - g| / max E
      for (int i = threadIdx.x; i < T; i += blockDim.x) {
        const double gi = __ldcg(&acc[i]);
        sg[i] = gi;
        mr = fmax(mr, fabs(p.E[i] - gi));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    if (lane == 0) s_red[wid] = mr;
    __syncthreads();
    mr = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) mr = fmax(mr, s_red[w]);
    res = mr / s_emax;
    if (res <= p.tol) {
      done = true;
      break;
    }
    if (it == p.max_iter) break;
    // majorise-minimise update λ <- λ ⊙ g / E
    if (p.omega == 1.0) {
      for (int i = threadIdx.x; i < T; i += blockDim.x) slam[i] = slam[i] * sg[i] / p.E[i];
    } else {
      // log-space step δ_i = log(g_i / E_i); its mean m is the common-scale direction, which
      // the MM step already solves exactly (the map is invariant to λ -> cλ), so only
      // δ − m is over-relaxed: λ_i <- λ_i exp(m + ω (δ_i − m)).  The block reduction runs in
      // the same order in every block (bitwise-identical λ copies).
      double part = 0.0;
      for (int i = threadIdx.x; i < T; i += blockDim.x) {
        const double d = log(sg[i] / p.E[i]);
        sg[i] = d;
        part += d;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      __syncthreads();  // every warp has read s_red (the stationarity max)
      if (lane == 0) s_red[wid] = part;
      __syncthreads();
      double m = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) m += s_red[w];
      m /= T;
      for (int i = threadIdx.x; i < T; i += blockDim.x)
        slam[i] = slam[i] * exp(m + p.omega * (sg[i] - m));
    }
    __syncthreads();
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
      p.lam_out[i] = slam[i];
      p.g[i] = sg[i];
    }
    if (threadIdx.x == 0) {
      p.status[0] = it;
      p.status[1] = done ? 1 : 0;
      *p.res_out = res;
    }
  }
}

// Stand-alone single pass (ggm_grid_marginals / final NLL): partials into [Σk][grid].
template <int J>
__global__ void __launch_bounds__(kThreads, 1) marginal_pass_kernel(GridDesc gd, const double* lam,
                                                                     double* partial) {
  extern __shared__ double dsm[];
  double* sg = dsm;
  double* slam = sg + gd.total;
  for (int i = threadIdx.x; i < gd.total; i += blockDim.x) sg[i] = 0.0;
  load_lambda(lam, gd.total, slam, false);
  __syncthreads();
  grid_pass<J>(gd, slam, sg, (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5),
               (int64_t)gridDim.x * kWarps);
  __syncthreads();
  for (int i = threadIdx.x; i < gd.total; i += blockDim.x)
    partial[(size_t)i * gridDim.x + blockIdx.x] = sg[i];
}

__global__ void reduce_partials(const double* partial, int nblk, int total, double* g) {
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= total) return;
  double sum = 0.0;
  for (int b = lane; b < nblk; b += 32) sum += partial[(size_t)e * nblk + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) g[e] = sum;
}

// Σ_j log s_j over the grid (fp64; a one-off diagnostic pass) -> logsum (atomic).
__global__ void logsum_kernel(GridDesc gd, const double* lam, double* logsum) {
  const int kin = gd.k[gd.inner];
  double acc = 0.0;
  const int lane = threadIdx.x & 31;
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < gd.rows;
       row += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    double base = 0.0;
    for (int a = 0; a < gd.n_outer; ++a) {
      const int ax = gd.outer_axes[a];
      base += lam[gd.off[ax] + (int)((row / gd.outer_stride[a]) % gd.k[ax])];
    }
    for (int m = lane; m < kin; m += 32) acc += log(base + lam[gd.off[gd.inner] + m]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) atomicAdd(logsum, acc);
}

// Final: choose result buffer, canonical gauge, write λ out; compute grid_min, floor.
__global__ void finalize_kernel(GridDesc gd, const double* lam_res, int gauge, double* lam_out,
                                double* scalars /* [0]=smin */) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mins[kMaxAxes];
  double smin = 0.0;
  for (int a = 0; a < gd.L; ++a) {
    double m = lam_res[gd.off[a]];
    for (int i = 1; i < gd.k[a]; ++i) m = fmin(m, lam_res[gd.off[a] + i]);
    mins[a] = m;
    smin += m;
  }
  for (int a = 0; a < gd.L; ++a) {
    const double shift = gauge == 0 ? (-mins[a] + smin / gd.L) : 0.0;
    for (int i = 0; i < gd.k[a]; ++i) lam_out[gd.off[a] + i] = lam_res[gd.off[a] + i] + shift;
  }
  scalars[0] = smin;
}

__global__ void check_E(const double* E, int total, int* bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const double e = E[i];
    if (!(e > 0.0) || !isfinite(e)) atomicOr(bad, 1);
  }
}

__global__ void init_lambda(const double* E, int total, double* lam) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x)
    lam[i] = 1.0 / E[i];  // Algorithm 1 line 5
}

static ggm_status make_desc(int L, const int* k, GridDesc* gd) {
  if (L < 1 || L > kMaxAxes) return fail(GGM_ERR_INVALID_ARGUMENT, "L=%d not in [1,%d]", L, kMaxAxes);
  if (!k) return fail(GGM_ERR_INVALID_ARGUMENT, "k is NULL");
  gd->L = L;
  gd->off[0] = 0;
  int inner = 0;
  double prod = 1.0;
  for (int a = 0; a < L; ++a) {
    if (k[a] < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "k[%d]=%d < 1", a, k[a]);
    gd->k[a] = k[a];
    gd->off[a + 1] = gd->off[a] + k[a];
    if (k[a] > k[inner]) inner = a;
    prod *= k[a];
  }
  if (prod >= 1099511627776.0) return fail(GGM_ERR_INVALID_ARGUMENT, "grid too large (>= 2^40)");
  if (k[inner] > 1024)
    return fail(GGM_ERR_UNSUPPORTED, "largest rank %d > 1024 not supported by grid_solve", k[inner]);
  gd->inner = inner;
  gd->n_outer = 0;
  gd->rows = 1;
  for (int a = 0; a < L; ++a)
    if (a != inner) {
      gd->outer_axes[gd->n_outer++] = a;
      gd->rows *= k[a];
    }
  int64_t stride = 1;
  for (int a = gd->n_outer - 1; a >= 0; --a) {
    gd->outer_stride[a] = stride;
    stride *= k[gd->outer_axes[a]];
  }
  gd->total = gd->off[L];
  return GGM_OK;
}

// Modality descriptor: axes `ax[0..L)` of the global axes (ranks kg, offsets offg), so the
// pass indexes λ and accumulates the marginals directly in the global concatenation.
static ggm_status make_desc_mod(int L, const int* ax, const int* kg, const int* offg, int T,
                                GridDesc* gd) {
  if (L < 1 || L > kMaxAxes) return fail(GGM_ERR_INVALID_ARGUMENT, "modality with %d axes", L);
  int kl[kMaxAxes];
  for (int a = 0; a < L; ++a) kl[a] = kg[ax[a]];
  ggm_status st = make_desc(L, kl, gd);
  if (st != GGM_OK) return st;
  for (int a = 0; a < L; ++a) gd->off[a] = offg[ax[a]];
  gd->off[L] = T;
  gd->total = T;
  return GGM_OK;
}

static int pick_J(int kin) { return kin <= 128 ? 4 : kin <= 256 ? 8 : kin <= 512 ? 16 : 32; }

static size_t pass_smem(const GridDesc& gd) {
  return (size_t)gd.total * 2 * sizeof(double) + 16;
}

template <int J>
static cudaError_t set_attrs(size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(solve_kernel<J>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(marginal_pass_kernel<J>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

static int grid_blocks(const GridDesc& gd) {
  const int64_t warps_needed = std::max<int64_t>(1, gd.rows);
  const int64_t blocks = (warps_needed + kWarps - 1) / kWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, num_sms()));
}

// Blocks for the cooperative solve: enough warps that each owns >= ~8 outer rows (a grid
// barrier costs microseconds; small grids run in one block).
static int solve_blocks(const GridDesc& gd, double extra_pts = 0.0) {
  const double pts = (double)gd.rows * gd.k[gd.inner] + extra_pts;
  const int64_t want = (int64_t)std::ceil(pts / (kWarps * 8.0 * 32.0 * 16.0));
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, num_sms()));
}

static cudaError_t launch_pass(const GridDesc& gd, const double* lam, double* partial, int nblk,
                               cudaStream_t s) {
  const size_t smem = pass_smem(gd);
  const int J = pick_J(gd.k[gd.inner]);
  cudaError_t e;
  switch (J) {
    case 4: e = set_attrs<4>(smem); if (e) return e; marginal_pass_kernel<4><<<nblk, kThreads, smem, s>>>(gd, lam, partial); break;
    case 8: e = set_attrs<8>(smem); if (e) return e; marginal_pass_kernel<8><<<nblk, kThreads, smem, s>>>(gd, lam, partial); break;
    case 16: e = set_attrs<16>(smem); if (e) return e; marginal_pass_kernel<16><<<nblk, kThreads, smem, s>>>(gd, lam, partial); break;
    default: e = set_attrs<32>(smem); if (e) return e; marginal_pass_kernel<32><<<nblk, kThreads, smem, s>>>(gd, lam, partial); break;
  }
  return cudaGetLastError();
}

template <int J>
static cudaError_t launch_solve(const SolveParams& sp, int nblk, size_t smem, cudaStream_t s) {
  cudaError_t e = set_attrs<J>(smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<J>, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  void* args[] = {const_cast<SolveParams*>(&sp)};
  return cudaLaunchCooperativeKernel((void*)solve_kernel<J>, dim3(nblk), dim3(kThreads), args, smem,
                                     s);
}

}  // namespace gs
}  // namespace ggm

using namespace ggm;
using namespace ggm::gs;

extern "C" void ggm_solve_opts_default(ggm_solve_opts* o) {
  if (!o) return;
  o->tol = 1e-7;
  o->max_iter = 20000;
  o->eps_scale = 1e-10;
  o->method = 0;
  o->gauge = 0;
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

extern "C" ggm_status ggm_grid_marginals(int L, const int* k, const double* lambda, double* g,
                                         double* logsum_out, void* stream) {
  GridDesc gd;
  ggm_status st = make_desc(L, k, &gd);
  if (st != GGM_OK) return st;
  if (!lambda || !g) return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nblk = grid_blocks(gd);
  DevBuf buf;
  GGM_CUDA_TRY(cudaMallocAsync(&buf.p, (size_t)gd.total * nblk * sizeof(double) + 64, s));
  double* partial = static_cast<double*>(buf.p);
  GGM_CUDA_TRY(launch_pass(gd, lambda, partial, nblk, s));
  reduce_partials<<<(gd.total + 7) / 8, 256, 0, s>>>(partial, nblk, gd.total, g);
  GGM_CUDA_TRY(cudaGetLastError());
  if (logsum_out) {
    double* dls = partial + (size_t)gd.total * nblk;
    GGM_CUDA_TRY(cudaMemsetAsync(dls, 0, sizeof(double), s));
    logsum_kernel<<<num_sms() * 4, 256, 0, s>>>(gd, lambda, dls);
    GGM_CUDA_TRY(cudaGetLastError());
    GGM_CUDA_TRY(cudaMemcpyAsync(logsum_out, dls, sizeof(double), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
  }
  GGM_CUDA_TRY(cudaFreeAsync(buf.p, s));
  buf.p = nullptr;
  return GGM_OK;
}

// The solve kernel with update exponent sp.omega; an over-relaxed run (omega > 1) that does
// not converge is repeated with the plain MM step (omega = 1, monotone NLL), and its
// iterations are returned in *extra.
static ggm_status solve_with_fallback(SolveParams sp, int J, int nblk, size_t smem,
                                      cudaStream_t s, const int* istat, int* extra) {
  auto launch = [&]() -> cudaError_t {
    switch (J) {
      case 4: return launch_solve<4>(sp, nblk, smem, s);
      case 8: return launch_solve<8>(sp, nblk, smem, s);
      case 16: return launch_solve<16>(sp, nblk, smem, s);
      default: return launch_solve<32>(sp, nblk, smem, s);
    }
  };
  *extra = 0;
  cudaError_t ce = launch();
  if (ce != cudaSuccess) return fail(GGM_ERR_CUDA, "solve_kernel launch: %s", cudaGetErrorString(ce));
  if (sp.omega != 1.0) {
    int h[2] = {0, 0};
    GGM_CUDA_TRY(cudaMemcpyAsync(h, istat, sizeof(h), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    if (!h[1]) {
      *extra = h[0];
      sp.omega = 1.0;
      ce = launch();
      if (ce != cudaSuccess)
        return fail(GGM_ERR_CUDA, "solve_kernel launch: %s", cudaGetErrorString(ce));
    }
  }
  return GGM_OK;
}

extern "C" ggm_status ggm_solve_eigvals(int L, const int* k, const double* E,
                                        const ggm_solve_opts* opts, double* lambda,
                                        ggm_solve_info* info, void* stream) {
  GridDesc gd;
  ggm_status st = make_desc(L, k, &gd);
  if (st != GGM_OK) return st;
  if (!E || !lambda) return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer");
  ggm_solve_opts o;
  ggm_solve_opts_default(&o);
  if (opts) o = *opts;
  if (!(o.tol > 0.0) || o.max_iter < 0 || !(o.eps_scale >= 0.0))
    return fail(GGM_ERR_INVALID_ARGUMENT, "invalid solve options");
  if (o.method != 0)
    return fail(GGM_ERR_UNSUPPORTED, "method %d not implemented on the GPU (use 0)", o.method);
  if (o.gauge != 0 && o.gauge != 1) return fail(GGM_ERR_INVALID_ARGUMENT, "gauge=%d", o.gauge);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nblk = solve_blocks(gd);
  const size_t T = gd.total;
  // scratch: lam_res, g, gacc[3T], scalars[4] (smin, logsum, res), status[4]
  const size_t bytes = sizeof(double) * (5 * T + 8) + 64;
  DevBuf buf;
  GGM_CUDA_TRY(cudaMallocAsync(&buf.p, bytes, s));
  double* lam_res = static_cast<double*>(buf.p);
  double* g = lam_res + T;
  double* gacc = g + T;
  double* scal = gacc + 3 * T;  // [0] smin, [1] logsum, [2] residual
  int* istat = reinterpret_cast<int*>(scal + 4);  // [0] iterations, [1] converged, [3] bad
  GGM_CUDA_TRY(cudaMemsetAsync(gacc, 0, sizeof(double) * (3 * T + 8) + 64, s));
  check_E<<<4, 256, 0, s>>>(E, gd.total, istat + 3);
  GGM_CUDA_TRY(cudaGetLastError());
  int hbad = 0;
  GGM_CUDA_TRY(cudaMemcpyAsync(&hbad, istat + 3, sizeof(int), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad) return fail(GGM_ERR_DOMAIN, "E must be finite and > 0 (Thm 4, P:742)");

  SolveParams sp;
  sp.gd[0] = gd;
  sp.M = 1;
  sp.T = gd.total;
  sp.E = E;
  sp.lam_out = lam_res;
  sp.g = g;
  sp.gacc = gacc;
  sp.status = istat;
  sp.res_out = scal + 2;
  sp.tol = o.tol;
  sp.max_iter = o.max_iter;
  sp.omega = mm_omega();
  const size_t smem = pass_smem(gd);
  int extra_it = 0;
  ggm_status sst = solve_with_fallback(sp, pick_J(gd.k[gd.inner]), nblk, smem, s, istat, &extra_it);
  if (sst != GGM_OK) return sst;
  int hstat[2] = {0, 0};
  GGM_CUDA_TRY(cudaMemcpyAsync(hstat, istat, sizeof(hstat), cudaMemcpyDeviceToHost, s));
  finalize_kernel<<<1, 32, 0, s>>>(gd, lam_res, o.gauge, lambda, scal);
  logsum_kernel<<<num_sms() * 4, 256, 0, s>>>(gd, lam_res, scal + 1);
  GGM_CUDA_TRY(cudaGetLastError());
  // residual of the returned λ (its marginals are in g)
  double hres = 0.0;
  {
    double hscal[3];
    GGM_CUDA_TRY(cudaMemcpyAsync(hscal, scal, sizeof(hscal), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    hres = hscal[2];
    if (info) {
      std::vector<double> hE(T), hL(T);
      GGM_CUDA_TRY(cudaMemcpy(hE.data(), E, T * sizeof(double), cudaMemcpyDeviceToHost));
      GGM_CUDA_TRY(cudaMemcpy(hL.data(), lam_res, T * sizeof(double), cudaMemcpyDeviceToHost));
      double lin = 0.0;
      for (size_t i = 0; i < T; ++i) lin += hE[i] * hL[i];
      std::vector<double> tr(L, 0.0);
      double mean = 0.0;
      for (int a = 0; a < L; ++a) {
        for (int i = gd.off[a]; i < gd.off[a + 1]; ++i) tr[a] += hE[i];
        mean += tr[a] / L;
      }
      double ti = 0.0;
      for (int a = 0; a < L; ++a) ti = std::max(ti, std::fabs(tr[a] - mean));
      info->iterations = hstat[0] + extra_it;
      info->stationarity = hres;
      info->nll = 0.5 * lin - 0.5 * hscal[1];
      info->grid_min = hscal[0];
      double emax = 0.0;
      for (size_t i = 0; i < T; ++i) emax = std::max(emax, 1.0 / hE[i]);
      info->floor_active = hscal[0] <= o.eps_scale * emax ? 1 : 0;
      info->trace_inconsistency = mean > 0 ? ti / mean : 0.0;
    }
  }
  GGM_CUDA_TRY(cudaFreeAsync(buf.p, s));
  buf.p = nullptr;
  if (!hstat[1])
    return fail(GGM_ERR_NO_CONVERGENCE, "no convergence in %d iterations (residual %.3e)",
                o.max_iter, hres);
  return GGM_OK;
}

// ------------------------------------------------------------------ multi-modal solve
// Thm 2 with Σ_γ: NLL = ½ Σ_l E_l·λ_l − ½ Σ_γ Σ_{j∈grid γ} log s^γ_j, gradient
// ½(E_l − Σ_{γ∋l} g^γ_l).  The majorise-minimise step is unchanged (one Jensen majoriser
// per modality, summed): λ ← λ ⊙ (Σ_γ g^γ) / E, so the same persistent kernel runs with one
// grid pass per modality per iteration.  Gauge (reading G2): shifts c with Σ_{l∈γ} c_l = 0
// for every γ leave all grid sums unchanged; gauge 0 subtracts the G-component of the axis
// minima (for one modality: the min-balanced gauge of ggm_solve_eigvals).
extern "C" ggm_status ggm_solve_eigvals_multi(int A, const int* k, const double* E, int M,
                                              const int* mod_ptr, const int* mod_axes,
                                              const ggm_solve_opts* opts, double* lambda,
                                              ggm_solve_info* info, void* stream) {
  if (A < 1 || A > 64 || !k || !E || !lambda || !mod_ptr || !mod_axes)
    return fail(GGM_ERR_INVALID_ARGUMENT, "invalid axes / null pointer");
  if (M < 1 || M > kMaxMods) return fail(GGM_ERR_INVALID_ARGUMENT, "M=%d not in [1,%d]", M, kMaxMods);
  std::vector<int> offg(A + 1, 0), seen(A, 0);
  for (int a = 0; a < A; ++a) {
    if (k[a] < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "k[%d] < 1", a);
    offg[a + 1] = offg[a] + k[a];
  }
  const int T = offg[A];
  SolveParams sp;
  memset(&sp, 0, sizeof(sp));
  double pts = 0.0;
  int J = 4;
  for (int g = 0; g < M; ++g) {
    const int L = mod_ptr[g + 1] - mod_ptr[g];
    const int* ax = mod_axes + mod_ptr[g];
    std::vector<int> here(A, 0);
    for (int a = 0; a < L; ++a) {
      if (ax[a] < 0 || ax[a] >= A) return fail(GGM_ERR_INVALID_ARGUMENT, "axis id out of range");
      if (here[ax[a]]++) return fail(GGM_ERR_INVALID_ARGUMENT, "repeated axis in a modality (P:181)");
      seen[ax[a]] = 1;
    }
    ggm_status st = make_desc_mod(L, ax, k, offg.data(), T, &sp.gd[g]);
    if (st != GGM_OK) return st;
    pts += (double)sp.gd[g].rows * sp.gd[g].k[sp.gd[g].inner];
    J = std::max(J, pick_J(sp.gd[g].k[sp.gd[g].inner]));
  }
  for (int a = 0; a < A; ++a)
    if (!seen[a]) return fail(GGM_ERR_INVALID_ARGUMENT, "axis %d occurs in no modality", a);
  ggm_solve_opts o;
  ggm_solve_opts_default(&o);
  if (opts) o = *opts;
  if (!(o.tol > 0.0) || o.max_iter < 0 || !(o.eps_scale >= 0.0))
    return fail(GGM_ERR_INVALID_ARGUMENT, "invalid solve options");
  if (o.method != 0)
    return fail(GGM_ERR_UNSUPPORTED, "method %d not implemented on the GPU (use 0)", o.method);
  if (o.gauge != 0 && o.gauge != 1) return fail(GGM_ERR_INVALID_ARGUMENT, "gauge=%d", o.gauge);
  sp.M = M;
  sp.T = T;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t bytes = sizeof(double) * (5 * (size_t)T + 8) + 64;
  DevBuf buf;
  GGM_CUDA_TRY(cudaMallocAsync(&buf.p, bytes, s));
  double* lam_res = static_cast<double*>(buf.p);
  double* g = lam_res + T;
  double* gacc = g + T;
  double* scal = gacc + 3 * (size_t)T;  // [1] logsum, [2] residual
  int* istat = reinterpret_cast<int*>(scal + 4);
  GGM_CUDA_TRY(cudaMemsetAsync(gacc, 0, sizeof(double) * (3 * (size_t)T + 8) + 64, s));
  check_E<<<4, 256, 0, s>>>(E, T, istat + 3);
  GGM_CUDA_TRY(cudaGetLastError());
  int hbad = 0;
  GGM_CUDA_TRY(cudaMemcpyAsync(&hbad, istat + 3, sizeof(int), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad) return fail(GGM_ERR_DOMAIN, "E must be finite and > 0 (Thm 4, P:742)");
  sp.E = E;
  sp.lam_out = lam_res;
  sp.g = g;
  sp.gacc = gacc;
  sp.status = istat;
  sp.res_out = scal + 2;
  sp.tol = o.tol;
  sp.max_iter = o.max_iter;
  sp.omega = mm_omega();
  const int nblk = solve_blocks(sp.gd[0], pts - (double)sp.gd[0].rows * sp.gd[0].k[sp.gd[0].inner]);
  const size_t smem = (size_t)T * 2 * sizeof(double) + 16;
  int extra_it = 0;
  ggm_status sst = solve_with_fallback(sp, J, nblk, smem, s, istat, &extra_it);
  if (sst != GGM_OK) return sst;
  for (int m = 0; m < M; ++m) logsum_kernel<<<num_sms() * 4, 256, 0, s>>>(sp.gd[m], lam_res, scal + 1);
  GGM_CUDA_TRY(cudaGetLastError());
  int hstat[2] = {0, 0};
  double hscal[3] = {0, 0, 0};
  std::vector<double> hL(T), hE(T);
  GGM_CUDA_TRY(cudaMemcpyAsync(hstat, istat, sizeof(hstat), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(hscal, scal, sizeof(hscal), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(hL.data(), lam_res, sizeof(double) * T, cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(hE.data(), E, sizeof(double) * T, cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  // gauge space G = null(incidence): orthonormal basis R of the row space by Gram-Schmidt;
  // P_G x = x - Σ_r (r·x) r
  std::vector<std::vector<double>> R;
  for (int gm = 0; gm < M; ++gm) {
    std::vector<double> v(A, 0.0);
    for (int q = mod_ptr[gm]; q < mod_ptr[gm + 1]; ++q) v[mod_axes[q]] = 1.0;
    for (int pass = 0; pass < 2; ++pass)
      for (const auto& r : R) {
        double dt = 0.0;
        for (int a = 0; a < A; ++a) dt += r[a] * v[a];
        for (int a = 0; a < A; ++a) v[a] -= dt * r[a];
      }
    double nv = 0.0;
    for (double x : v) nv += x * x;
    if (nv > 1e-20) {
      nv = std::sqrt(nv);
      for (double& x : v) x /= nv;
      R.push_back(v);
    }
  }
  auto proj_G = [&](const std::vector<double>& x) {
    std::vector<double> y = x;
    for (const auto& r : R) {
      double dt = 0.0;
      for (int a = 0; a < A; ++a) dt += r[a] * x[a];
      for (int a = 0; a < A; ++a) y[a] -= dt * r[a];
    }
    return y;
  };
  std::vector<double> mins(A), tr(A, 0.0);
  for (int a = 0; a < A; ++a) {
    double mn = hL[offg[a]];
    for (int i = offg[a]; i < offg[a + 1]; ++i) {
      mn = std::min(mn, hL[i]);
      tr[a] += hE[i];
    }
    mins[a] = mn;
  }
  const std::vector<double> shift = o.gauge == 0 ? proj_G(mins) : std::vector<double>(A, 0.0);
  std::vector<double> out(T);
  for (int a = 0; a < A; ++a)
    for (int i = offg[a]; i < offg[a + 1]; ++i) out[i] = hL[i] - shift[a];
  GGM_CUDA_TRY(cudaMemcpyAsync(lambda, out.data(), sizeof(double) * T, cudaMemcpyHostToDevice, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (info) {
    double lin = 0.0, emax = 0.0;
    for (int i = 0; i < T; ++i) {
      lin += hE[i] * hL[i];
      emax = std::max(emax, 1.0 / hE[i]);
    }
    double gmin = INFINITY;
    for (int gm = 0; gm < M; ++gm) {
      double sm = 0.0;
      for (int q = mod_ptr[gm]; q < mod_ptr[gm + 1]; ++q) sm += mins[mod_axes[q]];
      gmin = std::min(gmin, sm);
    }
    const std::vector<double> ptr = proj_G(tr);
    double trmean = 0.0, ti = 0.0;
    for (int a = 0; a < A; ++a) trmean += tr[a] / A;
    for (int a = 0; a < A; ++a) ti = std::max(ti, std::fabs(ptr[a]));
    info->iterations = hstat[0] + extra_it;
    info->stationarity = hscal[2];
    info->nll = 0.5 * lin - 0.5 * hscal[1];
    info->grid_min = gmin;
    info->floor_active = gmin <= o.eps_scale * emax ? 1 : 0;
    info->trace_inconsistency = trmean > 0 ? ti / trmean : 0.0;
  }
  GGM_CUDA_TRY(cudaFreeAsync(buf.p, s));
  buf.p = nullptr;
  if (!hstat[1])
    return fail(GGM_ERR_NO_CONVERGENCE, "no convergence in %d iterations (residual %.3e)",
                o.max_iter, hscal[2]);
  return GGM_OK;
}
