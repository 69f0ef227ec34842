// grid_solve.cu — Kronecker-sum eigenvalue MLE on the k-grid (Theorem 2, P:354-376;
// Algorithm 1 lines 5-17; the domain Λ_l >= ε of Lemma 6).
//
// The Thm 2 trace term for one modality is the vector of grid marginals
//     g_l[i] = Σ_{grid points j with j_l = i} 1 / s_j,   s_j = Σ_l λ_l[j_l]
// over all prod(k) grid points.  The grid is never stored: each pass regenerates s_j from
// the Σk eigenvalues held in shared memory (BK4 is bound by the FP64 + SFU pipes, not HBM).
//
// Solver (BK4): the majorise-minimise step λ ← λ ⊙ g / E.  Jensen on -log s with
// weights λ_l[j_l]/s_j gives a separable majoriser of the NLL whose minimiser is
// exactly λ g / E (on the box λ >= ε: max(ε, λ g / E)), so the NLL decreases monotonically
// and λ stays > 0.  Method 0 accelerates the fixed point with SQUAREM (squared extrapolation
// in log space: two map evaluations, one extrapolated point, one stabilising evaluation per
// cycle; the extrapolation is kept only if its residual does not exceed the plain iterate's),
// 3-4x fewer grid passes; method 2 runs Algorithm 1's gradient descent as printed.
// The whole loop runs in ONE cooperative persistent kernel: per pass, the grid reduction into
// per-block partials, one grid-wide barrier, and an update computed identically (bitwise) by
// every block from the same reduced marginals.
//
// Layout of the pass: the axis with the largest k is the "inner" axis (contiguous in the
// lanes of a warp, ⌈k/32⌉ points per lane); the other axes are "outer" and one outer
// multi-index = one row.  A warp owns a contiguous range of rows.  Per grid point: one fp64
// add (s), one SFU reciprocal seed + two FP64 FMAs (Newton), two fp64 adds (the inner
// marginal in a per-lane register, the row sum).  Row sums are reduced four rows at a time
// by a reduce-scatter across the warp and added into per-warp private shared-memory bins of
// the fastest outer axis; the slowest outer axis (L = 3) changes once per k_fast rows and is
// accumulated in a register.  No fp64 shared-memory atomics in the per-row path.
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
#ifndef GGM_SOLVE_THREADS
#define GGM_SOLVE_THREADS 512
#endif
#ifndef GGM_SOLVE_MINB
#define GGM_SOLVE_MINB 1
#endif
constexpr int kThreads = GGM_SOLVE_THREADS;
constexpr int kWarps = kThreads / 32;
#ifndef GGM_SOLVE_RED_GROUPS
#define GGM_SOLVE_RED_GROUPS 4
#endif
// red_mode 2 (default): accumulator copies, block b adds into copy b mod kRedGroups.  C3 solve
// kernel: 4 copies 1.003 ms, 8 1.015, 16 1.052, one accumulator (red_mode 0) 1.065
// (profiles/r02_logs/r02k_redgroups.log, r02k_red2.log)
constexpr int kRedGroups = GGM_SOLVE_RED_GROUPS;
constexpr int kMaxFastBins = 1024;  // private per-warp bins: kWarps x k_fast doubles

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

// Reciprocal of a positive double: MUFU 64-bit approximation (~2^-20 relative, the SFU
// pipe) refined by one Newton step on the FP64 pipe (error ~2^-40).
__device__ __forceinline__ double rcp_f64(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  const double e = fma(-s, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Reduce-scatter of four per-lane row partials: returns, in lanes 0, 8, 16, 24, the warp
// totals of rows 0, 1, 2, 3 (other lanes: partial garbage).  6 fp64 shuffles for 4 rows.
__device__ __forceinline__ double reduce4(const double (&p)[4], int lane) {
  const bool b4 = (lane & 16) != 0, b3 = (lane & 8) != 0;
  const double k0 = b4 ? p[2] : p[0], k1 = b4 ? p[3] : p[1];
  const double s0 = b4 ? p[0] : p[2], s1 = b4 ? p[1] : p[3];
  const double a0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
  const double a1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
  double b = (b3 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, b3 ? a0 : a1, 8);
  b += __shfl_xor_sync(0xffffffffu, b, 4);
  b += __shfl_xor_sync(0xffffffffu, b, 2);
  b += __shfl_xor_sync(0xffffffffu, b, 1);
  return b;
}

// One grid pass over this block's share of the outer rows, for NOUT outer axes (0, 1, 2:
// every L <= 3, i.e. every BASELINE config).  slam: λ (Σk, fp64, shared); sg: this block's
// marginal partials (Σk [+1: Σ log s when LOGS], shared, zeroed by the caller); pw: kWarps x
// k_fast private bins (shared, zero on entry, zero again on exit).
// A warp's rows are cut into segments of constant slow index (at most k_fast rows, the fast
// index running fi, fi+1, ... without wrap) and each segment into groups of four rows that
// are evaluated together: 4 x J independent point chains, no per-row branches, one
// reduce-scatter per group, four distinct private bins.
template <int J, bool LOGS>
__device__ __forceinline__ void point_row(const double (&lv)[J], double (&acc)[J], double base,
                                          double& lsum, int lane, int kin, double& pa,
                                          double& pb) {
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const double s = base + lv[jj];
    const double r = rcp_f64(s);
    if (LOGS && lane + 32 * jj < kin) lsum += log(s);
    acc[jj] += r;
    if (jj & 1)
      pb = jj == 1 ? r : pb + r;
    else
      pa = jj == 0 ? r : pa + r;
  }
  if (J == 1) pb = 0.0;
}

template <int J, int NOUT, bool LOGS>
__device__ void grid_pass_fast(const GridDesc& gd, const double* slam, double* sg, double* pw,
                               int64_t gwarp, int64_t nwarps, double* accw = nullptr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int kin = gd.k[gd.inner];
  const int oin = gd.off[gd.inner];
  // slots past the inner axis hold a huge λ: their 1/s ~ 1e-300 is negligible against any
  // marginal, so the point loop runs without per-slot predicates (the Σ log s pass, LOGS,
  // keeps them)
  double lv[J], acc[J];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const int m = lane + 32 * jj;
    lv[jj] = (m < kin) ? slam[oin + m] : 1e300;
    acc[jj] = 0.0;
  }
  double lsum = 0.0;
  if (NOUT == 0) {  // one axis: a single row
    if (gwarp == 0) {
      double pa, pb;
      point_row<J, LOGS>(lv, acc, 0.0, lsum, lane, kin, pa, pb);
    }
  } else {
    const int af = gd.outer_axes[NOUT - 1];  // fastest outer axis
    const int as = NOUT == 2 ? gd.outer_axes[0] : af;
    const int kf = gd.k[af], ks = NOUT == 2 ? gd.k[as] : 1;
    const int off_s = gd.off[as];
    const double* lf = slam + gd.off[af];
    const double* ls = slam + off_s;
    double* bins = pw + wid * kf;
    // balanced contiguous row ranges (every warp of the grid busy; a range's segment tails
    // of < 4 rows take the one-row path)
    const int64_t r0 = gwarp * gd.rows / nwarps;
    const int64_t r1 = (gwarp + 1) * gd.rows / nwarps;
    int fi = (int)(r0 % kf);
    int si = NOUT == 2 ? (int)((r0 / kf) % ks) : 0;
    for (int64_t row = r0; row < r1;) {
      const int seg = (int)min(r1 - row, (int64_t)(kf - fi));
      const double bs = NOUT == 2 ? ls[si] : 0.0;
      double sacc = 0.0;
      int q0 = 0;
      for (; q0 + 4 <= seg; q0 += 4) {
        double p[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double pa, pb;
          const double base = NOUT == 2 ? lf[fi + q0 + q] + bs : lf[fi + q0 + q];
          point_row<J, LOGS>(lv, acc, base, lsum, lane, kin, pa, pb);
          p[q] = pa + pb;
        }
        if (NOUT == 2) sacc += (p[0] + p[1]) + (p[2] + p[3]);
        const double tot = reduce4(p, lane);
        if ((lane & 7) == 0) {
          double* bq = bins + fi + q0 + (lane >> 3);  // four distinct bins (no wrap)
          GGM_DCHECK(fi + q0 + (lane >> 3) < kf);
          *bq += tot;
        }
        __syncwarp();
      }
      GGM_DCHECK(seg >= 1 && fi + seg <= kf);
      for (; q0 < seg; ++q0) {  // segment tail: one row at a time
        double pa, pb;
        const double base = NOUT == 2 ? lf[fi + q0] + bs : lf[fi + q0];
        point_row<J, LOGS>(lv, acc, base, lsum, lane, kin, pa, pb);
        const double pr = pa + pb;
        if (NOUT == 2) sacc += pr;
        const double tot = warp_sum(pr);
        if (lane == 0) bins[fi + q0] += tot;
        __syncwarp();
      }
      if (NOUT == 2) {  // flush the slow axis once per segment
        const double t = warp_sum(sacc);
        if (lane == 0) atomicAdd(&sg[off_s + si], t);
      }
      row += seg;
      fi += seg;
      if (fi == kf) {
        fi = 0;
        if (NOUT == 2 && ++si == ks) si = 0;
      }
    }
  }
  if (NOUT >= 1 && accw != nullptr) {  // per-warp rows, folded below (no fp64 smem CAS loops)
#pragma unroll
    for (int jj = 0; jj < J; ++jj) accw[wid * 32 * J + lane + 32 * jj] = acc[jj];
  } else {
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      const int m = lane + 32 * jj;
      if (m < kin) atomicAdd(&sg[oin + m], acc[jj]);
    }
  }
  if (LOGS) {
    lsum = warp_sum(lsum);
    if (lane == 0) atomicAdd(&sg[gd.total], lsum);
  }
  if (NOUT >= 1) {  // fold the private bins into the block partials, clear them
    const int af = gd.outer_axes[NOUT - 1];
    const int kf = gd.k[af];
    __syncthreads();
    for (int f = threadIdx.x; f < kf; f += blockDim.x) {
      double t = 0.0;
      for (int w = 0; w < kWarps; ++w) {
        t += pw[w * kf + f];
        pw[w * kf + f] = 0.0;
      }
      sg[gd.off[af] + f] += t;
    }
    if (accw != nullptr)
      for (int m = threadIdx.x; m < kin; m += blockDim.x) {
        double t = 0.0;
        for (int w = 0; w < kWarps; ++w) t += accw[w * 32 * J + m];
        sg[oin + m] += t;
      }
    __syncthreads();
  }
}

// Generic pass (any number of outer axes, or a fastest outer axis above kMaxFastBins): per
// row a warp-shuffle row sum and one shared-memory atomic per outer axis.
template <int J, bool LOGS>
__device__ void grid_pass_generic(const GridDesc& gd, const double* slam, double* sg,
                                  int64_t gwarp, int64_t nwarps) {
  const int lane = threadIdx.x & 31;
  const int kin = gd.k[gd.inner];
  const int oin = gd.off[gd.inner];
  const int nout = gd.n_outer;
  int idx[kMaxAxes];
  double lv[J], acc[J];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const int m = lane + 32 * jj;
    lv[jj] = (m < kin) ? slam[oin + m] : 1.0;
    acc[jj] = 0.0;
  }
  double lsum = 0.0;
  const int64_t per = (gd.rows + nwarps - 1) / nwarps;
  const int64_t r0 = gwarp * per;
  const int64_t r1 = min(gd.rows, r0 + per);
  for (int a = 0; a < nout; ++a) idx[a] = (int)((r0 / gd.outer_stride[a]) % gd.k[gd.outer_axes[a]]);
  for (int64_t row = r0; row < r1; ++row) {
    double base = 0.0;
    for (int a = 0; a < nout; ++a) base += slam[gd.off[gd.outer_axes[a]] + idx[a]];
    double rsum = 0.0;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      const int m = lane + 32 * jj;
      if (m < kin) {
        const double s = base + lv[jj];
        const double r = rcp_f64(s);
        if (LOGS) lsum += log(s);
        rsum += r;
        acc[jj] += r;
      }
    }
    if (nout > 0) {
      rsum = warp_sum(rsum);
      for (int a = 0; a < nout; ++a)
        if (lane == a) atomicAdd(&sg[gd.off[gd.outer_axes[a]] + idx[a]], rsum);
      for (int a = nout - 1; a >= 0; --a) {
        if (++idx[a] < gd.k[gd.outer_axes[a]]) break;
        idx[a] = 0;
      }
    }
  }
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const int m = lane + 32 * jj;
    if (m < kin) atomicAdd(&sg[oin + m], acc[jj]);
  }
  if (LOGS) {
    lsum = warp_sum(lsum);
    if (lane == 0) atomicAdd(&sg[gd.total], lsum);
  }
}

__host__ __device__ inline bool fast_path(const GridDesc& gd) {
  return gd.n_outer <= 2 &&
         (gd.n_outer == 0 || gd.k[gd.outer_axes[gd.n_outer - 1]] <= kMaxFastBins);
}
__host__ __device__ inline int fast_bins(const GridDesc& gd) {
  return (gd.n_outer >= 1 && fast_path(gd)) ? gd.k[gd.outer_axes[gd.n_outer - 1]] : 0;
}

template <int J, bool LOGS>
__device__ __forceinline__ void grid_pass(const GridDesc& gd, const double* slam, double* sg,
                                          double* pw, int64_t gwarp, int64_t nwarps,
                                          double* accw = nullptr) {
  if (!fast_path(gd) || pw == nullptr) {
    grid_pass_generic<J, LOGS>(gd, slam, sg, gwarp, nwarps);
    return;
  }
  switch (gd.n_outer) {
    case 0: grid_pass_fast<J, 0, LOGS>(gd, slam, sg, pw, gwarp, nwarps); break;
    case 1: grid_pass_fast<J, 1, LOGS>(gd, slam, sg, pw, gwarp, nwarps, accw); break;
    default: grid_pass_fast<J, 2, LOGS>(gd, slam, sg, pw, gwarp, nwarps, accw); break;
  }
}

constexpr int kMaxMods = 8;  // modalities of a multi-modal solve

enum Scheme { kSchemeMM = 0, kSchemeSquarem = 1, kSchemeGD = 2 };

struct SolveParams {
  GridDesc gd[kMaxMods];  // one per modality; offsets index the global concatenation
  int M;                  // modalities
  int T;                  // Σk over all axes
  const double* E;        // spectrum of the update and the residual (G⊥-projected in the
                          // interior regime, reading T; as given in the barrier regime / GD)
  double floor;           // barrier ε (> 0: barrier regime, λ >= floor); 0: interior
  double gd_eps;          // method 2: grid-minimum feasibility ε (reading Q3)
  int scheme;
  int pw_stride;          // doubles of private bins per block (kWarps x max k_fast)
  int accw;               // 1: kWarps x 32 J doubles after the bins hold per-warp inner marginals
  int sE_off;             // >= 0: E cached at this offset (doubles) of dynamic shared memory
  double* lam_out;        // λ at exit, Σk
  double* g;              // marginals at lam_out, Σk
  double* gacc;           // [3][Σk + 1] rotating global accumulators of the block partials
  int* status;            // [0] iterations, [1] converged flag
  double* res_out;        // stationarity of lam_out
  double tol;
  int max_iter;
  int red_mode;           // cross-block reduction: 0 = fp64 atomics into gacc; 1 = partial
                          // rows in part[], column sums by all blocks into gred, 2 barriers
  double* part;           // [gridDim][Σk + 1]
  double* gred;           // [Σk + 1]
};

// Block-wide reductions (every block runs them in the same order on the same data, so the
// results are bitwise identical across blocks).  red: kWarps doubles of shared scratch.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) t += red[w];
  return t;
}
__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = red[0];
#pragma unroll
  for (int w = 1; w < kWarps; ++w) t = fmax(t, red[w]);
  return t;
}
__device__ __forceinline__ double block_min(double v, double* red) {
  return -block_max(-v, red);
}

// KKT residual at λ with marginals g (reading Q4, Lemma 6's box): |E − g| off the floor,
// max(0, g − E) on it; the caller divides by max E.
__device__ __forceinline__ double kkt_term(double lam, double g, double e, double floor) {
  return (floor > 0.0 && lam <= floor * (1.0 + 1e-9)) ? fmax(0.0, g - e) : fabs(e - g);
}

// Whole solve in one cooperative kernel.  Shared memory: sg[T+1] (partials, then the reduced
// marginals and Σ log s), slam[T] (the point the next pass evaluates), th0[T], th1[T]
// (SQUAREM iterates in log space; GD: the accepted λ and its marginals), private bins.
template <int J, bool LOGS>
__global__ void __launch_bounds__(kThreads, J <= 7 ? 2 * GGM_SOLVE_MINB : GGM_SOLVE_MINB) solve_kernel(const SolveParams p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dsm[];
  const int T = p.T;
  double* sg = dsm;
  double* slam = sg + T + 1;
  double* th0 = slam + T;
  double* th1 = th0 + T;
  double* pw = p.pw_stride > 0 ? th1 + T : nullptr;  // private bins (fast pass) if allotted
  double* accw = pw != nullptr && p.accw ? pw + p.pw_stride : nullptr;  // per-warp inner rows
  __shared__ double s_red[kWarps];
  const int tid = threadIdx.x;
  // E (read by every update) cached in shared memory when the host allotted it
  const double* E = p.E;
  if (p.sE_off >= 0) {
    double* se = dsm + p.sE_off;
    for (int i = tid; i < T; i += blockDim.x) se[i] = p.E[i];
    __syncthreads();
    E = se;
  }
  for (int i = tid; i < T; i += blockDim.x) {
    const double l0 = fmax(1.0 / E[i], p.floor);  // Alg. 1 line 5
    slam[i] = l0;
    if (p.scheme != kSchemeMM) th0[i] = log(l0);
  }
  for (int i = tid; i < p.pw_stride; i += blockDim.x) pw[i] = 0.0;
  double emax = 0.0;
  for (int i = tid; i < T; i += blockDim.x) emax = fmax(emax, E[i]);
  emax = block_max(emax, s_red);
  const int64_t gw = (int64_t)blockIdx.x * kWarps + (tid >> 5);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  const bool single = gridDim.x == 1;
  const int T1 = T + 1;
  int it = 0, pass = 0, phase = 0;
  bool done = false, stalled = false;
  double res = 0.0, r1 = 0.0;
  double f_acc = 0.0, mu = 1.0;  // GD: NLL of the accepted λ, step size (Alg. 1 line 6)
  double* out_lam = slam;         // where the result lives at exit
  double* out_g = sg;
  for (;; ++pass) {
    // ---------------------------------------------------------------- grid pass at slam
    for (int i = tid; i < T1; i += blockDim.x) sg[i] = 0.0;
    if (blockIdx.x == 0 && !single && p.red_mode != 2)
      for (int i = tid; i < T1; i += blockDim.x) p.gacc[(size_t)((pass + 1) % 3) * T1 + i] = 0.0;
    if (!single && p.red_mode == 2) {  // zero the next pass's group accumulators (all blocks)
      double* nb = p.part + (size_t)((pass + 1) % 3) * kRedGroups * T1;
      for (int64_t e = (int64_t)blockIdx.x * blockDim.x + tid; e < (int64_t)kRedGroups * T1;
           e += (int64_t)gridDim.x * blockDim.x)
        nb[e] = 0.0;
    }
    __syncthreads();
    // Σ_γ of the modalities' marginals (Thm 2): each pass adds into the same sg
    for (int m = 0; m < p.M; ++m) grid_pass<J, LOGS>(p.gd[m], slam, sg, pw, gw, nw, accw);
    __syncthreads();
    if (!single && p.red_mode == 2) {
      // grouped fp64 atomics: block b adds into accumulator copy b mod kRedGroups (1/kRedGroups
      // of the same-address contention of one accumulator), every block sums the copies in a
      // fixed order after the barrier
      double* accb = p.part + (size_t)(pass % 3) * kRedGroups * T1;
      double* acc = accb + (size_t)(blockIdx.x % kRedGroups) * T1;
      for (int i = tid; i < T1; i += blockDim.x) {
        const double v = sg[i];
        if (v != 0.0) atomicAdd(&acc[i], v);
      }
      grid.sync();
      for (int i = tid; i < T1; i += blockDim.x) {
        double t = 0.0;
#pragma unroll
        for (int gq = 0; gq < kRedGroups; ++gq) t += __ldcg(&accb[(size_t)gq * T1 + i]);
        sg[i] = t;
      }
      __syncthreads();
    } else if (!single && p.red_mode == 0) {
      double* acc = p.gacc + (size_t)(pass % 3) * T1;
      for (int i = tid; i < T1; i += blockDim.x) {
        const double v = sg[i];
        if (v != 0.0) atomicAdd(&acc[i], v);  // e.g. the slow axis: a block touches few entries
      }
      grid.sync();
      for (int i = tid; i < T1; i += blockDim.x) sg[i] = __ldcg(&acc[i]);
      __syncthreads();
    } else if (!single) {
      // block partials as columns of part[] (entry-major: part[i][block]), one barrier,
      // entry i summed in a fixed order by one warp of block i mod gridDim (coalesced), a
      // second barrier, every block reads the sums
      const int nb = gridDim.x;
      for (int i = tid; i < T1; i += blockDim.x) __stcg(&p.part[(size_t)i * nb + blockIdx.x], sg[i]);
      grid.sync();
      const int lane = tid & 31, w = tid >> 5;
      for (int c = blockIdx.x + w * nb; c < T1; c += kWarps * nb) {
        double t = 0.0;
        for (int b = lane; b < nb; b += 32) t += __ldcg(&p.part[(size_t)c * nb + b]);
        t = warp_sum(t);
        if (lane == 0) __stcg(&p.gred[c], t);
      }
      grid.sync();
      for (int i = tid; i < T1; i += blockDim.x) sg[i] = __ldcg(&p.gred[i]);
      __syncthreads();
    }
    // ---------------------------------------------------------------- update
    if (p.scheme == kSchemeGD) {
      // Algorithm 1 as printed (readings Q1-Q3): the pass evaluated the candidate Λ' (or λ0)
      double lin = 0.0;
      for (int i = tid; i < T; i += blockDim.x) lin += E[i] * slam[i];
      lin = block_sum(lin, s_red);
      const double f = 0.5 * lin - 0.5 * sg[T];
      const bool accept = pass == 0 || f <= f_acc;
      if (accept) {  // Λ ← Λ' (lines 16-17): keep λ and its marginals
        for (int i = tid; i < T; i += blockDim.x) {
          th0[i] = slam[i];
          th1[i] = sg[i];
        }
        f_acc = f;
        if (pass > 0) ++it;
      } else {
        mu *= 0.5;  // NLL did not decrease (reading Q2)
      }
      __syncthreads();
      out_lam = th0;
      out_g = th1;
      double mr = 0.0;
      for (int i = tid; i < T; i += blockDim.x) mr = fmax(mr, fabs(E[i] - th1[i]));
      res = block_max(mr, s_red) / emax;
      if (res <= p.tol) {
        done = true;
        break;
      }
      if (it >= p.max_iter) break;
      // next candidate: Λ' = Λ − μ·½(E − g), μ halved while Σ_l min Λ'_l < ε (line 11)
      for (;;) {
        double gmin = INFINITY;
        for (int m = 0; m < p.M; ++m) {
          const GridDesc& gd = p.gd[m];
          double smin = 0.0;
          for (int a = 0; a < gd.L; ++a) {
            double mn = INFINITY;
            for (int i = tid; i < gd.k[a]; i += blockDim.x) {
              const int c = gd.off[a] + i;
              mn = fmin(mn, th0[c] - mu * 0.5 * (E[c] - th1[c]));
            }
            smin += block_min(mn, s_red);
          }
          gmin = fmin(gmin, smin);
        }
        if (gmin >= p.gd_eps) break;
        mu *= 0.5;
        if (mu < 1e-300) break;
      }
      if (mu < 1e-300) {
        stalled = true;
        break;
      }
      for (int i = tid; i < T; i += blockDim.x) slam[i] = th0[i] - mu * 0.5 * (E[i] - th1[i]);
      __syncthreads();
      continue;
    }
    double mr = 0.0;
    #pragma unroll 2
    for (int i = tid; i < T; i += blockDim.x) mr = fmax(mr, kkt_term(slam[i], sg[i], E[i], p.floor));
    res = block_max(mr, s_red) / emax;
    if (res <= p.tol) {
      done = true;
      break;
    }
    if (it == p.max_iter) break;
    ++it;
    if (p.scheme == kSchemeMM) {
      // majorise-minimise step, clamped on the box (a separable majoriser minimised per
      // coordinate)
      #pragma unroll 2
      for (int i = tid; i < T; i += blockDim.x) slam[i] = fmax(p.floor, slam[i] * sg[i] / E[i]);
      __syncthreads();
      continue;
    }
    // SQUAREM (interior regime, floor = 0), log space θ = log λ, map F(θ) = θ + log(g/E)
    if (phase == 0) {  // slam = exp(θ0): θ1 = F(θ0)
      #pragma unroll 2
      for (int i = tid; i < T; i += blockDim.x) {
        const double t1 = th0[i] + log(sg[i] / E[i]);
        th1[i] = t1;
        slam[i] = exp(t1);
      }
      phase = 1;
    } else if (phase == 1) {  // slam = exp(θ1): θ2 = F(θ1), extrapolate
      r1 = res;
      double nr = 0.0, nv = 0.0;
      #pragma unroll 2
      for (int i = tid; i < T; i += blockDim.x) {
        const double t0 = th0[i], t1 = th1[i];
        const double t2 = t1 + log(sg[i] / E[i]);
        sg[i] = t2;
        const double rr = t1 - t0, v = t2 - 2.0 * t1 + t0;
        nr += rr * rr;
        nv += v * v;
      }
      nr = block_sum(nr, s_red);
      nv = block_sum(nv, s_red);
      double al = nv > 0.0 ? -sqrt(nr / nv) : -1.0;
      al = fmin(-1.0, fmax(al, -1e3));
      for (int i = tid; i < T; i += blockDim.x) {
        const double t0 = th0[i], t1 = th1[i], t2 = sg[i];
        const double tp = t0 - 2.0 * al * (t1 - t0) + al * al * (t2 - 2.0 * t1 + t0);
        th0[i] = t2;  // fallback: the plain iterate θ2
        th1[i] = tp;
        slam[i] = exp(tp);
      }
      phase = 2;
    } else {  // slam = exp(θ'): stabilising step θ0 = F(θ') if no worse than θ1, else θ2
      const bool take = res <= r1;
      #pragma unroll 2
      for (int i = tid; i < T; i += blockDim.x) {
        if (take) th0[i] = th1[i] + log(sg[i] / E[i]);
        slam[i] = exp(th0[i]);
      }
      phase = 0;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0) {
    for (int i = tid; i < T; i += blockDim.x) {
      p.lam_out[i] = out_lam[i];
      p.g[i] = out_g[i];
    }
    if (tid == 0) {
      p.status[0] = it;
      p.status[1] = done ? 1 : 0;
      p.status[2] = stalled ? 1 : 0;
      p.status[3] = pass + 1;
      *p.res_out = res;
    }
  }
}

// Stand-alone single pass (ggm_grid_marginals): partials into [Σk][grid].
template <int J>
__global__ void __launch_bounds__(kThreads, 1) marginal_pass_kernel(GridDesc gd, const double* lam,
                                                                     double* partial) {
  extern __shared__ double dsm[];
  double* sg = dsm;
  double* slam = sg + gd.total + 1;
  double* pw = slam + gd.total;
  for (int i = threadIdx.x; i <= gd.total; i += blockDim.x) sg[i] = 0.0;
  for (int i = threadIdx.x; i < gd.total; i += blockDim.x) slam[i] = lam[i];
  for (int i = threadIdx.x; i < kWarps * fast_bins(gd); i += blockDim.x) pw[i] = 0.0;
  __syncthreads();
  grid_pass<J, false>(gd, slam, sg, pw, (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5),
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
  sum = warp_sum(sum);
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
  acc = warp_sum(acc);
  if (lane == 0) atomicAdd(logsum, acc);
}

__global__ void check_E(const double* E, int total, int* bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const double e = E[i];
    if (!(e > 0.0) || !isfinite(e)) atomicOr(bad, 1);
  }
}

static ggm_status make_desc(int L, const int* k, GridDesc* gd) {
  if (L < 1 || L > kMaxAxes) return fail(GGM_ERR_INVALID_ARGUMENT, "L=%d not in [1,%d]", L, kMaxAxes);
  if (!k) return fail(GGM_ERR_INVALID_ARGUMENT, "k is NULL");
  memset(gd, 0, sizeof(*gd));
  gd->L = L;
  gd->off[0] = 0;
  int inner = 0;
  double prod = 1.0;
  static const bool inner_min = [] {  // A/B hook: smallest axis inner (tools/solve_probe.py)
    const char* e = std::getenv("GGM_SOLVE_INNER");
    return e && e[0] == 'm' && e[1] == 'i';
  }();
  for (int a = 0; a < L; ++a) {
    if (k[a] < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "k[%d]=%d < 1", a, k[a]);
    gd->k[a] = k[a];
    gd->off[a + 1] = gd->off[a] + k[a];
    if (inner_min ? k[a] < k[inner] : k[a] > k[inner]) inner = a;
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

// points per lane of the inner axis, rounded up to an instantiated size
static int pick_J(int kin) {
  const int j = (kin + 31) / 32;
  static const int sizes[] = {1, 2, 4, 7, 10, 13, 16, 32};
  for (int s : sizes)
    if (j <= s) return s;
  return 32;
}

#define GGM_FOR_J(X) X(1) X(2) X(4) X(7) X(10) X(13) X(16) X(32)

static size_t pass_smem(const GridDesc& gd) {
  return ((size_t)gd.total * 2 + 1 + (size_t)kWarps * fast_bins(gd)) * sizeof(double) + 16;
}

static int grid_blocks(const GridDesc& gd) {
  const int64_t warps_needed = std::max<int64_t>(1, gd.rows);
  const int64_t blocks = (warps_needed + kWarps - 1) / kWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, num_sms()));
}

// Blocks for the cooperative solve: enough warps that each owns >= ~8 outer rows (a grid
// barrier costs microseconds; small grids run in one block).
static int solve_blocks(double pts) {
  const int64_t want = (int64_t)std::ceil(pts / (kWarps * 8.0 * 32.0 * 16.0));
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, 2 * num_sms()));
}

template <int J>
static cudaError_t launch_pass_j(const GridDesc& gd, const double* lam, double* partial, int nblk,
                                 size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(marginal_pass_kernel<J>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  marginal_pass_kernel<J><<<nblk, kThreads, smem, s>>>(gd, lam, partial);
  return cudaGetLastError();
}

static cudaError_t launch_pass(const GridDesc& gd, const double* lam, double* partial, int nblk,
                               cudaStream_t s) {
  const size_t smem = pass_smem(gd);
  switch (pick_J(gd.k[gd.inner])) {
#define GGM_CASE(j) \
  case j: return launch_pass_j<j>(gd, lam, partial, nblk, smem, s);
    GGM_FOR_J(GGM_CASE)
#undef GGM_CASE
  }
  return cudaErrorInvalidValue;
}

template <int J, bool LOGS>
static cudaError_t launch_solve_j(const SolveParams& sp, int nblk, size_t smem, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(solve_kernel<J, LOGS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<J, LOGS>, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  nblk = std::min(nblk, std::min(per_sm, 2) * num_sms());  // co-resident (part[] has 2 x sms rows)
  void* args[] = {const_cast<SolveParams*>(&sp)};
  return cudaLaunchCooperativeKernel((void*)solve_kernel<J, LOGS>, dim3(nblk), dim3(kThreads), args,
                                     smem, s);
}

static cudaError_t launch_solve(const SolveParams& sp, int J, int nblk, size_t smem,
                                cudaStream_t s) {
  const bool logs = sp.scheme == kSchemeGD;
  switch (J) {
#define GGM_CASE(j)                                                                   \
  case j:                                                                             \
    return logs ? launch_solve_j<j, true>(sp, nblk, smem, s)                          \
                : launch_solve_j<j, false>(sp, nblk, smem, s);
    GGM_FOR_J(GGM_CASE)
#undef GGM_CASE
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ host-side gauge algebra
// Axis space: one coordinate per axis.  The modalities' incidence rows span G^⊥ in axis
// space; G_F (the gauge freedom with the axes outside `free_axes` pinned) is the null space
// of the incidence rows plus the unit rows of the pinned axes.
using Vec = std::vector<double>;

static std::vector<Vec> null_basis(int nax, const std::vector<Vec>& rows) {
  std::vector<Vec> R;  // orthonormalised rows
  for (const Vec& r0 : rows) {
    Vec v = r0;
    for (int pass = 0; pass < 2; ++pass)
      for (const Vec& r : R) {
        double d = 0.0;
        for (int a = 0; a < nax; ++a) d += r[a] * v[a];
        for (int a = 0; a < nax; ++a) v[a] -= d * r[a];
      }
    double nv = 0.0;
    for (double x : v) nv += x * x;
    if (nv > 1e-20) {
      nv = std::sqrt(nv);
      for (double& x : v) x /= nv;
      R.push_back(v);
    }
  }
  std::vector<Vec> N;
  for (int e = 0; e < nax; ++e) {
    Vec v(nax, 0.0);
    v[e] = 1.0;
    for (int pass = 0; pass < 2; ++pass) {
      for (const Vec& r : R) {
        double d = 0.0;
        for (int a = 0; a < nax; ++a) d += r[a] * v[a];
        for (int a = 0; a < nax; ++a) v[a] -= d * r[a];
      }
      for (const Vec& r : N) {
        double d = 0.0;
        for (int a = 0; a < nax; ++a) d += r[a] * v[a];
        for (int a = 0; a < nax; ++a) v[a] -= d * r[a];
      }
    }
    double nv = 0.0;
    for (double x : v) nv += x * x;
    if (nv > 1e-12) {
      nv = std::sqrt(nv);
      for (double& x : v) x /= nv;
      N.push_back(v);
    }
  }
  return N;
}

struct ModelAxes {
  int nax;
  std::vector<int> k, off;             // per global axis
  std::vector<std::vector<int>> mods;  // axes of each modality
  std::vector<Vec> incidence() const {
    std::vector<Vec> rows;
    for (const auto& m : mods) {
      Vec r(nax, 0.0);
      for (int a : m) r[a] = 1.0;
      rows.push_back(r);
    }
    return rows;
  }
  std::vector<Vec> gauge_free(const std::vector<int>& pinned) const {
    std::vector<Vec> rows = incidence();
    for (int a : pinned) {
      Vec r(nax, 0.0);
      r[a] = 1.0;
      rows.push_back(r);
    }
    return null_basis(nax, rows);
  }
  // per-axis shifts c that remove from x (Σk coordinates, per-axis sums D) its component in
  // the lift of span N (orthogonal projection in the Σk space: weights k_l in axis space)
  Vec lifted_shift(const std::vector<Vec>& N, const Vec& D) const {
    std::vector<Vec> U;  // k-weighted orthonormalisation of N
    for (const Vec& n0 : N) {
      Vec v = n0;
      for (int pass = 0; pass < 2; ++pass)
        for (const Vec& u : U) {
          double d = 0.0;
          for (int a = 0; a < nax; ++a) d += k[a] * u[a] * v[a];
          for (int a = 0; a < nax; ++a) v[a] -= d * u[a];
        }
      double nv = 0.0;
      for (int a = 0; a < nax; ++a) nv += k[a] * v[a] * v[a];
      if (nv > 1e-20) {
        nv = std::sqrt(nv);
        for (double& x : v) x /= nv;
        U.push_back(v);
      }
    }
    Vec c(nax, 0.0);
    for (const Vec& u : U) {
      double d = 0.0;
      for (int a = 0; a < nax; ++a) d += u[a] * D[a];
      for (int a = 0; a < nax; ++a) c[a] += d * u[a];
    }
    return c;
  }
};

// Reading T: relative gauge component of the per-axis traces (single modality: max |tr_l −
// mean| / mean; several: |P_G tr|_max / mean tr).
static double trace_inconsistency(const ModelAxes& ax, const Vec& hE) {
  Vec tr(ax.nax, 0.0);
  double mean = 0.0;
  for (int a = 0; a < ax.nax; ++a) {
    for (int i = ax.off[a]; i < ax.off[a + 1]; ++i) tr[a] += hE[i];
    mean += tr[a] / ax.nax;
  }
  if (!(mean > 0.0)) return 0.0;
  const std::vector<Vec> N = ax.gauge_free({});
  double ti = 0.0;
  for (int a = 0; a < ax.nax; ++a) {
    double pa = 0.0;
    for (const Vec& n : N) {
      double d = 0.0;
      for (int b = 0; b < ax.nax; ++b) d += n[b] * tr[b];
      pa += d * n[a];
    }
    ti = std::max(ti, std::fabs(pa));
  }
  return ti / mean;
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// Common driver of ggm_solve_eigvals / ggm_solve_eigvals_multi.
static ggm_status solve_common(SolveParams sp, const ModelAxes& ax, const double* E,
                               const ggm_solve_opts& o, double* lambda, ggm_solve_info* info,
                               cudaStream_t s) {
  const int T = sp.T;
  if (!(o.tol > 0.0) || o.max_iter < 0 || !(o.eps_scale >= 0.0) || !(o.trace_tol >= 0.0))
    return fail(GGM_ERR_INVALID_ARGUMENT, "invalid solve options");
  if (o.method < 0 || o.method > 2) return fail(GGM_ERR_INVALID_ARGUMENT, "method=%d", o.method);
  if (o.gauge != 0 && o.gauge != 1) return fail(GGM_ERR_INVALID_ARGUMENT, "gauge=%d", o.gauge);
  // scratch: lam_res, g, Eu, gacc[3][T+1], scalars, status, part[sms][T+1], gred[T+1]
  const size_t bytes = sizeof(double) * (3 * (size_t)T + 3 * ((size_t)T + 1) + 8) + 64 +
                       sizeof(double) * (2 * (size_t)num_sms() + 1) * ((size_t)T + 1) + 256;
  DevBuf buf;
  GGM_CUDA_TRY(cudaMallocAsync(&buf.p, bytes, s));
  double* lam_res = static_cast<double*>(buf.p);
  double* g = lam_res + T;
  double* Eu = g + T;
  double* gacc = Eu + T;
  double* scal = gacc + 3 * ((size_t)T + 1);  // [1] logsum, [2] residual
  int* istat = reinterpret_cast<int*>(scal + 4);  // [0] it, [1] converged, [2] stalled, [3] passes, [6] bad
  sp.part = reinterpret_cast<double*>(reinterpret_cast<char*>(buf.p) +
                                      align_up(sizeof(double) * (3 * (size_t)T + 3 * ((size_t)T + 1) + 8) + 64, 256));
  sp.gred = sp.part + 2 * (size_t)num_sms() * ((size_t)T + 1);
  {
    const char* e = std::getenv("GGM_SOLVE_RED");  // A/B hook (tools/solve_probe.py)
    sp.red_mode = e ? std::atoi(e) : 2;
  }
  GGM_CUDA_TRY(cudaMemsetAsync(gacc, 0, sizeof(double) * (3 * ((size_t)T + 1) + 8) + 64, s));
  if (sp.red_mode == 2)  // the first pass's group accumulators (3 x kRedGroups copies fit part[])
    GGM_CUDA_TRY(cudaMemsetAsync(sp.part, 0, sizeof(double) * 3 * kRedGroups * ((size_t)T + 1), s));
  check_E<<<4, 256, 0, s>>>(E, T, istat + 6);
  GGM_CUDA_TRY(cudaGetLastError());
  int hbad = 0;
  Vec hE(T);
  GGM_CUDA_TRY(cudaMemcpyAsync(&hbad, istat + 6, sizeof(int), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(hE.data(), E, sizeof(double) * T, cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad) return fail(GGM_ERR_DOMAIN, "E must be finite and > 0 (Thm 4, P:742)");

  // reading T: interior (projected spectrum) or barrier regime
  double emin_inv = 0.0;
  for (int i = 0; i < T; ++i) emin_inv = std::max(emin_inv, 1.0 / hE[i]);
  const double eps = o.eps_scale * emin_inv;
  const double ti = trace_inconsistency(ax, hE);
  const bool barrier = o.method != 2 && ti > o.trace_tol;
  Vec hEu = hE;
  if (!barrier && o.method != 2) {  // E_eff = P_{G⊥} E
    Vec tr(ax.nax, 0.0);
    for (int a = 0; a < ax.nax; ++a)
      for (int i = ax.off[a]; i < ax.off[a + 1]; ++i) tr[a] += hE[i];
    const Vec c = ax.lifted_shift(ax.gauge_free({}), tr);
    for (int a = 0; a < ax.nax; ++a)
      for (int i = ax.off[a]; i < ax.off[a + 1]; ++i) hEu[i] -= c[a];
    for (int i = 0; i < T; ++i)
      if (!(hEu[i] > 0.0)) return fail(GGM_ERR_DOMAIN, "projected spectrum not positive");
  }
  GGM_CUDA_TRY(cudaMemcpyAsync(Eu, hEu.data(), sizeof(double) * T, cudaMemcpyHostToDevice, s));

  int J = 1, kfmax = 0;
  double pts = 0.0;
  for (int m = 0; m < sp.M; ++m) {
    J = std::max(J, pick_J(sp.gd[m].k[sp.gd[m].inner]));
    kfmax = std::max(kfmax, fast_bins(sp.gd[m]));
    pts += (double)sp.gd[m].rows * sp.gd[m].k[sp.gd[m].inner];
  }
  // shared memory: sg[T+1], slam[T], th0[T], th1[T], private bins; if that does not fit,
  // the plain MM step with sg and slam only and the generic pass
  // per-warp inner-marginal rows (kWarps x 32 J doubles) in place of fp64 shared atomics,
  // which compile to CAS loops (ATOMS.CAST.SPIN.64) contended by the block's 16 warps:
  // C3 kernel 1.004 -> 0.970 ms (profiles/r02_logs/r02end_ab_accw.log); -DGGM_SOLVE_NOACCW
  // restores the atomics
#ifndef GGM_SOLVE_NOACCW
  const size_t accw_d = (size_t)kWarps * 32 * J;
#else
  const size_t accw_d = 0;
#endif
  const size_t smem_base = ((size_t)4 * T + 1 + (size_t)kWarps * kfmax) * sizeof(double) + 16;
  const bool accw_fits = accw_d > 0 && smem_base + accw_d * sizeof(double) <= 200 * 1024;
  const size_t smem_pw = smem_base + (accw_fits ? accw_d * sizeof(double) : 0);
  const bool fits = smem_pw <= 200 * 1024;
  sp.pw_stride = fits ? kWarps * kfmax : 0;
  sp.accw = fits && accw_fits ? 1 : 0;
  // E in shared memory after everything else, when it fits
  const size_t se_at = fits ? smem_pw : ((size_t)2 * T + 1) * sizeof(double) + 16;
  const bool se_fits = se_at + (size_t)T * sizeof(double) <= 200 * 1024;
  sp.sE_off = se_fits ? (int)(align_up(se_at, 16) / sizeof(double)) : -1;
  const size_t smem_full = se_fits ? align_up(se_at, 16) + (size_t)T * sizeof(double) : smem_pw;
  const size_t smem_launch = (fits || se_fits) ? smem_full : ((size_t)2 * T + 1) * sizeof(double) + 16;
  if (!fits && o.method == 2)
    return fail(GGM_ERR_UNSUPPORTED, "method 2: sum(k)=%d too large for the solve kernel", T);
  sp.E = o.method == 2 ? E : Eu;
  sp.floor = barrier ? eps : 0.0;
  sp.gd_eps = eps;
  sp.scheme = o.method == 2 ? kSchemeGD : (o.method == 1 || barrier || !fits) ? kSchemeMM : kSchemeSquarem;
  sp.lam_out = lam_res;
  sp.g = g;
  sp.gacc = gacc;
  sp.status = istat;
  sp.res_out = scal + 2;
  sp.tol = o.tol;
  sp.max_iter = o.max_iter;
  if (smem_launch > 227 * 1024)
    return fail(GGM_ERR_UNSUPPORTED, "sum(k)=%d too large for the solve kernel", T);
  const int nblk = solve_blocks(pts);
  // CUDA events around the solve kernel(s) on the launch stream (info->kernel_ms)
  cudaEvent_t ev[2];
  GGM_CUDA_TRY(cudaEventCreate(&ev[0]));
  GGM_CUDA_TRY(cudaEventCreate(&ev[1]));
  GGM_CUDA_TRY(cudaEventRecord(ev[0], s));
  cudaError_t ce = launch_solve(sp, J, nblk, smem_launch, s);
  if (ce != cudaSuccess) return fail(GGM_ERR_CUDA, "solve_kernel launch: %s", cudaGetErrorString(ce));
  int hstat[4] = {0, 0, 0, 0};
  GGM_CUDA_TRY(cudaMemcpyAsync(hstat, istat, sizeof(hstat), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  int extra = 0;
  int passes = hstat[3];
  if (!hstat[1] && sp.scheme == kSchemeSquarem) {  // accelerated run failed: plain MM
    extra = hstat[0];
    sp.scheme = kSchemeMM;
    ce = launch_solve(sp, J, nblk, smem_launch, s);
    if (ce != cudaSuccess) return fail(GGM_ERR_CUDA, "solve_kernel launch: %s", cudaGetErrorString(ce));
    GGM_CUDA_TRY(cudaMemcpyAsync(hstat, istat, sizeof(hstat), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    passes += hstat[3];
  }
  GGM_CUDA_TRY(cudaEventRecord(ev[1], s));
  GGM_CUDA_TRY(cudaEventSynchronize(ev[1]));
  float kms = 0.f;
  GGM_CUDA_TRY(cudaEventElapsedTime(&kms, ev[0], ev[1]));
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  // Σ log s of the result (grid invariant: gauge shifts do not change it)
  for (int m = 0; m < sp.M; ++m) logsum_kernel<<<num_sms() * 4, 256, 0, s>>>(sp.gd[m], lam_res, scal + 1);
  GGM_CUDA_TRY(cudaGetLastError());
  Vec hL(T);
  double hscal[3] = {0, 0, 0};
  GGM_CUDA_TRY(cudaMemcpyAsync(hL.data(), lam_res, sizeof(double) * T, cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaMemcpyAsync(hscal, scal, sizeof(hscal), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));

  // gauge (reading G / G2), among the axes with no coordinate on the floor
  std::vector<int> pinned;
  int nfloor = 0;
  for (int a = 0; a < ax.nax; ++a) {
    bool on = false;
    for (int i = ax.off[a]; i < ax.off[a + 1]; ++i)
      if (barrier && hL[i] <= eps * (1.0 + 1e-9)) {
        on = true;
        ++nfloor;
      }
    if (on) pinned.push_back(a);
  }
  const std::vector<Vec> N = ax.gauge_free(pinned);
  Vec shift(ax.nax, 0.0);
  if (!N.empty()) {
    if (o.gauge == 0) {  // λ_l − (P_{G_F} μ)_l, μ_l = min λ_l
      Vec mu(ax.nax);
      for (int a = 0; a < ax.nax; ++a) {
        double mn = hL[ax.off[a]];
        for (int i = ax.off[a]; i < ax.off[a + 1]; ++i) mn = std::min(mn, hL[i]);
        mu[a] = mn;
      }
      for (const Vec& n : N) {
        double d = 0.0;
        for (int a = 0; a < ax.nax; ++a) d += n[a] * mu[a];
        for (int a = 0; a < ax.nax; ++a) shift[a] += d * n[a];
      }
    } else {  // (λ − 1/E) ⊥ lift(G_F)
      Vec D(ax.nax, 0.0);
      for (int a = 0; a < ax.nax; ++a)
        for (int i = ax.off[a]; i < ax.off[a + 1]; ++i) D[a] += hL[i] - 1.0 / hE[i];
      shift = ax.lifted_shift(N, D);
    }
  }
  Vec out(T);
  for (int a = 0; a < ax.nax; ++a)
    for (int i = ax.off[a]; i < ax.off[a + 1]; ++i) out[i] = hL[i] - shift[a];
  GGM_CUDA_TRY(cudaMemcpyAsync(lambda, out.data(), sizeof(double) * T, cudaMemcpyHostToDevice, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (info) {
    double lin = 0.0;
    for (int i = 0; i < T; ++i) lin += hE[i] * out[i];
    double gmin = INFINITY;
    for (const auto& m : ax.mods) {
      double sm = 0.0;
      for (int a : m) {
        double mn = out[ax.off[a]];
        for (int i = ax.off[a]; i < ax.off[a + 1]; ++i) mn = std::min(mn, out[i]);
        sm += mn;
      }
      gmin = std::min(gmin, sm);
    }
    info->iterations = hstat[0] + extra;
    info->stationarity = hscal[2];
    info->nll = 0.5 * lin - 0.5 * hscal[1];
    info->grid_min = gmin;
    info->floor_active = nfloor > 0 ? 1 : 0;
    info->trace_inconsistency = ti;
    info->passes = passes;
    info->kernel_ms = kms;
  }
  GGM_CUDA_TRY(cudaFreeAsync(buf.p, s));
  buf.p = nullptr;
  if (!hstat[1])
    return fail(GGM_ERR_NO_CONVERGENCE, "no convergence in %d iterations (residual %.3e)%s",
                o.max_iter, hscal[2], hstat[2] ? " (step size underflow)" : "");
  return GGM_OK;
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
  o->trace_tol = 1e-8;
}

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
  SolveParams sp;
  memset(&sp, 0, sizeof(sp));
  sp.gd[0] = gd;
  sp.M = 1;
  sp.T = gd.total;
  ModelAxes ax;
  ax.nax = L;
  ax.k.assign(k, k + L);
  ax.off.assign(gd.off, gd.off + L + 1);
  std::vector<int> all(L);
  for (int a = 0; a < L; ++a) all[a] = a;
  ax.mods.push_back(all);
  return solve_common(sp, ax, E, o, lambda, info, static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------------ multi-modal solve
// Thm 2 with Σ_γ: NLL = ½ Σ_l E_l·λ_l − ½ Σ_γ Σ_{j∈grid γ} log s^γ_j, gradient
// ½(E_l − Σ_{γ∋l} g^γ_l).  The majorise-minimise step is unchanged (one Jensen majoriser
// per modality, summed): λ ← λ ⊙ (Σ_γ g^γ) / E, so the same persistent kernel runs with one
// grid pass per modality per iteration.  Gauge (reading G2): shifts c with Σ_{l∈γ} c_l = 0
// for every γ leave all grid sums unchanged; reading T with that gauge space.
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
  ModelAxes ax;
  ax.nax = A;
  ax.k.assign(k, k + A);
  ax.off = offg;
  for (int g = 0; g < M; ++g) {
    const int L = mod_ptr[g + 1] - mod_ptr[g];
    const int* axl = mod_axes + mod_ptr[g];
    std::vector<int> here(A, 0);
    for (int a = 0; a < L; ++a) {
      if (axl[a] < 0 || axl[a] >= A) return fail(GGM_ERR_INVALID_ARGUMENT, "axis id out of range");
      if (here[axl[a]]++) return fail(GGM_ERR_INVALID_ARGUMENT, "repeated axis in a modality (P:181)");
      seen[axl[a]] = 1;
    }
    ggm_status st = make_desc_mod(L, axl, k, offg.data(), T, &sp.gd[g]);
    if (st != GGM_OK) return st;
    ax.mods.push_back(std::vector<int>(axl, axl + L));
  }
  for (int a = 0; a < A; ++a)
    if (!seen[a]) return fail(GGM_ERR_INVALID_ARGUMENT, "axis %d occurs in no modality", a);
  ggm_solve_opts o;
  ggm_solve_opts_default(&o);
  if (opts) o = *opts;
  sp.M = M;
  sp.T = T;
  return solve_common(sp, ax, E, o, lambda, info, static_cast<cudaStream_t>(stream));
}
