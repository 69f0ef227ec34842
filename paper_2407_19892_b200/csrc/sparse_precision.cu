// sparse_precision.cu — fused recomposition + per-row sparsification of
//   Ψ = V diag(λ) V^T   (Cor. of Thm 2; Alg. 1 lines 18-20)
// evaluated in 128 x 256 tiles on sm_100a tensor cores (tcgen05.mma, fp32 accumulators in
// TMEM), with the per-row top-t / threshold selection fused into the epilogue so that the
// n x n matrix is never written ("we eigen-recompose and threshold simultaneously").
//
// Kernels:
//   BK1a absmax_check   max_{i,r} |V_ir|·sqrt(λ_r), finiteness / λ>0 flags
//   BK1b scale_finalize power-of-two scale s = 2^e with max|U|·s <= 2^14
//   BK1c split_tile     U·s = hi + lo (two fp16 terms) written in the pre-swizzled
//                       (SWIZZLE_128B, K-major) 128-row block layout the MMA reads
//   BK2  fused_recon_topk  persistent, warp-specialised: 1 producer warp (bulk async
//                       copies), 1 MMA-issuer warp (3 MMAs / K-step: hi·hi, hi·lo, lo·hi),
//                       8 epilogue warps (tcgen05.ld thread = row, register top-t).  Three
//                       tile enumerations ("kinds"): plain (rows x all columns), seed (rows x
//                       a strided column sample -> per-row lower bounds of the t-th |ψ|) and
//                       symmetric (each unordered 128x128 block pair once, cyclic window;
//                       the transposed direction emits candidates above the seed bound)
//   BK3  merge_partials / merge_sym / coo_to_csr  CSR assembly
// The CTA-pair instantiations always keep A resident, so the streamed-A producer loop is
// statically unreachable there (diagnostic 128).
#pragma nv_diag_suppress 128
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "ggm_internal.h"
#include "ptx_sm100.cuh"

namespace ggm {
namespace sp {

constexpr int kRowsPerBlock = 128;        // M (rows of Ψ per CTA tile; TMEM lanes)
constexpr int kTileN = 256;               // N (columns of Ψ per tile; 2 operand blocks)
constexpr int kAtomElems = 64;            // fp16 elements per 128-byte swizzle row
constexpr int kAtomBytes = kRowsPerBlock * 128;  // one (128-row block, K atom) = 16 KB
constexpr int kMaxStages = 4;  // operand pipeline: 4 x 32 KB (A resident) or 2 x 96 KB
// Warp layout: warpgroup 0 = producer (+TMEM alloc), MMA issuer and 2 idle warps, shrunk to
// kRegsCtl registers (setmaxnreg); then EPW epilogue warps (EPW/4 per TMEM lane quadrant)
// grown to regs_epi(EPW).  The list epilogue (kPlain, and the seed for t > 10) runs 8 warps
// with 224 registers; the candidate / seed epilogues run 16 warps with 104 registers, which
// halves each warp's TMEM read-out and processing per tile and doubles the warps available
// to hide their latency.  (With 10 warps one SM sub-partition would hold 3 warps and cap
// every thread at 168 registers.)
constexpr int kFirstEpiWarp = 4;
#ifndef GGM_LEAN_ISSUE
#define GGM_LEAN_ISSUE 1
#endif
#ifndef GGM_LEAN_ISSUERS
#define GGM_LEAN_ISSUERS 1  // 2: the lean hi-only loop alternates tiles between warps 1 and 2
#endif
#ifndef GGM_MMA_THROTTLE
#define GGM_MMA_THROTTLE 0
#endif
#ifndef GGM_MMA_WARP
#define GGM_MMA_WARP 1  // control warp (1..3) that issues the MMAs; its SM sub-partition is
#endif                  // the one of TMEM lane quadrant GGM_MMA_WARP
#ifndef GGM_WAIT_HINT
#define GGM_WAIT_HINT 1
#endif
#if GGM_WAIT_HINT
#define LEAN_WAIT mbar_wait_sleep
#else
#define LEAN_WAIT mbar_wait
#endif
constexpr int kRegsCtl = 56;
__host__ __device__ constexpr int threads_of(int EPW) { return (kFirstEpiWarp + EPW) * 32; }
// setmaxnreg.inc draws only on what warpgroup 0 released: 8 warps: 384 threads launch at 168,
// 128 x (168 - 56) = 256 x (224 - 168); 16 warps: 640 threads launch at 96,
// 128 x (96 - 56) >= 512 x (104 - 96).
__host__ __device__ constexpr int regs_epi(int EPW) { return EPW == 16 ? 104 : 224; }
constexpr int kTmemCols = 512;            // 2 accumulator buffers x 256 columns
constexpr int kMaxResidentAtoms = 2;
// A (128 rows x KA atoms x hi/lo) stays resident in shared memory when KA <= 2 (k <= 128)
constexpr int kScratchBytes = 32 * 1024;  // epilogue shared scratch (per CTA)
constexpr int kScratchFloats = 32 * 32;   // per warp at 8 epilogue warps (half at 16)
constexpr int kSeedFrac = 32;       // seed pass: the n/32 largest-norm columns (see make_plan)
constexpr int kSeedMinTiles = 48;  // ... but at least 48 tiles while that is <= 1/8 of the axis

__host__ __device__ inline size_t block_bytes(int KA) { return (size_t)2 * KA * kAtomBytes; }

struct DevScalars {
  unsigned int absmax_bits;  // float bits of max |U|
  int flags;                 // 1 = non-finite V, 2 = lambda <= 0 or non-finite
  int exp2;                  // e: s = 2^e
  int cand_overflow;         // kSym: candidate pool exhausted -> exact fallback
  unsigned long long coo_count;
  unsigned long long cand_alloc;  // kSym: entries reserved from the candidate pool
  unsigned int rn_max_bits;       // kSym: float bits of max_i ||U_i||
  unsigned long long cand_emitted;  // kSym: candidates written (<= cand_alloc)
};
// candidate-pool reservation granularity (entries): one chunk must hold the worst case of
// one 32x32 warp chunk in both directions, so a fresh reservation always fits
constexpr int kCandChunk = 2048;
static_assert(kCandChunk >= 2 * 32 * 32, "a warp chunk's candidates must fit one reservation");
constexpr int kRecCutRatio = 4;  // re-evaluation cuts when the pool averages > 4t per row
constexpr int kRecCutMinT = 16;  // cuts (and the screened values they need) from t = 16
#ifndef GGM_WSPLIT
#define GGM_WSPLIT 8
#endif
// rare path, transposed direction: entries are tested against the minimum bound of their
// GGM_CMASK_W-column group (8; 32 = the chunk minimum) or, GGM_CMASK_W = 1, their own
// column's bound (profiles/r02_logs/ab_cmask*.log)
#ifndef GGM_CMASK_W
#define GGM_CMASK_W 8
#endif
static_assert(GGM_CMASK_W == 1 || GGM_CMASK_W == 8 || GGM_CMASK_W == 32, "GGM_CMASK_W: 1, 8 or 32");
constexpr int kWindowSplit = GGM_WSPLIT;  // kSym/kSymList CTA-pair units per row block (sub-windows)
constexpr int64_t kSymAutoN = 16384;  // automatic symmetric scheme from this axis length (measured crossover 8192-16384)

// ------------------------------------------------------------------ BK1a
__global__ void absmax_check(const float* __restrict__ V, const double* __restrict__ lam,
                             int64_t n, int k, DevScalars* sc) {
  __shared__ float red[32];
  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      double l = lam[c];
      if (!(l > 0.0) || !isfinite(l)) atomicOr(&sc->flags, 2);
    }
  }
  __shared__ double sl[1024];
  const bool staged = k <= 1024;
  if (staged)
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      const double l = lam[c];
      sl[c] = sqrt(l > 0.0 ? l : 0.0);
    }
  __syncthreads();
  float m = 0.f;
  int bad = 0;
  const int64_t total = n * (int64_t)k;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  if (staged && (k & 3) == 0 && (reinterpret_cast<uintptr_t>(V) & 15) == 0) {
    // float4 form: 4 consecutive columns of one row per load (k ≡ 0 mod 4, aligned V)
    const float4* V4 = reinterpret_cast<const float4*>(V);
    const int64_t total4 = total >> 2;
    const int k4 = k >> 2;
    const int cstep4 = (int)(step % k4);
    int c4 = (int)(i0 % k4);
    for (int64_t idx = i0; idx < total4; idx += step) {
      const float4 v = __ldg(V4 + idx);
      if (!isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w)) bad = 1;
      const int c = 4 * c4;
      m = fmaxf(m, fmaxf(fmaxf((float)(fabs((double)v.x) * sl[c]), (float)(fabs((double)v.y) * sl[c + 1])),
                         fmaxf((float)(fabs((double)v.z) * sl[c + 2]), (float)(fabs((double)v.w) * sl[c + 3]))));
      c4 += cstep4;
      if (c4 >= k4) c4 -= k4;
    }
  } else {
  const int cstep = (int)(step % k);
  int c = (int)(i0 % k);  // column of idx, advanced incrementally (no division per element)
  for (int64_t idx = i0; idx < total; idx += step) {
    float v = V[idx];
    if (!isfinite(v)) bad = 1;
    double sq;
    if (staged) {
      sq = sl[c];
    } else {
      const double l = lam[c];
      sq = sqrt(l > 0.0 ? l : 0.0);
    }
    float u = (float)(fabs((double)v) * sq);
    m = fmaxf(m, u);
    c += cstep;
    if (c >= k) c -= k;
  }
  }
  if (bad) atomicOr(&sc->flags, 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) atomicMax(&sc->absmax_bits, __float_as_uint(m));
  }
}

// kSym: per-row norm ||U_i|| = sqrt(Σ_r λ_r V_ir²) (fp64, one warp per row) and its maximum
__global__ void row_norms(const float* __restrict__ V, const double* __restrict__ lam, int64_t n,
                          int k, float* __restrict__ rn, unsigned int* __restrict__ rn_max_bits) {
  const int lane = threadIdx.x & 31;
  float wmax = 0.f;
  if ((k & 3) == 0 && k <= 1024 && (reinterpret_cast<uintptr_t>(V) & 15) == 0) {
    // float4 form: 8 lanes per row, 4 rows per warp step (λ staged in shared memory)
    __shared__ double sl[1024];
    for (int c = threadIdx.x; c < k; c += blockDim.x) sl[c] = lam[c];
    __syncthreads();
    const int l8 = lane & 7, k4 = k >> 2;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t wstep = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i0 = w0 * 4; i0 < n; i0 += wstep * 4) {
      const int64_t i = i0 + (lane >> 3);
      double acc = 0.0;
      if (i < n) {
        const float4* v4 = reinterpret_cast<const float4*>(V + i * k);
        for (int j = l8; j < k4; j += 8) {
          const float4 x = __ldg(v4 + j);
          const double* l = sl + 4 * j;
          acc += l[0] * (double)x.x * (double)x.x + l[1] * (double)x.y * (double)x.y +
                 l[2] * (double)x.z * (double)x.z + l[3] * (double)x.w * (double)x.w;
        }
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (i < n) {
        const float f = (float)sqrt(acc);
        if (l8 == 0) rn[i] = f;
        wmax = fmaxf(wmax, f);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    if (lane == 0) atomicMax(rn_max_bits, __float_as_uint(wmax));
    return;
  }
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double acc = 0.0;
    for (int c = lane; c < k; c += 32) {
      const double x = (double)V[i * k + c];
      acc += lam[c] * x * x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const float f = (float)sqrt(acc);
    if (lane == 0) rn[i] = f;
    wmax = fmaxf(wmax, f);
  }
  if (lane == 0) atomicMax(rn_max_bits, __float_as_uint(wmax));
}

// Screening error bound of entry (i, j) in accumulator units (x = U·2^e, hi = fp16(x),
// lo = fp16(x - hi)).  For a normal fp16 hi, |x - hi| <= 2^-11 |hi|; below the fp16 normal range
// (|x| < 2^-14, i.e. |U| < 2^-28 max|U|) the rounding error is absolute, <= 2^-25, and |lo - (x -
// hi)| <= 2^-25 likewise.  Hence for both the seed relation |ψ3 - ψ1| = |Σ hi lo + lo hi| and the
// screening relation |ψ - ψ1| (ψ the exact product of the fp32 inputs):
//   |ψ - ψ1| <= 2^-10 (1 + 2^-11) ||x_i|| ||x_j|| + 2^-24 sqrt(k) (||x_i|| + ||x_j||) + fp32 terms,
// bounded by 1.1 · 2^-10 ||x_i|| M + 2^-23 sqrt(k) (||x_i|| + M), M = max_j ||x_j|| (the relative
// term alone is not a bound for rows with near-zero norms).
__device__ __forceinline__ float screen_margin(float rn_s, float umax_s, int k) {
  return 1.1f * ldexpf(rn_s * umax_s, -10) + ldexpf(sqrtf((float)k) * (rn_s + umax_s), -23);
}

// kSym: seed value b1_i (t-th largest |hi·hi| chunk maximum, accumulator units) -> a lower
// bound of the row's t-th 3-term magnitude (b1 minus screen_margin; fp32 accumulation
// differences, k 2^-24 ||x_i|| ||x_j||, are covered by the factor 1.1).
__global__ void seed_bounds(float* __restrict__ thr, const float* __restrict__ rn,
                            const unsigned int* __restrict__ rn_max_bits, int64_t n, int k,
                            const DevScalars* __restrict__ sc) {
  const float s = ldexpf(1.f, sc->exp2);
  const float umax = __uint_as_float(*rn_max_bits) * s;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float b1 = thr[i];
    const float margin = screen_margin(rn[i] * s, umax, k);
    thr[i] = b1 > 0.f ? fmaxf(b1 - margin, -1.f) : -1.f;
  }
}

// kSym screening thresholds: the main pass computes hi·hi only (|ψ1 - ψ| <= screen_margin),
// so entry (i, j) is kept for row i if |ψ1| >= b_i - screen_margin(i) (and symmetrically for
// row j): every entry with |ψ| >= b_i survives.  Bound order p (perm[p] = original id);
// padding stays +inf.
__global__ void screen_bounds(const float* __restrict__ thr_p, const float* __restrict__ rn,
                              const int32_t* __restrict__ perm,
                              const unsigned int* __restrict__ rn_max_bits, int64_t n, int k,
                              int64_t nthr, const DevScalars* __restrict__ sc,
                              float* __restrict__ thr_s) {
  const float s = ldexpf(1.f, sc->exp2);
  const float umax = __uint_as_float(*rn_max_bits) * s;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nthr;
       p += (int64_t)gridDim.x * blockDim.x) {
    const float b = thr_p[p];
    if (p < n && b < INFINITY) {
      const float margin = screen_margin(rn[perm[p]] * s, umax, k);
      thr_s[p] = b > -1.f ? b - margin : b;
    } else {
      thr_s[p] = b;
    }
  }
}

__global__ void fill_tau(float* __restrict__ thr, int64_t n, float tau,
                         const DevScalars* __restrict__ sc) {
  const float ts = ldexpf(tau, 2 * sc->exp2);  // ψ units -> accumulator units
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    thr[i] = ts;
}
__global__ void cap_tau(float* __restrict__ thr, int64_t n, float tau,
                        const DevScalars* __restrict__ sc) {
  const float ts = ldexpf(tau, 2 * sc->exp2);  // ψ units -> accumulator units
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    thr[i] = fminf(thr[i], ts);
}
// overall rules, global-threshold pass: the pairs (i < j, original ids) of the exact
// candidates with |ψ| > τ, once each (both directions are candidates: bounds <= τ), as pair
// keys i*n + j and signed values; *count counts all (only the first cap are written)
__global__ void sym_upper_pairs(const uint32_t* __restrict__ skey, const uint2* __restrict__ sval,
                                int64_t ncand, int64_t n, const int32_t* __restrict__ perm,
                                float tau, int64_t cap, unsigned long long* count,
                                uint64_t* __restrict__ pkey, float* __restrict__ score) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ncand; base += stride) {
    const int64_t e = base + threadIdx.x;
    bool keep = false;
    int64_t i = 0, j = 0;
    float v = 0.f;
    if (e < ncand) {
      const uint32_t t = skey[e];
      if (t != 0xFFFFFFFFu) {
        const uint2 x = sval[e];
        v = __uint_as_float(x.y);
        i = perm[t];
        j = perm[x.x];
        keep = i < j && fabsf(v) > tau;
      }
    }
    const uint32_t bm = __ballot_sync(0xffffffffu, keep);
    unsigned long long b0 = 0;
    if (lane == 0 && bm) b0 = atomicAdd(count, (unsigned long long)__popc(bm));
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if (keep) {
      const int64_t pos = (int64_t)b0 + __popc(bm & ((1u << lane) - 1u));
      if (pos < cap) {
        pkey[pos] = (uint64_t)i * (uint64_t)n + (uint64_t)j;
        score[pos] = v;
      }
    }
  }
}
// symmetric threshold mode: candidates with |ψ| > τ (exact values) -> COO (original row * n +
// original column, ψ); count in *count (entries beyond capacity are counted, not written)
__global__ void sym_threshold_coo(const uint32_t* __restrict__ skey, const uint2* __restrict__ sval,
                                  int64_t ncand, int64_t n, const int32_t* __restrict__ perm,
                                  float tau, int64_t capacity, unsigned long long* count,
                                  int64_t* __restrict__ key_out, float* __restrict__ val_out) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ncand; base += stride) {
    const int64_t e = base + threadIdx.x;
    bool keep = false;
    uint32_t j = 0;
    uint2 x = make_uint2(0, 0);
    if (e < ncand) {
      j = skey[e];
      x = sval[e];
      keep = j != 0xFFFFFFFFu && fabsf(__uint_as_float(x.y)) > tau;
    }
    const uint32_t bm = __ballot_sync(0xffffffffu, keep);
    unsigned long long b0 = 0;
    if (lane == 0 && bm) b0 = atomicAdd(count, (unsigned long long)__popc(bm));
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if (keep) {
      const int64_t pos = (int64_t)b0 + __popc(bm & ((1u << lane) - 1u));
      if (pos < capacity) {
        key_out[pos] = (int64_t)perm[j] * n + perm[x.x];
        val_out[pos] = __uint_as_float(x.y);
      }
    }
  }
}

__global__ void chunk_min32(const float* __restrict__ thr, int64_t nchunks,
                            float* __restrict__ out, int width = 32) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    float m = INFINITY;
    for (int e = 0; e < width; ++e) m = fminf(m, thr[c * width + e]);
    out[c] = m;
  }
}

// ------------------------------------------------------------------ BK1b
__global__ void scale_finalize(DevScalars* sc) {
  float m = __uint_as_float(sc->absmax_bits);
  int e = 0;
  if (m > 0.f && isfinite(m)) {
    int ex;
    frexpf(m, &ex);          // m = f·2^ex, f in [0.5,1)  =>  m < 2^ex
    e = 14 - ex;             // max|U|·2^e < 2^14: hi fits fp16 with headroom; fp32 sums safe
    e = max(-100, min(100, e));
  }
  sc->exp2 = e;
}

// ------------------------------------------------------------------ BK1c
// dst holds `nblocks` 128-row blocks: [block][hi atoms 0..KA-1][lo atoms 0..KA-1], each
// atom 128 rows x 128 bytes, 16-byte chunk c of row r stored at chunk (c ^ (r & 7))
// (the SWIZZLE_128B K-major canonical layout; SBO = 1024 B between 8-row groups).
// A K slot is 16 fp16 (32 B, one MMA K step); slot s of the hi/lo array holds hi/lo of
// elements 16s..16s+15 for s < KS.  With a packed tail (TS > 0, r = k - 16 KS), the
// products of the last r elements go into TS slots that hold 3r values each:
//   hi array slot KS+u : TB = [hi(x_tail) | lo(x_tail) | hi(x_tail)]   (B side)
//   lo array slot KS+u : TA = [hi(x_tail) | hi(x_tail) | lo(x_tail)]   (A side)
// so one MMA TA·TB^T = hi·hi + hi·lo + lo·hi over the tail (positions 16u.. of the packed
// sequence).  Remaining slots are zero.
__device__ __forceinline__ void split2(double x, __half& h, __half& l) {
  h = __double2half(x);
  l = __double2half(x - (double)__half2float(h));
}
// One thread per (row, 16-byte chunk): the 8 elements are split once and both the hi-array
// and the lo-array chunk are written (sqrt(λ) staged in shared memory; 32-bit index math).
constexpr int kSplitMaxK = 1024;
__global__ void split_tile_generic(const float* __restrict__ V, const double* __restrict__ lam,
                           int64_t n, int k, int KA, int KS, int TS, int64_t row0,
                           int64_t nrows_pad, const DevScalars* __restrict__ sc,
                           uint8_t* __restrict__ dst, const int32_t* __restrict__ perm = nullptr) {
  __shared__ double sl[kSplitMaxK];
  const bool staged = k <= kSplitMaxK;
  if (staged)
    for (int c = threadIdx.x; c < k; c += blockDim.x) sl[c] = sqrt(lam[c]);
  __syncthreads();
  const int cpr = KA * 8;  // 16-byte chunks of one array per row
  const int64_t total = nrows_pad * cpr;
  const double s = ldexp(1.0, sc->exp2);
  const int r = k - 16 * KS;  // tail elements (packed when TS > 0)
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t row;
    int ch;
    if (total < (int64_t(1) << 31)) {
      const uint32_t i32 = (uint32_t)idx;
      row = i32 / (uint32_t)cpr;
      ch = (int)(i32 - (uint32_t)row * (uint32_t)cpr);
    } else {
      row = idx / cpr;
      ch = (int)(idx % cpr);
    }
    int64_t g = row0 + row;
    const bool real = g < n;
    if (perm && real) g = perm[g];  // symmetric scheme: rows in bound order
    const int slot = ch >> 1;
    __align__(16) __half oh[8];
    __align__(16) __half ol[8];
    const float* vrow = V + g * k;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int pos = (ch & 1) * 8 + e;  // position within the slot
      __half h = __float2half(0.f), l = __float2half(0.f);
      __half v0 = h, v1 = h;
      if (real) {
        if (slot < KS || TS == 0) {
          const int c = slot * 16 + pos;
          if (c < k) {
            split2((double)vrow[c] * (staged ? sl[c] : sqrt(lam[c])) * s, h, l);
            v0 = h;
            v1 = l;
          }
        } else if (slot < KS + TS) {
          const int q = (slot - KS) * 16 + pos;  // position in the packed tail sequence
          if (q < 3 * r) {
            const int seg = q / r;
            const int c = 16 * KS + q % r;
            split2((double)vrow[c] * (staged ? sl[c] : sqrt(lam[c])) * s, h, l);
            // B (hi array): [hi | lo | hi];  A (lo array): [hi | hi | lo]
            v0 = seg == 1 ? l : h;
            v1 = seg == 2 ? l : h;
          }
        }
      }
      oh[e] = v0;
      ol[e] = v1;
    }
    const int64_t b = row / kRowsPerBlock;
    const int rr = (int)(row % kRowsPerBlock);
    const int a = ch >> 3, c8 = ch & 7;
    const size_t base = (size_t)b * block_bytes(KA) + (size_t)rr * 128 + (size_t)((c8 ^ (rr & 7)) * 16);
    *reinterpret_cast<uint4*>(dst + base + (size_t)a * kAtomBytes) = *reinterpret_cast<const uint4*>(oh);
    *reinterpret_cast<uint4*>(dst + base + (size_t)(KA + a) * kAtomBytes) =
        *reinterpret_cast<const uint4*>(ol);
  }
}

// Fast form (8·KA ≤ 256 chunks per row, i.e. k ≤ 2048): a block is `rpb` rows × 8·KA
// chunks, so every thread keeps one fixed chunk and its 8 source columns, scales
// sqrt(λ_c)·s (as an fp32 pair sh + sl, |sl| ≤ 2⁻²⁴ sh) and tail positions in registers
// across its grid-stride rows.  The split runs in fp32: p = fl(v·sh) with its exact
// FMA error, hi = fp16(p), lo = fp16((p − hi) + err + v·sl), so hi + lo carries x = v·sqrt(λ)·s
// to ~2⁻²² relative as before and |x − hi| ≤ 2⁻¹¹(1 + 2⁻¹²)|x| (inside the 1.1 slack of the
// screening margins) — without the fp64 conversions of the generic form.  Full slots of a
// k ≡ 0 (mod 4) factor are read with two float4 loads.
__global__ void split_tile_fast(const float* __restrict__ V, const double* __restrict__ lam,
                                int64_t n, int k, int KA, int KS, int TS, int64_t row0,
                                int64_t nrows_pad, const DevScalars* __restrict__ sc,
                                uint8_t* __restrict__ dst, const int32_t* __restrict__ perm) {
  const int cpr = KA * 8;
  const int rpb = blockDim.x / cpr;
  const int ch = threadIdx.x % cpr, rsub = threadIdx.x / cpr;
  if (rsub >= rpb) return;
  const double s = ldexp(1.0, sc->exp2);
  const int slot = ch >> 1;
  const int r = k - 16 * KS;
  int src[8], seg[8];
  float sh[8], sl[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int pos = (ch & 1) * 8 + e;
    src[e] = -1;
    seg[e] = 0;
    if (slot < KS || TS == 0) {
      const int c = slot * 16 + pos;
      if (c < k) src[e] = c;
    } else if (slot < KS + TS) {
      const int q = (slot - KS) * 16 + pos;
      if (q < 3 * r) {
        seg[e] = q / r;
        src[e] = 16 * KS + q % r;
      }
    }
    const double d = src[e] >= 0 ? sqrt(lam[src[e]]) * s : 0.0;
    sh[e] = (float)d;
    sl[e] = (float)(d - (double)sh[e]);
  }
  const int c0 = slot * 16 + (ch & 1) * 8;
  const bool vec = (slot < KS || TS == 0) && (k & 3) == 0 && c0 + 8 <= k;
  const int a = ch >> 3, c8 = ch & 7;
  for (int64_t row = (int64_t)blockIdx.x * rpb + rsub; row < nrows_pad;
       row += (int64_t)gridDim.x * rpb) {
    int64_t g = row0 + row;
    const bool real = g < n;
    if (perm && real) g = perm[g];  // symmetric scheme: rows in bound order
    float x[8];
    if (real && vec) {
      const float4* vp = reinterpret_cast<const float4*>(V + g * k + c0);
      const float4 x0 = __ldg(vp), x1 = __ldg(vp + 1);
      x[0] = x0.x; x[1] = x0.y; x[2] = x0.z; x[3] = x0.w;
      x[4] = x1.x; x[5] = x1.y; x[6] = x1.z; x[7] = x1.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = (real && src[e] >= 0) ? __ldg(V + g * k + src[e]) : 0.f;
    }
    __align__(16) __half oh[8];
    __align__(16) __half ol[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float pr = x[e] * sh[e];
      const float err = fmaf(x[e], sh[e], -pr);
      const __half h = __float2half_rn(pr);
      const __half l = __float2half_rn((pr - __half2float(h)) + fmaf(x[e], sl[e], err));
      // plain slots: hi / lo; packed tail: B (hi array) [hi | lo | hi], A (lo array) [hi | hi | lo]
      oh[e] = seg[e] == 1 ? l : h;
      ol[e] = (seg[e] == 2 || (seg[e] == 0 && !(slot >= KS && TS > 0))) ? l : h;
      if (src[e] < 0) {
        oh[e] = __float2half(0.f);
        ol[e] = __float2half(0.f);
      }
    }
    const int64_t b = row / kRowsPerBlock;
    const int rr = (int)(row % kRowsPerBlock);
    const size_t base = (size_t)b * block_bytes(KA) + (size_t)rr * 128 + (size_t)((c8 ^ (rr & 7)) * 16);
    *reinterpret_cast<uint4*>(dst + base + (size_t)a * kAtomBytes) = *reinterpret_cast<const uint4*>(oh);
    *reinterpret_cast<uint4*>(dst + base + (size_t)(KA + a) * kAtomBytes) =
        *reinterpret_cast<const uint4*>(ol);
  }
}

// Operand split of rows [row0, row0 + nrows_pad) (padding rows past n are zero): the fast
// form when a row's chunks fit one 256-thread block, the generic grid-stride form otherwise.
static void launch_split(cudaStream_t st, int sms, const float* V, const double* lam, int64_t n,
                         int k, int KA, int KS, int TS, int64_t row0, int64_t nrows_pad,
                         const DevScalars* sc, uint8_t* dst, const int32_t* perm = nullptr) {
  const int cpr = KA * 8;
  if (cpr <= 256) {
    const int rpb = 256 / cpr;
    const int64_t blocks = (nrows_pad + rpb - 1) / rpb;
    split_tile_fast<<<(int)std::max<int64_t>(1, std::min<int64_t>(blocks, sms * 16)), cpr * rpb,
                      0, st>>>(V, lam, n, k, KA, KS, TS, row0, nrows_pad, sc, dst, perm);
  } else {
    const int64_t tot = nrows_pad * cpr;
    split_tile_generic<<<(int)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, sms * 16)),
                         256, 0, st>>>(V, lam, n, k, KA, KS, TS, row0, nrows_pad, sc, dst, perm);
  }
}

// ------------------------------------------------------------------ BK2
// ------------------------------------------------------------------ BK2
// kSymList: the kSym block-pair enumeration (each unordered 128-row block pair once) with the
// list-form epilogue; used for the row masses of the overall rules (mode 2: row sums into
// the rows, column sums into the columns of every off-diagonal tile)
enum Kind : int { kPlain = 0, kSeed = 1, kSym = 2, kSymList = 3 };

struct FusedParams {
  const uint8_t* A;  // row-block operand (rows [row_begin,row_end)), tiled layout
  const uint8_t* B;  // column operand (all n rows, padded to 256), tiled layout
  int KA;            // K atoms of 64
  int KS;            // full K slots of 16 (3 MMAs each: hi·hi, hi·lo, lo·hi)
  int TS;            // packed tail slots (1 MMA each), see split_tile
  int resident;      // 1: A kept in shared memory for a whole row block
  int64_t n, row_begin, rows;
  int kind;          // Kind
  int RB, NT, C, TPC;
  int NB;            // kSym: 128-row blocks of the axis (row_begin == 0, rows == n)
  int SS;            // kSeed: number of 256-column tiles in the sample (the first ones)
  int mode, t;
  float tau;
  const DevScalars* sc;
  int64_t* row_ptr;
  int32_t* col;
  float* val;
  int32_t* pcol;     // partial per-row lists [C][rows][t] (plain C > 1, kSym: C = 1)
  float* pval;
  int64_t* coo_key;  // mode 1 candidates
  float* coo_val;
  unsigned long long* coo_count;
  int64_t capacity;
  float* thr_out;          // kSeed: per-row t-th largest sampled |ψ| (accumulator units)
  double* mass_out;        // mode 2: row masses Σ_{j≠i} |ψ_ij| in accumulator units (atomic
                           // partials; times 2^-2e by scale_pow2 after the pass)
  unsigned long long* hist_out;  // mode 3 (plain): counts of upper entries (j > i) with
                                 // |ψ| > τ in 256 log buckets b = min(255, (bits|ψ| - bits τ) >> hshift)
  int hshift;
  const float* thr;        // kSym: per-(permuted) column lower bound of that row's t-th
                           //       magnitude (accumulator units, +inf = padding)
  const float* thr_min;    // kSym: min of thr over each 32-column chunk (bound order)
  const float* thr_min8;   // kSym: min of thr over each 8-column group (the rare path's
                           // column-direction mask)
  const int32_t* perm;     // kSym: permuted index -> original row/column id
  uint32_t* cand_key;      // kSym: candidate pool: target row j (UINT32_MAX = unused slot)
  uint2* cand_val;         //       (source row i, ψ bits)
  int64_t cand_total;      //       pool capacity; warps reserve kCandChunk-entry chunks
  int screen;        // kSym: hi*hi screening MMAs only (candidates re-evaluated exactly)
  int cand_vals;     // kSym: 1 = store each candidate's value (no screening: the final value;
                     // screening: the screened value, read only by the re-evaluation cuts)
  int pair;          // CTA-pair kernel (host-side selection; the kernel's template PAIR)
  int wsplit;            // kSym / kSymList CTA pairs: each row block's window is cut into
                         // wsplit consecutive sub-windows, one unit each (unit u: sub-window
                         // u / NB of row block u % NB) — finer units balance the last wave
  int unit_step;         // units unit_lo, unit_lo + unit_step, ... < unit_hi (1: contiguous;
                         // nranks: the rank-strided share of the distributed symmetric scheme)
  int unit_lo, unit_hi;  // units processed by this launch (a rank's share in the sharded
                         // symmetric scheme; [0, all units) otherwise)
  int pm_n, pm_r;        // kSym part-major share (pm_n > 0, pm_n | wsplit): rank pm_r of pm_n
                         // takes sub-windows pm_r, pm_r + pm_n, ... of EVERY row block, in
                         // row-block order (unit_lo/hi/step unused)
#ifdef GGM_EPI_DEBUG
  int dbg;  // timing experiments only (GGM_DEBUG_EPI): 1 = TMEM loads only, 2 = no epilogue work
#endif
};
// Epilogue timing experiments exist only in -DGGM_EPI_DEBUG builds (tools/build_variant.sh);
// in the release library the switch is the constant 0 and no environment variable is read.
#ifdef GGM_EPI_DEBUG
#define GGM_DBG(p) ((p).dbg)
#else
#define GGM_DBG(p) 0
#endif

// Operand pipeline.  1 CTA, A resident (k <= 128): a stage holds B hi and B lo of one K atom
// for both 128-row operand blocks of the tile = 64 KB, 2 stages (the seed pass fills only the
// hi half).  1 CTA, A streamed: A hi+lo and B hi+lo of one K atom = 96 KB, 2 stages.  CTA
// pair (cta_group::2, A resident): each CTA holds only ITS 128-row half of the B tile, so a
// stage is 32 KB and the pipeline is 4 deep; per-SM L2->SMEM traffic per 128x256 tile halves
// (the 1-CTA kernel is bounded by the ~42 B/clk/SM L2 throughput at k = 100).
__host__ __device__ inline int num_stages(int resident, int pair) {
  return pair ? 4 : 2;
}
__host__ __device__ inline size_t stage_bytes(int resident, int pair) {
  return (size_t)(pair ? 2 : (resident ? 4 : 6)) * kAtomBytes;
}
__host__ inline size_t fused_smem_bytes(int KA, int resident, int pair) {
  size_t a = resident ? block_bytes(KA) : 0;
  return 1024 /*align slack*/ + a + num_stages(resident, pair) * stage_bytes(resident, pair) +
         256 /*barriers*/ + kScratchBytes;
}

// Tile enumeration shared by the producer, MMA and epilogue roles.  A unit is one row block
// ub (128 rows, or 256 rows = two 128-row blocks for a CTA pair) plus a column chunk for
// kPlain; tile s of the unit covers two 128-column operand blocks K0, K1 (the two N-halves
// of one x256 MMA tile; h1 = second half valid).  Units are strided over the CTAs (or CTA
// pairs): u = u0, u0 + ustep, ...
struct TileRef {
  int K0, K1;
  bool h1;
};
__device__ __forceinline__ int sym_window(int rb, int NB) {
  // blocks K = rb + d (mod NB), d < W: each unordered pair {I, K} exactly once
  return (NB & 1) ? (NB + 1) / 2 : NB / 2 + (rb < NB / 2 ? 1 : 0);
}
template <int KIND, bool PAIR>
__device__ __forceinline__ int unit_tiles(const FusedParams& p, int u, int& ub) {
  if (KIND == kPlain) {
    ub = u / p.C;
    const int j0 = (u % p.C) * p.TPC;
    return min(p.NT, j0 + p.TPC) - j0;
  }
  ub = u;
  if (KIND == kSeed) return p.SS;  // the sample: the first SS column tiles
  // kSym: window over p.NB blocks (128-column blocks, or 256-column super blocks for pairs)
  if (!PAIR) return (sym_window(ub, p.NB) + 1) / 2;
  const int part = u / p.NB;
  ub = u - part * p.NB;
  const int W = sym_window(ub, p.NB);
  return (part + 1) * W / p.wsplit - part * W / p.wsplit;
}
// Visit the kSym window [ub, ub + W) starting at X = the last unit of this wave (all CTAs of
// a wave contain X in their windows), so concurrently running CTAs stream the same column
// blocks in lockstep and share them through L2.
template <int KIND>
__host__ __device__ __forceinline__ int unit_count(const FusedParams& p) {
  if (KIND == kSym && p.pm_n > 0) return (p.wsplit / p.pm_n) * p.NB;
  return (p.unit_hi - p.unit_lo + p.unit_step - 1) / p.unit_step;
}
// Folded part-major share (pm_n ranks, wsplit sub-windows per row block, Q = wsplit / pm_n
// slots per row block and rank): sub-window j is paired with wsplit-1-j (the near-diagonal
// sub-windows emit fewer candidates than the far ones: C5, N = 8, 2.10M vs 2.88M per rank
// unfolded), rank r owns the pairs j = r, r + pm_n, ...; with one slot (Q = 1) it takes j on
// even and wsplit-1-j on odd row blocks.  Local unit uj = lp·NB + ub (row blocks in order).
template <int KIND>
__host__ __device__ __forceinline__ int unit_of(const FusedParams& p, int uj) {
  if (KIND == kSym && p.pm_n > 0) {
    const int lp = uj / p.NB, ub = uj - lp * p.NB;
    const int j = p.pm_r + p.pm_n * (lp >> 1);
    const bool far = ((lp + ub) & 1) != 0;
    return (far ? p.wsplit - 1 - j : j) * p.NB + ub;
  }
  return p.unit_lo + uj * p.unit_step;
}
template <int KIND>
__device__ __forceinline__ int sym_start(const FusedParams& p, int uj, int ub, int u0, int ustep,
                                         int w0, int w1) {
  const int X = unit_of<KIND>(p, min(unit_count<KIND>(p) - 1, uj - u0 + ustep - 1)) % p.NB;
  const int delta = (X - ub + p.NB) % p.NB;
  return (delta >= w0 && delta < w1) ? delta : w0;
}
// Incremental enumeration (no integer division per tile).
template <int KIND, bool PAIR>
struct TileIter {
  int K0, K1;
  bool h1;
  int s, ub, W, o;  // kSym: o = window offset of the current tile
  int w0, w1;       // kSym: this unit's sub-window [w0, w1) of the window
  __device__ __forceinline__ void start(const FusedParams& p, int u, int uj, int ub_, int u0,
                                        int ustep) {
    ub = ub_;
    s = 0;
    h1 = true;
    if (KIND >= kSym) {
      W = sym_window(ub, p.NB);
      const int part = PAIR ? u / p.NB : 0;
      w0 = PAIR ? part * W / p.wsplit : 0;
      w1 = PAIR ? (part + 1) * W / p.wsplit : W;
      o = sym_start<KIND>(p, uj, ub, u0, ustep, w0, w1);
      place(p);
    } else {
      const int j = KIND == kPlain ? (u % p.C) * p.TPC : 0;
      K0 = 2 * j;
      K1 = 2 * j + 1;
    }
  }
  __device__ __forceinline__ void place(const FusedParams& p) {
    if (PAIR) {  // one 256-column super block J per tile
      int J = ub + o;
      if (J >= p.NB) J -= p.NB;
      K0 = 2 * J;
      K1 = 2 * J + 1;
    } else {  // two 128-column blocks (window offsets o, o+1)
      int o1 = o + 1;
      if (o1 >= W) o1 -= W;
      K0 = ub + o;
      if (K0 >= p.NB) K0 -= p.NB;
      h1 = 2 * s + 1 < W;
      K1 = ub + o1;
      if (K1 >= p.NB) K1 -= p.NB;
      if (!h1) K1 = K0;
    }
  }
  __device__ __forceinline__ void next(const FusedParams& p) {
    ++s;
    if (KIND >= kSym) {
      o += PAIR ? 1 : 2;
      if (o >= w1) o -= w1 - w0;
      place(p);
    } else {
      K0 += 2;
      K1 += 2;
    }
  }
};

// Per-thread (= per-row) top-t list kept entirely in registers.  Slots are sorted
// ASCENDING by magnitude; slots p >= t hold +inf and never move, so the eviction threshold
// is always mag[0] (compile-time index, no local memory).  A new value with a > mag[0]
// drops mag[0]; an arrival equal to kept magnitudes is placed below them, so among equal
// magnitudes the earlier (smaller) column survives (ties -> smaller j, reading Q9).
template <int MAXT>
struct TopList {
  float mag[MAXT];
  float sval[MAXT];
  int idx[MAXT];
  __device__ __forceinline__ void init(int t) {
#pragma unroll
    for (int p = 0; p < MAXT; ++p) {
      mag[p] = (p < t) ? -1.f : __int_as_float(0x7f800000);
      sval[p] = 0.f;
      idx[p] = -1;
    }
  }
  // kSym: start from a known lower bound b of the row's t-th magnitude (phantom entries,
  // idx -1, just below b: any |ψ| >= b displaces them; never emitted)
  __device__ __forceinline__ void init_bound(int t, float b) {
    const float lb = b > 0.f ? __int_as_float(__float_as_int(b) - 1) : -1.f;
#pragma unroll
    for (int p = 0; p < MAXT; ++p) {
      mag[p] = (p < t) ? lb : __int_as_float(0x7f800000);
      sval[p] = 0.f;
      idx[p] = -1;
    }
  }
  __device__ __forceinline__ float thr() const { return mag[0]; }
  __device__ __forceinline__ void insert(float a, float v, int j) {
#pragma unroll
    for (int p = 0; p < MAXT - 1; ++p) {
      const bool up = a > mag[p + 1];
      const bool here = a > mag[p];
      if (up) {
        mag[p] = mag[p + 1];
        sval[p] = sval[p + 1];
        idx[p] = idx[p + 1];
      } else if (here) {
        mag[p] = a;
        sval[p] = v;
        idx[p] = j;
      }
    }
    if (a > mag[MAXT - 1]) {
      mag[MAXT - 1] = a;
      sval[MAXT - 1] = v;
      idx[MAXT - 1] = j;
    }
  }
  // Insert with the full order (|v| desc, then j asc) — for merging lists whose columns
  // interleave.  "Better" = larger magnitude, or equal magnitude and smaller column.
  __device__ __forceinline__ static bool better(float a, int j, float b, int k) {
    return a > b || (a == b && j < k);
  }
  __device__ __forceinline__ void merge_insert(float a, float v, int j) {
    if (!better(a, j, mag[0], idx[0])) return;  // not better than the current t-th entry
#pragma unroll
    for (int p = 0; p < MAXT - 1; ++p) {
      const bool up = better(a, j, mag[p + 1], idx[p + 1]);
      const bool here = better(a, j, mag[p], idx[p]);
      if (up) {
        mag[p] = mag[p + 1];
        sval[p] = sval[p + 1];
        idx[p] = idx[p + 1];
      } else if (here) {
        mag[p] = a;
        sval[p] = v;
        idx[p] = j;
      }
    }
    if (better(a, j, mag[MAXT - 1], idx[MAXT - 1])) {
      mag[MAXT - 1] = a;
      sval[MAXT - 1] = v;
      idx[MAXT - 1] = j;
    }
  }
  // Emit slots [0, t) in ascending column order.
  __device__ __forceinline__ void emit_sorted(int t, int32_t* col, float* val, float sd) const {
#pragma unroll
    for (int a = 0; a < MAXT; ++a) {
      if (a < t) {
        int rank = 0;
#pragma unroll
        for (int b = 0; b < MAXT; ++b)
          if (b < t && idx[b] < idx[a]) ++rank;
        col[rank] = idx[a];
        val[rank] = sval[a] * sd;
      }
    }
  }
};

__device__ __forceinline__ float max32_abs(const float (&v)[32]) {
  // four independent chains over columns j, j+4, ..., j+28 (pairs fuse into FMNMX3)
  float m0 = fabsf(v[0]), m1 = fabsf(v[1]), m2 = fabsf(v[2]), m3 = fabsf(v[3]);
#pragma unroll
  for (int e = 4; e < 28; e += 8) {
    m0 = fmaxf(m0, fmaxf(fabsf(v[e + 0]), fabsf(v[e + 4])));
    m1 = fmaxf(m1, fmaxf(fabsf(v[e + 1]), fabsf(v[e + 5])));
    m2 = fmaxf(m2, fmaxf(fabsf(v[e + 2]), fabsf(v[e + 6])));
    m3 = fmaxf(m3, fmaxf(fabsf(v[e + 3]), fabsf(v[e + 7])));
  }
  m0 = fmaxf(m0, fabsf(v[28]));
  m1 = fmaxf(m1, fabsf(v[29]));
  m2 = fmaxf(m2, fabsf(v[30]));
  m3 = fmaxf(m3, fabsf(v[31]));
  return fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
}

// Column sums of |v| over the warp's 32 rows for its 32 columns (reduce-scatter transpose:
// 31 shuffles); lane L returns the sum of column L.  Masked entries (bit e of ex) count 0.
// The absolute values are folded into the first stage's adds (FADD |a| + |b|), and the
// masking select runs only for lanes with masked entries (diagonal / padding tiles).
__device__ __forceinline__ float col_abs_sums32(const uint32_t (&vr)[32], uint32_t ex, int lane) {
  float v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(vr[e]);
  if (ex != 0u) {
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = ((ex >> e) & 1u) ? 0.f : v[e];
  }
  float a[16];
  {
    const bool up = (lane & 16) != 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float keep = up ? v[e + 16] : v[e];
      const float send = up ? v[e] : v[e + 16];
      a[e] = fabsf(keep) + fabsf(__shfl_xor_sync(0xffffffffu, send, 16));
    }
  }
#pragma unroll
  for (int st = 8; st >= 1; st >>= 1) {
    const bool up = (lane & st) != 0;
#pragma unroll
    for (int e = 0; e < st; ++e) {
      const float keep = up ? a[e + st] : a[e];
      const float send = up ? a[e] : a[e + st];
      a[e] = keep + __shfl_xor_sync(0xffffffffu, send, st);
    }
  }
  return a[0];
}

// An epilogue warp is done with a TMEM accumulator buffer: arrive on the (pair leader's)
// tempty barrier.
// The data was already waited into registers (tcgen05.wait::ld), so the arrive needs no
// cluster-scope release fence: the leader's own warps arrive locally, the peer's remotely.
template <bool PAIR>
__device__ __forceinline__ void release_tmem(uint64_t* bar) {
  if (PAIR && cluster_ctarank() != 0)
    mbar_arrive_cluster(bar, 0);
  else
    mbar_arrive(bar);
}

// One 32-row x 32-column chunk of the accumulator (thread = row, 32 columns in registers).
// Fast path: one FMNMX3 chain of |v| against the row's current t-th magnitude (and, kSym, the
// exact per-column test |ψ_ij| >= bound_j for the transposed direction).  Rare paths walk
// the warp-union of the hit columns in ascending order and re-read each such column from
// TMEM (tcgen05.ld 32x32b.x1: every lane gets its own row's value), so no register array is
// ever indexed dynamically and no shared-memory staging is needed.
struct CandCursor {
  int64_t base, used;  // current reservation [base, base + kCandChunk) of the pool
};
// Marks the unused tail of the warp's reservation (key UINT32_MAX sorts after every row), so
// the pool needs no up-front fill: the host sorts only the reserved prefix [0, cand_alloc).
// A cursor without a live reservation (initial, or pool exhausted) has used == kCandChunk.
__device__ __forceinline__ void close_chunk(const FusedParams& p, const CandCursor& cc, int lane) {
  for (int64_t q = cc.base + cc.used + lane; q < cc.base + kCandChunk; q += 32)
    p.cand_key[q] = 0xFFFFFFFFu;
}
template <int MAXT, int KIND>
__device__ __forceinline__ void epi_chunk(const FusedParams& p, const uint32_t (&vr)[32],
                                          uint32_t tchunk, int64_t col0, int64_t gi, int64_t lr,
                                          bool valid, bool need_mask, float tau_s, float sd2,
                                          TopList<MAXT>& top, double& macc, int lane,
                                          float* hist_smem, float* colacc = nullptr) {
  // the loaded registers are only read (never rewritten), so the compiler keeps them in the
  // tcgen05.ld destination block without copies
  float m = max32_abs(reinterpret_cast<const float(&)[32]>(vr));
  uint32_t excl = 0;  // diagonal (j == i: not an edge, Q8) and padding columns (j >= n)
  if (need_mask) {
    const int64_t dd = gi - col0;
    if ((uint64_t)dd < 32ull) excl |= 1u << dd;
    const int64_t nn = p.n - col0;
    if (nn < 32) excl |= nn <= 0 ? 0xffffffffu : (0xffffffffu << nn);
    m = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e)
      m = fmaxf(m, ((excl >> e) & 1u) ? 0.f : fabsf(__uint_as_float(vr[e])));
  }
  if (p.mode == 2) {  // row mass (degree down-weighting): Σ |ψ_ij| over j != i, j < n
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e) sum += ((excl >> e) & 1u) ? 0.f : fabsf(__uint_as_float(vr[e]));
    macc += (double)sum;
    if (KIND == kSymList && colacc != nullptr) {  // off-diagonal tile: also the columns' mass
      const float cs = col_abs_sums32(vr, valid ? excl : 0xffffffffu, lane);
      atomicAdd(colacc + lane, cs);
    }
    return;
  }
  if (p.mode == 3) {  // log-bucket histogram of upper-triangle |ψ| > τ (overall rules)
    if (__any_sync(0xffffffffu, m > tau_s) && valid) {
      const int64_t dd = gi - col0;  // columns e <= dd are j <= i
      const uint32_t low = dd < 0 ? 0u : (dd >= 31 ? 0xffffffffu : ((2u << dd) - 1u));
      const uint32_t ex = excl | low;
      unsigned int* hist = reinterpret_cast<unsigned int*>(hist_smem);
      const uint32_t tb = __float_as_uint(tau_s);
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float x = fabsf(__uint_as_float(vr[e]));
        if (!((ex >> e) & 1u) && x > tau_s)
          atomicAdd(hist + min(255u, (__float_as_uint(x) - tb) >> p.hshift), 1u);
      }
    }
    return;
  }
  const float thr = p.mode == 0 ? top.thr() : tau_s;
  if (__any_sync(0xffffffffu, m > thr)) {
    uint32_t mask = 0;
#pragma unroll
    for (int e = 0; e < 32; ++e) mask |= (fabsf(__uint_as_float(vr[e])) > thr ? 1u : 0u) << e;
    mask &= ~excl;
    if (p.mode == 0) {
      // visit this row's candidates in column order (ties -> smaller j, Q9)
      uint32_t um = __reduce_or_sync(0xffffffffu, mask);
      while (um) {
        const int e = __ffs(um) - 1;
        um &= um - 1;
        const float x = __uint_as_float(tmem_ld1(tchunk + e));
        if ((mask >> e) & 1u) {
          const float a = fabsf(x);
          if (a > top.thr()) top.insert(a, x, (int)(col0 + e));
        }
      }
    } else {
      if (!valid) mask = 0;
      const int cnt = __popc(mask);
      const int total = __reduce_add_sync(0xffffffffu, cnt);
      unsigned long long b0 = 0;
      if (lane == 0 && total) b0 = atomicAdd(p.coo_count, (unsigned long long)total);
      int64_t at = (int64_t)__shfl_sync(0xffffffffu, b0, 0);
      uint32_t um = __reduce_or_sync(0xffffffffu, mask);
      const uint32_t lt = (1u << lane) - 1u;
      while (um) {
        const int e = __ffs(um) - 1;
        um &= um - 1;
        const float x = __uint_as_float(tmem_ld1(tchunk + e));
        const bool mine = (mask >> e) & 1u;
        const uint32_t bm = __ballot_sync(0xffffffffu, mine);
        const int64_t pos = at + __popc(bm & lt);
        if (mine && pos < p.capacity) {
          p.coo_key[pos] = lr * p.n + col0 + e;
          p.coo_val[pos] = x * sd2;
        }
        at += __popc(bm);
      }
    }
  }
}

// Epilogue role (8 warps), list form (kPlain, kSeed): TMEM -> registers, fused per-row
// top-t / threshold.  Warp w handles TMEM lane quadrant q = w & 3 (thread = row) and column
// half h of every 256-column tile, i.e. one 128-column operand block = 4 chunks of 32
// columns, loaded with tcgen05.ld.32x32b.x32 into two alternating register buffers (the next
// chunk's load is in flight while the current one is reduced).  Two warps share each row;
// their lists are merged through shared memory at the end of a unit.
template <int MAXT, int KIND, bool PAIR>
__device__ __forceinline__ void epilogue_role(const FusedParams& p, uint32_t tmem_base,
                                              uint64_t* tfull, uint64_t* tempty, int warp,
                                              int lane, float* scratch_all, int u0, int ustep,
                                              int rank) {
  const int ew = warp - kFirstEpiWarp;  // 0..7; slot of (quadrant q, half h) = h*4 + ((q-first)&3)
  const int q = warp & 3;   // TMEM lane quadrant accessible to this warp
  const int h = ew >> 2;    // column half of each tile
  const int r = q * 32 + lane;
  const float sd = ldexpf(1.f, -p.sc->exp2);  // ψ = acc · 2^-e · 2^-e
  const float sd2 = sd * sd;
  const float tau_s = ldexpf(ldexpf(p.tau, p.sc->exp2), p.sc->exp2);
  const int t = p.t;
  int buf = 0;
  uint32_t tphase = 0;
  TopList<MAXT> top;
  if (p.mode == 3) {  // CTA histogram in the (otherwise unused) merge scratch
    for (int b = ew * 32 + lane; b < 256; b += 256) reinterpret_cast<unsigned int*>(scratch_all)[b] = 0u;
    asm volatile("bar.sync 5, 256;" ::: "memory");
  }
  // kSymList mass: column-sum accumulators [tile parity][half][128] in the merge scratch
  constexpr bool kColMass = KIND == kSymList;
  if (kColMass) {
    for (int b = ew * 32 + lane; b < 512; b += 256) scratch_all[b] = 0.f;
    asm volatile("bar.sync 5, 256;" ::: "memory");
  }
  int tpar = 0;
  for (int uj = u0; uj < unit_count<KIND>(p); uj += ustep) {
    const int u = unit_of<KIND>(p, uj);
    int ub;
    const int ntiles = unit_tiles<KIND, PAIR>(p, u, ub);
    const int rb = PAIR ? 2 * ub + rank : ub;  // this CTA's 128-row block

    const int64_t lr = (int64_t)rb * kRowsPerBlock + r;
    const bool valid = lr < p.rows;
    const int64_t gi = p.row_begin + lr;
    // global rows of this unit [rlo, rhi): tiles whose columns meet them hold the diagonal
    const int64_t rlo = p.row_begin + (int64_t)rb * kRowsPerBlock;
    const int64_t rhi = rlo + kRowsPerBlock;
    top.init(t);
    double macc = 0.0;
    TileIter<KIND, PAIR> ti;
    ti.start(p, u, uj, ub, u0, ustep);
    for (int s = 0; s < ntiles; ++s, ti.next(p)) {
      const int Kh = h ? ti.K1 : ti.K0;
      const bool live = (h == 0 || ti.h1) && GGM_DBG(p) != 2;
      const int64_t cb = (int64_t)Kh * kRowsPerBlock;  // first column of this warp's block
      const bool need_mask = (cb < rhi && cb + kRowsPerBlock > rlo) || (cb + kRowsPerBlock > p.n);
      mbar_wait(&tfull[buf], tphase);
      tc_fence_after();
      const uint32_t taddr =
          tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kTileN + h * (kTileN / 2));
      // kSymList: column sums only off the diagonal (super) block, whose tile holds both
      // (i, j) and (j, i)
      const bool diag_blk = PAIR ? (Kh >> 1) == ub : Kh == ub;
      float* cacc = (kColMass && p.mode == 2 && !diag_blk) ? scratch_all + (tpar * 2 + h) * 128 : nullptr;
      if (live) {
        uint32_t va[32], vb[32];
        tmem_ld32_nowait(taddr, va);
#pragma unroll 1
        for (int c = 0; c < (kTileN / 2) / 32; c += 2) {
          tmem_wait_ld(va);
          tmem_ld32_nowait(taddr + (c + 1) * 32, vb);
          if (GGM_DBG(p) != 1)
            epi_chunk<MAXT, KIND>(p, va, taddr + c * 32, cb + c * 32, gi, lr, valid, need_mask,
                                  tau_s, sd2, top, macc, lane, scratch_all,
                                  cacc ? cacc + c * 32 : nullptr);
          else if (va[0] == 12345u && va[31] == 54321u)
            p.row_ptr[0] = (int64_t)va[7];
          tmem_wait_ld(vb);
          if (c + 2 < (kTileN / 2) / 32) tmem_ld32_nowait(taddr + (c + 2) * 32, va);
          if (GGM_DBG(p) != 1)
            epi_chunk<MAXT, KIND>(p, vb, taddr + (c + 1) * 32, cb + (c + 1) * 32, gi, lr, valid,
                                  need_mask, tau_s, sd2, top, macc, lane, scratch_all,
                                  cacc ? cacc + (c + 1) * 32 : nullptr);
          else if (vb[0] == 12345u && vb[31] == 54321u)
            p.row_ptr[0] = (int64_t)vb[7];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) release_tmem<PAIR>(&tempty[buf]);
      if (++buf == 2) {
        buf = 0;
        tphase ^= 1;
      }
      if (kColMass && p.mode == 2) {
        // the 4 quadrant warps of this half have added their column sums: one warp flushes
        // (and clears) them; the other parity buffer takes the next tile meanwhile
        asm volatile("bar.sync %0, 128;" ::"r"(6 + h) : "memory");
        if (q == 0 && live && !diag_blk) {
          float* acc = scratch_all + (tpar * 2 + h) * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int64_t j = cb + c * 32 + lane;
            const float v = acc[c * 32 + lane];
            acc[c * 32 + lane] = 0.f;
            if (j < p.n && v != 0.f) atomicAdd(p.mass_out + j, (double)v);
          }
        }
        tpar ^= 1;
      }
    }
    if (p.mode == 2) {  // both column halves add their partial row mass (accumulator units)
      if (valid) atomicAdd(p.mass_out + lr, macc);
      continue;
    }
    if (p.mode != 0) continue;  // modes 1, 3: nothing per row
    // merge the two column halves of each row: half 1 publishes (values into its own
    // scratch, columns into the half-0 warp's), half 0 merges and emits.
    float* pv = scratch_all + (4 + ((q - kFirstEpiWarp) & 3)) * kScratchFloats;
    float* pc = scratch_all + ((q - kFirstEpiWarp) & 3) * kScratchFloats;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
    if (h == 1) {
#pragma unroll
      for (int a = 0; a < MAXT; ++a) {
        pv[a * 32 + lane] = top.sval[a];
        pc[a * 32 + lane] = __int_as_float(top.idx[a]);
      }
    }
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
    if (h == 0) {
#pragma unroll 1
      for (int a = 0; a < t; ++a) {
        const float x = pv[a * 32 + lane];
        const int jx = __float_as_int(pc[a * 32 + lane]);
        if (jx >= 0) top.merge_insert(fabsf(x), x, jx);
      }
      if (valid) {
        if (KIND == kSeed) {
          p.thr_out[lr] = top.thr();  // t-th largest sampled magnitude (-1: fewer than t)
        } else if (KIND == kPlain && p.C == 1) {
          // the list is full (t <= n-1 real columns scanned); emit in ascending column
          top.emit_sorted(t, p.col + lr * t, p.val + lr * t, sd2);
          p.row_ptr[lr] = lr * t;
          if (lr == p.rows - 1) p.row_ptr[p.rows] = p.rows * t;
        } else {
          const int cc2 = KIND == kPlain ? u % p.C : 0;
          const int64_t base = ((int64_t)cc2 * p.rows + lr) * t;
#pragma unroll
          for (int a = 0; a < MAXT; ++a) {
            if (a < t) {
              p.pcol[base + a] = top.idx[a];
              p.pval[base + a] = top.sval[a] * sd2;
            }
          }
        }
      }
    }
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
  }
  if (p.mode == 3) {
    asm volatile("bar.sync 5, 256;" ::: "memory");
    const unsigned int* hist = reinterpret_cast<const unsigned int*>(scratch_all);
    for (int b = ew * 32 + lane; b < 256; b += 256)
      if (hist[b]) atomicAdd(p.hist_out + b, (unsigned long long)hist[b]);
  }
}

// Epilogue role of the seed pass (kSeed): per row, the t-th largest of the 32-column chunk
// maxima of |hi·hi| over the sampled column tiles.  t chunk maxima are t distinct entries,
// so this is a lower bound of the row's t-th magnitude in the same arithmetic (converted to
// a bound on the 3-term values by seed_bounds).  Magnitude-only list, one predicated insert
// of the chunk maximum per lane: no per-entry work beyond the FMNMX3 chain.
template <int MAXT>
struct MagList {
  float m[MAXT];  // ascending; slots >= t hold +inf
  __device__ __forceinline__ void init(int t) {
#pragma unroll
    for (int p = 0; p < MAXT; ++p) m[p] = (p < t) ? -1.f : __int_as_float(0x7f800000);
  }
  __device__ __forceinline__ void insert(float a) {
#pragma unroll
    for (int p = 0; p < MAXT - 1; ++p) m[p] = a > m[p + 1] ? m[p + 1] : (a > m[p] ? a : m[p]);
    if (a > m[MAXT - 1]) m[MAXT - 1] = a;
  }
};
// Epilogue geometry for EPW warps: warp (quadrant q = warp & 3, part) reads TMEM lanes
// 32q..32q+31 and columns [part*W, part*W + W) of each 256-column tile, W = 256 / (EPW/4),
// i.e. NC = W/32 chunks; those columns are operand block (part*W)/128 (K0 or K1) from column
// offset (part*W) % 128.
template <int EPW>
struct EpiGeom {
  static constexpr int P = EPW / 4;        // warps per quadrant
  static constexpr int W = kTileN / P;     // columns per warp per tile
  static constexpr int NC = W / 32;        // 32-column chunks per warp per tile
  int q, part, r;
  __device__ __forceinline__ EpiGeom(int warp, int lane) {
    const int ew = warp - kFirstEpiWarp;
    q = warp & 3;
    part = ew >> 2;
    r = q * 32 + lane;
  }
  __device__ __forceinline__ bool second() const { return part * W >= 128; }
  __device__ __forceinline__ int col_off() const { return (part * W) & 127; }
};

template <int MAXT, bool PAIR, int EPW>
__device__ __forceinline__ void epilogue_seed(const FusedParams& p, uint32_t tmem_base,
                                              uint64_t* tfull, uint64_t* tempty, int warp,
                                              int lane, float* scratch_all, int u0, int ustep,
                                              int rank) {
  using G = EpiGeom<EPW>;
  const G g(warp, lane);
  const int t = p.t;
  int buf = 0;
  uint32_t tphase = 0;
  MagList<MAXT> top;
  for (int uj = u0; uj < unit_count<kSeed>(p); uj += ustep) {
    const int u = unit_of<kSeed>(p, uj);
    int ub;
    const int ntiles = unit_tiles<kSeed, PAIR>(p, u, ub);
    const int rb = PAIR ? 2 * ub + rank : ub;
    const int64_t gi = (int64_t)rb * kRowsPerBlock + g.r;
    top.init(t);
    TileIter<kSeed, PAIR> ti;
    ti.start(p, u, uj, ub, u0, ustep);
    for (int s = 0; s < ntiles; ++s, ti.next(p)) {
      const int Kh = g.second() ? ti.K1 : ti.K0;
      const int64_t cb = (int64_t)Kh * kRowsPerBlock + g.col_off();
      const bool need_mask = Kh == rb || cb + G::W > p.n;
      mbar_wait(&tfull[buf], tphase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(g.q * 32) << 16) +
                             (uint32_t)(buf * kTileN + g.part * G::W);
      uint32_t v[G::NC][32];
#ifndef GGM_EPI_LD32
      if constexpr (G::NC == 2) {  // one x64 load (as the candidate epilogue)
        tmem_ld64_nowait(taddr, v[0], v[G::NC - 1]);
      } else {
#pragma unroll
        for (int c = 0; c < G::NC; ++c) tmem_ld32_nowait(taddr + c * 32, v[c]);
      }
#else
#pragma unroll
      for (int c = 0; c < G::NC; ++c) tmem_ld32_nowait(taddr + c * 32, v[c]);
#endif
#pragma unroll
      for (int c = 0; c < G::NC; ++c) tmem_wait_ld(v[c]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) release_tmem<PAIR>(&tempty[buf]);
      if (++buf == 2) {
        buf = 0;
        tphase ^= 1;
      }
      if (GGM_DBG(p) != 0) {
        if (v[0][0] == 12345u && v[G::NC - 1][31] == 54321u) p.thr_out[0] = __uint_as_float(v[0][7]);
        continue;
      }
#pragma unroll
      for (int c = 0; c < G::NC; ++c) {
        float m = max32_abs(reinterpret_cast<const float(&)[32]>(v[c]));
        if (need_mask) {
          const int64_t col0 = cb + c * 32;
          m = 0.f;
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (col0 + e != gi && col0 + e < p.n) m = fmaxf(m, fabsf(__uint_as_float(v[c][e])));
        }
        if (m > top.m[0]) top.insert(m);
      }
    }
    // merge the quadrant's P lists: parts 1..P-1 publish, part 0 inserts and writes
    float* slot = scratch_all + (size_t)(warp - kFirstEpiWarp) * (kScratchBytes / 4 / EPW);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g.q), "r"(32 * G::P) : "memory");
    if (g.part != 0) {
#pragma unroll
      for (int a = 0; a < MAXT; ++a) slot[a * 32 + lane] = top.m[a];
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g.q), "r"(32 * G::P) : "memory");
    if (g.part == 0) {
      for (int pp = 1; pp < G::P; ++pp) {
        const float* o = scratch_all + (size_t)(warp - kFirstEpiWarp + 4 * pp) * (kScratchBytes / 4 / EPW);
#pragma unroll 1
        for (int a = 0; a < t; ++a) {
          const float x = o[a * 32 + lane];
          if (x > top.m[0]) top.insert(x);
        }
      }
      if (gi < p.n) p.thr_out[gi] = top.m[0];  // -1: fewer than t chunks sampled
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g.q), "r"(32 * G::P) : "memory");
  }
}

// Per-lane register select v[e] for a lane-varying e (binary tree of 31 selects; a dynamic
// index into a register array would go through local memory).
__device__ __forceinline__ float sel32(const uint32_t* v, uint32_t e) {
  uint32_t a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = (e & 16u) ? v[i + 16] : v[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (e & 8u) ? a[i + 8] : a[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = (e & 4u) ? a[i + 4] : a[i];
#pragma unroll
  for (int i = 0; i < 2; ++i) a[i] = (e & 2u) ? a[i + 2] : a[i];
  return __uint_as_float((e & 1u) ? a[1] : a[0]);
}

// Epilogue role of the row-mass pass (kSymList, mode 2; degree down-weighting of the overall
// rules): w_i = Σ_{j≠i} |ψ_ij| over each unordered block pair (I, J) computed once —
// row sums of the tile into rows I (in-thread, registers), column sums into rows J (off the
// diagonal block) by a reduce-scatter transpose per 32x32 chunk, the four quadrant warps of a
// column slice combined in shared memory, one fp64 red per column per tile.  16 warps (4 per
// lane quadrant, 64 columns each); the TMEM buffer is released as soon as the warp's last
// chunk is in registers, before its sums run.
template <bool PAIR, int EPW>
__device__ __forceinline__ void epilogue_mass(const FusedParams& p, uint32_t tmem_base,
                                              uint64_t* tfull, uint64_t* tempty, int warp,
                                              int lane, float* scratch_all, int u0, int ustep,
                                              int rank) {
  using G = EpiGeom<EPW>;
  const G g(warp, lane);
  const int lq = lane & 3, lg = lane >> 2;  // 16x256b fragment coordinates
  const int64_t n = p.n;
  const uint32_t trow = tmem_base + ((uint32_t)(g.q * 32) << 16) + (uint32_t)(g.part * G::W);
  const int coff = g.col_off();
  const bool second = g.second();
  const uint32_t tfull_a0 = smem_u32(&tfull[0]), tfull_a1 = smem_u32(&tfull[1]);
  const bool remote_rel = PAIR && rank != 0;
  const uint32_t tempty_a0 = remote_rel ? mbar_map_cluster(&tempty[0], 0) : smem_u32(&tempty[0]);
  const uint32_t tempty_a1 = remote_rel ? mbar_map_cluster(&tempty[1], 0) : smem_u32(&tempty[1]);
  // column-sum partials: [tile parity][part][quadrant][G::W] floats, plain stores (every
  // live off-diagonal tile overwrites its slot), combined after the part's barrier
  int buf = 0, tpar = 0;
  uint32_t tphase = 0;
  for (int uj = u0; uj < unit_count<kSymList>(p); uj += ustep) {
    const int u = unit_of<kSymList>(p, uj);
    int ub;
    const int ntiles = unit_tiles<kSymList, PAIR>(p, u, ub);
    const int rb = PAIR ? 2 * ub + rank : ub;
    // this thread's rows (16x256b layout): lr = rbase + lg + 8 j; its row-sum row: j = lq
    const int64_t rbase = (int64_t)rb * kRowsPerBlock + g.q * 32;
    const bool rows_valid = rbase + 32 <= p.rows;
    const int64_t lr = rbase + lg + 8 * lq;
    const bool valid = lr < p.rows;
    double macc = 0.0;
    float racc = 0.f;  // row sums of up to 16 tiles (fp32), then into macc (fp64)
    TileIter<kSymList, PAIR> ti;
    ti.start(p, u, uj, ub, u0, ustep);
    for (int s = 0; s < ntiles; ++s) {
      const int Kh = second ? ti.K1 : ti.K0;
      const bool live = !second || ti.h1;
      // the diagonal (super) block holds both (i, j) and (j, i): row sums only
      const bool diag_blk = PAIR ? (ti.K0 >> 1) == ub : Kh == rb;
      const int64_t cb = (int64_t)Kh * kRowsPerBlock + coff;
      const int64_t gr0 = p.row_begin + rbase;  // the warp's rows: [gr0, gr0 + 32)
      const bool need_mask = (gr0 < cb + G::W && cb < gr0 + 32) || cb + G::W > n;
      ti.next(p);
      mbar_wait_a(buf ? tfull_a1 : tfull_a0, tphase);
      tc_fence_after();
      const uint32_t taddr = trow + (uint32_t)(buf * kTileN);
      const uint32_t cur = buf;
      buf ^= 1;
      tphase ^= (uint32_t)(buf == 0);
      float* cpart = scratch_all + (size_t)(tpar * G::P + g.part) * 4 * G::W;  // [quadrant][W]
#pragma unroll
      for (int c = 0; c < G::NC; ++c) {
        // 32 rows x 32 columns in the 16x256b layout (two 16-lane loads): this thread holds
        // rows lg + 8j (j = 0..3; v[16(j >> 1) + 4cg + 2(j & 1) + b]) at columns
        // 8cg + 2lq + b (cg = 0..3, b = 0..1), so both the row and the column sums start
        // with thread-local adds and end in short reduce-scatters (3 + 7 shuffles instead of
        // the 31-shuffle transpose of the 32x32b layout)
        uint32_t v[32];
        if (live) {
          tmem_ld16x256_x4_nowait(taddr + c * 32, v);
          tmem_ld16x256_x4_nowait(taddr + ((uint32_t)16 << 16) + c * 32, v + 16);
          tmem_wait_ld(v);
        }
        if (c == G::NC - 1) {  // the warp's slice is in registers: release the buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            const uint32_t ta = cur ? tempty_a1 : tempty_a0;
            if (remote_rel)
              mbar_arrive_cluster_a(ta);
            else
              mbar_arrive_a(ta);
          }
        }
        if (!live) continue;
        const int64_t col0 = cb + c * 32;
        if (need_mask || !rows_valid) {
          // diagonal (j == i, not an edge: Q8), padding columns (j >= n), rows past the axis
#pragma unroll
          for (int x = 0; x < 32; ++x) {
            const int j = 2 * (x >> 4) + ((x >> 1) & 1);
            const int64_t col = col0 + 8 * ((x >> 2) & 3) + 2 * lq + (x & 1);
            const int64_t lrj = rbase + lg + 8 * j;
            if (col == p.row_begin + lrj || col >= n || lrj >= p.rows) v[x] = 0u;
          }
        }
        float rs[4], cs8[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int o = 16 * (j >> 1) + 2 * (j & 1);
          float a = fabsf(__uint_as_float(v[o])) + fabsf(__uint_as_float(v[o + 1]));
#pragma unroll
          for (int cg = 1; cg < 4; ++cg)
            a += fabsf(__uint_as_float(v[o + 4 * cg])) + fabsf(__uint_as_float(v[o + 4 * cg + 1]));
          rs[j] = a;
        }
#pragma unroll
        for (int cg = 0; cg < 4; ++cg)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int o = 4 * cg + b;
            cs8[2 * cg + b] = (fabsf(__uint_as_float(v[o])) + fabsf(__uint_as_float(v[o + 2]))) +
                              (fabsf(__uint_as_float(v[o + 16])) + fabsf(__uint_as_float(v[o + 18])));
          }
        {  // row sums: reduce-scatter over lq (lanes ^2, ^1) -> this lane: row lg + 8 lq
          const bool up2 = (lq & 2) != 0;
          float a0 = (up2 ? rs[2] : rs[0]) + __shfl_xor_sync(0xffffffffu, up2 ? rs[0] : rs[2], 2);
          float a1 = (up2 ? rs[3] : rs[1]) + __shfl_xor_sync(0xffffffffu, up2 ? rs[1] : rs[3], 2);
          const bool up1 = (lq & 1) != 0;
          const float r = (up1 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, up1 ? a0 : a1, 1);
          racc += r;
        }
        if (!diag_blk) {  // column sums: reduce-scatter over lg (lanes ^16, ^8, ^4)
          float a4[4];
          const bool u16 = (lg & 4) != 0;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            a4[e] = (u16 ? cs8[e + 4] : cs8[e]) + __shfl_xor_sync(0xffffffffu, u16 ? cs8[e] : cs8[e + 4], 16);
          const bool u8 = (lg & 2) != 0;
          float a2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e)
            a2[e] = (u8 ? a4[e + 2] : a4[e]) + __shfl_xor_sync(0xffffffffu, u8 ? a4[e] : a4[e + 2], 8);
          const bool u4 = (lg & 1) != 0;
          const float cs = (u4 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, u4 ? a2[0] : a2[1], 4);
          // this lane: column 8 (lg >> 1) + 2 lq + (lg & 1) of the chunk
          cpart[g.q * G::W + c * 32 + 8 * (lg >> 1) + 2 * lq + (lg & 1)] = cs;
        }
      }
      if ((s & 15) == 15) {
        macc += (double)racc;
        racc = 0.f;
      }
      if (!diag_blk && live) {
        // the part's 4 quadrant warps have stored their column partials: each warp combines
        // and flushes 16 of the part's W columns (balanced; no shared-memory atomics); the
        // other parity slice takes the next tile meanwhile
        asm volatile("bar.sync %0, 128;" ::"r"(8 + g.part) : "memory");
        constexpr int CPW = G::W / 4;  // columns flushed per warp
        for (int cc = lane; cc < CPW; cc += 32) {
          const int col = g.q * CPW + cc;
          const float x = (cpart[col] + cpart[G::W + col]) + (cpart[2 * G::W + col] + cpart[3 * G::W + col]);
          const int64_t j = cb + col;
          if (j < n && x != 0.f) atomicAdd(p.mass_out + j, (double)x);
        }
        // the slot parity alternates between barrier tiles only: a slot is rewritten two
        // barriers after it was read (a diagonal tile in between has no barrier)
        tpar ^= 1;
      }
    }
    if (valid) atomicAdd(p.mass_out + lr, macc + (double)racc);  // every column slice adds its part
  }
}

// Epilogue role, candidate form (kSym): every row i carries a lower bound b_i of its t-th
// magnitude (the seed pass); rows and columns are in bound order.  Entry ψ_ij of a tile is
// emitted as a candidate of row i if |ψ| >= b_i (row direction) and, for off-diagonal
// blocks, of row j if |ψ| >= min of the bounds of j's 8-column group (transposed direction,
// each unordered block pair being evaluated once; a superset of |ψ| >= b_j, GGM_CMASK_W).  No per-row list is kept: the whole 128-column block of the warp is
// loaded into registers and the TMEM buffer released before the filter runs; a final merge
// selects each row's top t among its candidates.  Fast path per 32 columns: one FMNMX3
// chain + two compares (row bound; chunk minimum of the column bounds).
template <int KIND, bool PAIR, int EPW>
__device__ __forceinline__ void epilogue_emit(const FusedParams& p, uint32_t tmem_base,
                                              uint64_t* tfull, uint64_t* tempty, int warp,
                                              int lane, float* scratch_all, int u0, int ustep,
                                              int rank) {
  // Per tile and warp the work is: wait for the accumulator, load the warp's W columns,
  // release the buffer, one FMNMX3 chain per 32 columns against min(row bound, the
  // precomputed minimum of the chunk's column bounds).  Everything else is hoisted: column
  // bounds are read from global memory only on the rare path, indices are 32-bit
  // (n < 2^31), and the per-chunk minima come from p.thr_min (one broadcast load).
  using G = EpiGeom<EPW>;
  const G g(warp, lane);
  (void)scratch_all;
#ifdef GGM_EPI_DEBUG
  const int dbg = p.dbg;  // 1: skip the filter, 2: skip TMEM loads, 3: no rare path
#else
  constexpr int dbg = 0;
#endif
  const float sd = ldexpf(1.f, -p.sc->exp2);
  const float sd2 = sd * sd;
  const uint32_t lt = (1u << lane) - 1u;
  DevScalars* scw = const_cast<DevScalars*>(p.sc);
  const int n = (int)p.n;
  const float* __restrict__ thr = p.thr;
  const float* __restrict__ thr_min = p.thr_min;
  const uint32_t trow = tmem_base + ((uint32_t)(g.q * 32) << 16) + (uint32_t)(g.part * G::W);
  const int coff = g.col_off();
  const bool second = g.second();
  // barrier addresses of both accumulator buffers, computed once: tfull is waited on
  // locally; tempty lives in the pair leader (remote arrive from the peer CTA)
  const uint32_t tfull_a0 = smem_u32(&tfull[0]), tfull_a1 = smem_u32(&tfull[1]);
  const bool remote_rel = PAIR && rank != 0;
  const uint32_t tempty_a0 = remote_rel ? mbar_map_cluster(&tempty[0], 0) : smem_u32(&tempty[0]);
  const uint32_t tempty_a1 = remote_rel ? mbar_map_cluster(&tempty[1], 0) : smem_u32(&tempty[1]);
  int buf = 0;
  uint32_t tphase = 0;
  CandCursor cc{0, kCandChunk};
  unsigned long long emitted = 0;  // candidates this warp wrote (warp-uniform)
#ifdef GGM_MMA_PROF
  long long pe_t0 = clock64(), pe_w = 0, pe_n = 0;
#endif
  for (int uj = u0; uj < unit_count<KIND>(p); uj += ustep) {
    const int u = unit_of<KIND>(p, uj);
    int ub;
    const int ntiles = unit_tiles<KIND, PAIR>(p, u, ub);
    const int rb = PAIR ? 2 * ub + rank : ub;
    const int gi = rb * kRowsPerBlock + g.r;  // permuted row index
    const bool valid = gi < n;
    const float bi = valid ? __ldg(thr + gi) : INFINITY;  // row bound (accumulator units)
    TileIter<KIND, PAIR> ti;
    ti.start(p, u, uj, ub, u0, ustep);
    for (int s = 0; s < ntiles; ++s) {
      const int Kh = second ? ti.K1 : ti.K0;
      const bool live = (!second || ti.h1) && dbg != 2;
      // off-diagonal blocks emit the transposed direction; for a CTA pair, the diagonal
      // 256x256 super tile covers both directions of its blocks in the row direction
      const bool emit_cols = PAIR ? (ti.K0 >> 1) != ub : Kh != rb;
      const int cb = Kh * kRowsPerBlock + coff;
      const bool need_mask = Kh == rb || cb + G::W > n;
      ti.next(p);
      float cmin[G::NC];
#pragma unroll
      for (int c = 0; c < G::NC; ++c)
        cmin[c] = emit_cols ? __ldg(thr_min + (cb >> 5) + c) : INFINITY;
#if GGM_CMASK_W == 1
      // the tile's column bounds, one per lane and chunk (coalesced, before the wait): the
      // exact column mask broadcasts them with shuffles
      float thl[G::NC];
#pragma unroll
      for (int c = 0; c < G::NC; ++c) thl[c] = emit_cols ? __ldg(thr + cb + 32 * c + lane) : INFINITY;
#endif
#ifdef GGM_MMA_PROF
      const long long pe_c = clock64();
#endif
      mbar_wait_a(buf ? tfull_a1 : tfull_a0, tphase);
#ifdef GGM_MMA_PROF
      pe_w += clock64() - pe_c;
      ++pe_n;
#endif
      tc_fence_after();
      const uint32_t taddr = trow + (uint32_t)(buf * kTileN);
#ifndef GGM_EPI_STREAM
      // both 32-column chunks loaded back to back, one wait, then the buffer is released
      // before either filter runs (the streamed form — load, filter, load, release — holds
      // the buffer through the first chunk's filter: C4 main 3.80 vs 3.75 ms,
      // profiles/r02_logs/r02d_ab_epiblock.log)
      uint32_t v[G::NC][32];
      if (live) {
#ifndef GGM_EPI_LD32
        // one 32x32b.x64 load for the warp's 64 columns (C4 main 3.78 -> 3.74 ms against two
        // x32 loads, same session: profiles/r02_logs/r02ab_ld64.log)
        if constexpr (G::NC == 2) {
          tmem_ld64_nowait(taddr, v[0], v[G::NC - 1]);
        } else {
#pragma unroll
          for (int c = 0; c < G::NC; ++c) tmem_ld32_nowait(taddr + c * 32, v[c]);
        }
#else
#pragma unroll
        for (int c = 0; c < G::NC; ++c) tmem_ld32_nowait(taddr + c * 32, v[c]);
#endif
#pragma unroll
        for (int c = 0; c < G::NC; ++c) tmem_wait_ld(v[c]);
      }
      // the accumulator buffer is free as soon as the block is in registers
      tc_fence_before();
      __syncwarp();
      if (lane == 0) release_tmem<PAIR>(&tempty[buf]);
      buf ^= 1;
      tphase ^= (uint32_t)(buf == 0);
      if (!live || dbg == 1) {
        if (live && v[0][0] == 12345u && v[G::NC - 1][31] == 54321u) p.row_ptr[0] = (int64_t)v[0][7];
        continue;
      }
#define VC v[c]
#else
      // one 32-column chunk in registers at a time (32 value registers instead of W: no
      // rematerialisation at 96 registers/thread); the buffer is released as soon as the
      // last chunk is in registers, before its filter runs
      const uint32_t cur_buf = buf;
      buf ^= 1;
      tphase ^= (uint32_t)(buf == 0);
      auto release_cur = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          const uint32_t ta = cur_buf ? tempty_a1 : tempty_a0;
          if (remote_rel)
            mbar_arrive_cluster_a(ta);
          else
            mbar_arrive_a(ta);
        }
      };
      if (!live || dbg == 1) {
        release_cur();
        continue;
      }
#ifdef GGM_EPI_DEBUG
      // 5: dbg 3 except that the warps on the MMA issuer's sub-partition (warp % 4 == 1)
      //    only load and release (is the slowdown issue contention on that SMSP?)
      //    6: the same for quadrant 2 (control); 7: quadrant 1 of the leader CTA only;
      //    8: quadrant 3 of both CTAs
      if (dbg == 4 || (dbg == 5 && (warp & 3) == 1) || (dbg == 6 && (warp & 3) == 2) ||
          (dbg == 7 && (warp & 3) == 1 && rank == 0) || (dbg == 8 && (warp & 3) == 3)) {
        uint32_t vv[G::NC][32];
#pragma unroll
        for (int c = 0; c < G::NC; ++c) tmem_ld32_nowait(taddr + c * 32, vv[c]);
#pragma unroll
        for (int c = 0; c < G::NC; ++c) tmem_wait_ld(vv[c]);
        release_cur();
        if (vv[0][0] == 12345u && vv[G::NC - 1][31] == 54321u) p.row_ptr[0] = (int64_t)vv[0][7];
        continue;
      }
#endif
#define VC vc
#endif
#if !defined(GGM_EPI_STREAM) && !defined(GGM_EPI_VOTE_PER_CHUNK)
      // one vote for the warp's whole slice (both chunks' maxima, independent chains): the
      // common tile has no entry above any bound and leaves after a single __any_sync
      float mpre[G::NC];
      if (!need_mask) {
        bool hit = false;
#pragma unroll
        for (int c = 0; c < G::NC; ++c) {
          mpre[c] = max32_abs(reinterpret_cast<const float(&)[32]>(v[c]));
          hit |= mpre[c] >= bi || mpre[c] >= cmin[c];
        }
        if (!__any_sync(0xffffffffu, valid && hit)) continue;
      }
#endif
#pragma unroll
      for (int c = 0; c < G::NC; ++c) {
        const int col0 = cb + c * 32;
#ifdef GGM_EPI_STREAM
        uint32_t vc[32];
        tmem_ld32_nowait(taddr + c * 32, vc);
        tmem_wait_ld(vc);
        if (c == G::NC - 1) release_cur();  // the last chunk is in registers
#endif
#if !defined(GGM_EPI_STREAM) && !defined(GGM_EPI_VOTE_PER_CHUNK)
        float m = need_mask ? 0.f : mpre[c];
#else
        float m = max32_abs(reinterpret_cast<const float(&)[32]>(VC));
#endif
        uint32_t excl = 0;  // diagonal (Q8) and padding columns
        if (need_mask) {
          const int dd = gi - col0;
          if ((unsigned)dd < 32u) excl |= 1u << dd;
          const int nn = n - col0;
          if (nn < 32) excl |= nn <= 0 ? 0xffffffffu : (0xffffffffu << nn);
          m = 0.f;
#pragma unroll
          for (int e = 0; e < 32; ++e)
            m = fmaxf(m, ((excl >> e) & 1u) ? 0.f : fabsf(__uint_as_float(VC[e])));
        }
        const bool rh = valid && m >= bi;
        const bool ch = valid && m >= cmin[c];
        if (!__any_sync(0xffffffffu, rh || ch) || dbg >= 3) continue;  // dbg 3, 5: no rare path
        // rare path: exact per-entry masks, then each lane walks its own hits
        uint32_t mr = 0, mc = 0;
        if (rh) {
#pragma unroll
          for (int e = 0; e < 32; ++e) mr |= (fabsf(__uint_as_float(VC[e])) >= bi ? 1u : 0u) << e;
          mr &= ~excl;
        }
#if GGM_CMASK_W == 1
        if (__any_sync(0xffffffffu, ch)) {  // exact: entry (i, j) against bound b_j
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float th = __shfl_sync(0xffffffffu, thl[c], e);
            mc |= (ch && fabsf(__uint_as_float(VC[e])) >= th ? 1u : 0u) << e;
          }
          mc &= ~excl;
        }
#else
        if (ch) {
          // against the minimum bound of the entry's GGM_CMASK_W-column group (columns are in
          // bound order, so the groups' bounds are nearly equal): a superset of the exact
          // transposed-direction candidates, made exact by the re-evaluation and the merge
#if GGM_CMASK_W == 8
          const float4 g8 = __ldg(reinterpret_cast<const float4*>(p.thr_min8 + (col0 >> 3)));
#endif
#pragma unroll
          for (int e = 0; e < 32; ++e) {
#if GGM_CMASK_W == 8
            const float th = e < 8 ? g8.x : e < 16 ? g8.y : e < 24 ? g8.z : g8.w;
#else
            const float th = cmin[c];
#endif
            mc |= (fabsf(__uint_as_float(VC[e])) >= th ? 1u : 0u) << e;
          }
          mc &= ~excl;
        }
#endif
        const int total = __reduce_add_sync(0xffffffffu, __popc(mr) + __popc(mc));
        if (total == 0) continue;
        if (cc.used + total > kCandChunk) {  // reserve a fresh chunk of the pool
          close_chunk(p, cc, lane);
          unsigned long long b0 = 0;
          if (lane == 0) b0 = atomicAdd(&scw->cand_alloc, (unsigned long long)kCandChunk);
          cc.base = (int64_t)__shfl_sync(0xffffffffu, b0, 0);
          cc.used = 0;
          if (cc.base + kCandChunk > p.cand_total) {
            if (lane == 0) atomicOr(&scw->cand_overflow, 1);
            cc.used = kCandChunk;  // pool exhausted: the host recomputes exactly
          }
        }
        if (cc.used + total > kCandChunk) continue;
        int64_t at = cc.base + cc.used;
        cc.used += total;
        emitted += (unsigned long long)total;
        uint32_t mh = mr | mc;
        while (__any_sync(0xffffffffu, mh != 0)) {
          const uint32_t e = mh ? (uint32_t)(__ffs(mh) - 1) : 0u;
          const bool hr = mh && ((mr >> e) & 1u);
          const bool hc = mh && ((mc >> e) & 1u);
          const uint32_t br = __ballot_sync(0xffffffffu, hr);
          const uint32_t bc = __ballot_sync(0xffffffffu, hc);
          if (mh) {
            const uint32_t xb = p.cand_vals ? __float_as_uint(sel32(VC, e) * sd2) : 0u;
            if (hr) {  // candidate (i -> j): target row i
              const int64_t pos = at + __popc(br & lt);
              GGM_DCHECK(pos < p.cand_total && gi < n && col0 + (int)e < n);
              p.cand_key[pos] = (uint32_t)gi;
              p.cand_val[pos] = make_uint2((uint32_t)(col0 + (int)e), xb);
            }
            if (hc) {  // candidate (j -> i): target row j
              const int64_t pos = at + __popc(br) + __popc(bc & lt);
              GGM_DCHECK(pos < p.cand_total && gi < n && col0 + (int)e < n);
              p.cand_key[pos] = (uint32_t)(col0 + (int)e);
              p.cand_val[pos] = make_uint2((uint32_t)gi, xb);
            }
            mh &= mh - 1;
          }
          at += __popc(br) + __popc(bc);
        }
      }
    }
  }
  close_chunk(p, cc, lane);
  if (lane == 0 && emitted) atomicAdd(&scw->cand_emitted, emitted);
#ifdef GGM_MMA_PROF
  if (lane == 0 && (blockIdx.x & 15) == 0 && (warp == kFirstEpiWarp || warp == kFirstEpiWarp + EPW - 1))
    printf("EPIPROF cta %d warp %d tiles %lld total %lld wait_tfull %lld\n", (int)blockIdx.x, warp,
           pe_n, clock64() - pe_t0, pe_w);
#endif
}
#undef VC

// Epilogue warps per kind: 16 for the candidate and seed epilogues (t <= 10), else 8.
#ifndef GGM_SEED_EPW
#define GGM_SEED_EPW 16
#endif
#ifndef GGM_SYM_EPW
#define GGM_SYM_EPW 16
#endif
__host__ __device__ constexpr int epw_of(int KIND, int MAXT) {
  return KIND == kSym ? GGM_SYM_EPW
         : KIND == kSymList ? 16
         : (KIND == kSeed && MAXT <= 10) ? GGM_SEED_EPW : 8;
}

template <int MAXT, int KIND, bool PAIR, int EPW = epw_of(KIND, MAXT)>
__global__ void __launch_bounds__(threads_of(EPW), 1)
    fused_recon_topk(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, const FusedParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base (pointer arithmetic keeps the shared address space visible to the
  // compiler, so epilogue accesses through derived pointers compile to LDS/STS); the offset
  // is the same in both CTAs of a pair (same kernel, same dynamic smem size)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int KA = p.KA;
  const int resident = PAIR ? 1 : p.resident;
  const size_t a_bytes = resident ? block_bytes(KA) : 0;
  const size_t st_bytes = stage_bytes(resident, PAIR);
  uint8_t* sA = smem;
  uint8_t* sStage = smem + a_bytes;
  const int NS = num_stages(resident, PAIR);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + NS * st_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* tfull = bars + 2 * kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tempty + 2;
  uint64_t* aempty = afull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);
  float* scratch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = PAIR ? (int)cluster_ctarank() : 0;
  const int u0 = PAIR ? (int)blockIdx.x >> 1 : (int)blockIdx.x;
  const int ustep = PAIR ? (int)gridDim.x >> 1 : (int)gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], PAIR ? 2 * EPW : EPW);  // pair: both CTAs' epilogue warps
    }
    mbar_init(afull, 1);
    // two issuer warps (lean hi-only pair loop) each commit once per unit
    mbar_init(aempty, (GGM_LEAN_ISSUE && GGM_LEAN_ISSUERS == 2 && PAIR &&
                       (KIND == kSeed || p.screen)) ? 2 : 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    if (PAIR)
      tmem_alloc_pair(tmem_slot, kTmemCols);
    else
      tmem_alloc(tmem_slot, kTmemCols);
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (p.sc->flags != 0) {
    // invalid input: skip all work (status reported by the host after synchronising)
  } else if (warp >= kFirstEpiWarp) {
    setmaxnreg_inc<regs_epi(EPW)>();
    if (KIND == kSym)
      epilogue_emit<KIND, PAIR, EPW>(p, tmem_base, tfull, tempty, warp, lane, scratch, u0, ustep,
                                     rank);
    else if (KIND == kSeed)
      epilogue_seed<MAXT, PAIR, EPW>(p, tmem_base, tfull, tempty, warp, lane, scratch, u0, ustep,
                                     rank);
    else if (KIND == kSymList)
      epilogue_mass<PAIR, EPW>(p, tmem_base, tfull, tempty, warp, lane, scratch, u0, ustep, rank);
    else
      epilogue_role<MAXT, KIND, PAIR>(p, tmem_base, tfull, tempty, warp, lane, scratch, u0, ustep,
                                      rank);
  } else {
    setmaxnreg_dec<kRegsCtl>();
    if (warp == 0 && lane == 0) {
      // ===================== producer: async copies global -> shared ===================
      const uint64_t pol_b = policy_evict_last();
      const uint64_t pol_a = policy_evict_first();
      const size_t bb = block_bytes(KA);
      const int lines_per_block = 2 * KA * kRowsPerBlock;  // 128-byte lines per 128-row block
      if (PAIR) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      }
      int stage = 0;
      uint32_t phase = 0;
      int a_iter = 0;
      for (int uj = u0; uj < unit_count<KIND>(p); uj += ustep) {
        const int u = unit_of<KIND>(p, uj);
        int ub;
        const int ntiles = unit_tiles<KIND, PAIR>(p, u, ub);
        const int rb = PAIR ? 2 * ub + rank : ub;
        const uint8_t* Ablk = p.A + (size_t)rb * bb;
        if (resident) {
          if (a_iter > 0) mbar_wait(aempty, (a_iter - 1) & 1);
          if (PAIR) {
            // both CTAs' A bytes are credited to the leader's barrier
            if (rank == 0) mbar_arrive_expect_tx(afull, (uint32_t)(2 * bb));
            for (int a = 0; a < 2 * KA; ++a)
              tma_load_2d_pair(sA + (size_t)a * kAtomBytes, &tmA, 0,
                               rb * lines_per_block + a * kRowsPerBlock, afull, pol_a);
          } else {
            mbar_arrive_expect_tx(afull, (uint32_t)bb);
            bulk_g2s(sA, Ablk, (uint32_t)bb, afull, pol_a);
          }
          ++a_iter;
        }
        TileIter<KIND, PAIR> ti;
        ti.start(p, u, uj, ub, u0, ustep);
        for (int s = 0; s < ntiles; ++s, ti.next(p)) {
          if (PAIR) {
            // this CTA's half of the B tile: operand block K0 + rank, hi (+ lo) per K atom
            const int bline = (ti.K0 + rank) * lines_per_block;
            const bool hi_only = KIND == kSeed || p.screen;
            const uint32_t sbytes = (uint32_t)(hi_only ? 1 : 2) * kAtomBytes;
            for (int a = 0; a < KA; ++a) {
              mbar_wait(&empty[stage], phase ^ 1);
              if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * sbytes);
              uint8_t* st = sStage + stage * st_bytes;
              tma_load_2d_pair(st, &tmB, 0, bline + a * kRowsPerBlock, &full[stage], pol_b);
              if (!hi_only)
                tma_load_2d_pair(st + kAtomBytes, &tmB, 0, bline + (KA + a) * kRowsPerBlock,
                                 &full[stage], pol_b);
              if (++stage == NS) {
                stage = 0;
                phase ^= 1;
              }
            }
            continue;
          }
          const uint8_t* B0 = p.B + (size_t)ti.K0 * bb;
          const uint8_t* B1 = p.B + (size_t)ti.K1 * bb;
          if (resident) {
            // B hi (block K0 | block K1), then B lo, of each K atom: 256 rows per atom,
            // uniform 1 KB SBO (the seed pass reads only the hi array)
            const bool hi_only = KIND == kSeed || p.screen;
            const uint32_t sbytes = (uint32_t)(hi_only ? 2 : 4) * kAtomBytes;
            for (int a = 0; a < KA; ++a) {
              mbar_wait(&empty[stage], phase ^ 1);
              uint8_t* st = sStage + stage * st_bytes;
              mbar_arrive_expect_tx(&full[stage], sbytes);
              for (int hl = 0; hl < (hi_only ? 1 : 2); ++hl) {
                const size_t ao = (size_t)(hl * KA + a) * kAtomBytes;
                bulk_g2s(st + 2 * hl * kAtomBytes, B0 + ao, kAtomBytes, &full[stage], pol_b);
                bulk_g2s(st + (2 * hl + 1) * kAtomBytes, B1 + ao, kAtomBytes, &full[stage], pol_b);
              }
              if (++stage == NS) {
                stage = 0;
                phase ^= 1;
              }
            }
            continue;
          }
          for (int a = 0; a < KA; ++a) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = sStage + stage * st_bytes;
            mbar_arrive_expect_tx(&full[stage], (uint32_t)st_bytes);
            bulk_g2s(st, Ablk + (size_t)a * kAtomBytes, kAtomBytes, &full[stage], pol_a);
            bulk_g2s(st + kAtomBytes, Ablk + (size_t)(KA + a) * kAtomBytes, kAtomBytes,
                     &full[stage], pol_a);
            uint8_t* sb = st + 2 * kAtomBytes;
            bulk_g2s(sb, B0 + (size_t)a * kAtomBytes, kAtomBytes, &full[stage], pol_b);
            bulk_g2s(sb + kAtomBytes, B1 + (size_t)a * kAtomBytes, kAtomBytes, &full[stage],
                     pol_b);
            bulk_g2s(sb + 2 * kAtomBytes, B0 + (size_t)(KA + a) * kAtomBytes, kAtomBytes,
                     &full[stage], pol_b);
            bulk_g2s(sb + 3 * kAtomBytes, B1 + (size_t)(KA + a) * kAtomBytes, kAtomBytes,
                     &full[stage], pol_b);
            if (++stage == NS) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    } else if (rank == 0 &&
               (warp == GGM_MMA_WARP ||
                (GGM_LEAN_ISSUE && GGM_LEAN_ISSUERS == 2 && PAIR && (KIND == kSeed || p.screen) &&
                 warp == 2))) {
      // ===================== MMA issuer: warp 1 (of the pair leader) =====================
      // The whole warp runs the loop (warp-uniform descriptors); one elected lane issues the
      // tcgen05.mma / commit instructions.  With one thread and per-lane registers, every
      // MMA cost ~27 issue slots on an SM sub-partition shared with 4 epilogue warps.
      constexpr uint32_t idesc = idesc_f16_f32(PAIR ? 2 * kRowsPerBlock : kRowsPerBlock, kTileN);
      const bool issuer = elect_one();
      const bool three = KIND != kSeed && !p.screen;  // hi*lo and lo*hi products too
      int stage = 0;
      uint32_t phase = 0;
      int buf = 0;
      uint32_t tphase = 0;
      int a_iter = 0;
#ifdef GGM_MMA_PROF
      long long pr_t0 = clock64(), pr_te = 0, pr_tf = 0, pr_ta = 0, pr_n = 0, pr_c, pr_is = 0;
#define PROF_W(acc, stmt) do { pr_c = clock64(); stmt; acc += clock64() - pr_c; } while (0)
#else
#define PROF_W(acc, stmt) stmt
#endif
#if GGM_LEAN_ISSUE
      if (PAIR && !three) {
        // Lean hi-only issue loop (screening main pass, seed pass): the MMA warp shares its
        // SM sub-partition with 4 busy epilogue warps, so every instruction on its path
        // costs issue slots (profiles/r01i_mma_prof.md).  All descriptors are loop
        // invariant: A resident (atoms 0/1, hi and lo arrays), B stage s = stage 0 + s·st_bytes
        // (the 14-bit address field, addr >> 4, does not overflow below 256 KB); per atom
        // the hi slots and the packed-tail slots are 4-bit masks.
        const uint64_t dAh0 = sw128_desc(smem_u32(sA)), dAh1 = dAh0 + (kAtomBytes >> 4);
        const uint64_t dAl0 = dAh0 + (uint64_t)((KA * kAtomBytes) >> 4);
        const uint64_t dAl1 = dAl0 + (kAtomBytes >> 4);
        const uint64_t dB0 = sw128_desc(smem_u32(sStage));
        const uint32_t st16 = (uint32_t)(st_bytes >> 4);
#if GGM_MMA_THROTTLE
        int fs1 = -1, fs2 = -1;  // stages (and phases) of the last two issued atoms
        uint32_t fp1 = 0, fp2 = 0;
#endif
        uint32_t hm[2], tm[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          hm[a] = tm[a] = 0;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const int slot = 4 * a + ks;
            if (slot < p.KS) hm[a] |= 1u << ks;
            else if (slot < p.KS + p.TS) tm[a] |= 1u << ks;
          }
        }
        for (int uj = u0; uj < unit_count<KIND>(p); uj += ustep) {
          const int u = unit_of<KIND>(p, uj);
          int ub;
          const int ntiles = unit_tiles<KIND, PAIR>(p, u, ub);
          PROF_W(pr_ta, mbar_wait(afull, a_iter & 1));
          tc_fence_after();
          for (int s = 0; s < ntiles; ++s) {
#ifdef GGM_MMA_PROF
            ++pr_n;
#endif
            if (GGM_LEAN_ISSUERS == 2 && buf != warp - 1) {  // the other issuer's tile
              stage += KA;
              while (stage >= NS) {
                stage -= NS;
                phase ^= 1;
              }
              if (++buf == 2) {
                buf = 0;
                tphase ^= 1;
              }
              continue;
            }
            PROF_W(pr_te, LEAN_WAIT(&tempty[buf], tphase ^ 1));
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + (uint32_t)(buf * kTileN);
            for (int a = 0; a < KA; ++a) {
              PROF_W(pr_tf, LEAN_WAIT(&full[stage], phase));
#if GGM_MMA_THROTTLE
              // at most two atoms of MMAs outstanding: wait for the one before the last
              // (its commit on empty[] completes phase fp2) so the tcgen05.mma issue does not
              // block this sub-partition's dispatch on a full MMA queue
              if (fs2 >= 0) PROF_W(pr_is, LEAN_WAIT(&empty[fs2], fp2));
#endif
              tc_fence_after();
              const uint64_t dB = dB0 + (uint64_t)(stage * st16);
              const uint64_t dAh = a ? dAh1 : dAh0, dAl = a ? dAl1 : dAl0;
              const uint32_t h = a ? hm[1] : hm[0], tl = a ? tm[1] : tm[0];
              if (issuer) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                  const uint64_t o = (uint64_t)(2 * ks);
                  if ((h | tl) >> ks & 1u)
                    mma_f16<PAIR>(d_tmem, ((h >> ks) & 1u ? dAh : dAl) + o, dB + o, idesc,
                                  (a | ks) ? 1u : 0u);
                }
                mma_commit_any<PAIR>(&empty[stage]);
              }
              __syncwarp();
#if GGM_MMA_THROTTLE
              fs2 = fs1;
              fp2 = fp1;
              fs1 = stage;
              fp1 = phase;
#endif
              if (++stage == NS) {
                stage = 0;
                phase ^= 1;
              }
            }
            if (issuer) mma_commit_any<PAIR>(&tfull[buf]);
            __syncwarp();
            if (++buf == 2) {
              buf = 0;
              tphase ^= 1;
            }
          }
          if (issuer) mma_commit_any<PAIR>(aempty);
          __syncwarp();
          ++a_iter;
        }
      } else
#endif
      for (int uj = u0; uj < unit_count<KIND>(p); uj += ustep) {
        const int u = unit_of<KIND>(p, uj);
        int ub;
        const int ntiles = unit_tiles<KIND, PAIR>(p, u, ub);
        if (resident) {
          PROF_W(pr_ta, mbar_wait(afull, a_iter & 1));
          tc_fence_after();
        }
        for (int s = 0; s < ntiles; ++s) {
#ifdef GGM_MMA_PROF
          ++pr_n;
#endif
#if defined(GGM_MMA_NOWAIT)
          if (0)
#endif
          PROF_W(pr_te, mbar_wait(&tempty[buf], tphase ^ 1));
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(buf * kTileN);
          for (int a = 0; a < KA; ++a) {
#if defined(GGM_MMA_NOWAIT) && GGM_MMA_NOWAIT > 1
            if (0)
#endif
            PROF_W(pr_tf, mbar_wait(&full[stage], phase));
            tc_fence_after();
            uint8_t* st = sStage + stage * st_bytes;
            uint32_t aHi_s, aLo_s, bHi_s, bLo_s;
            if (resident) {
              aHi_s = smem_u32(sA + (size_t)a * kAtomBytes);
              aLo_s = smem_u32(sA + (size_t)(KA + a) * kAtomBytes);
              bHi_s = smem_u32(st);
              bLo_s = bHi_s + (PAIR ? 1 : 2) * kAtomBytes;
            } else {
              aHi_s = smem_u32(st);
              aLo_s = aHi_s + kAtomBytes;
              bHi_s = aHi_s + 2 * kAtomBytes;
              bLo_s = aHi_s + 4 * kAtomBytes;
            }
            // descriptors of the atom bases; K step ks = +2 on the address field (32 B)
            const uint64_t dAh = sw128_desc(aHi_s), dAl = sw128_desc(aLo_s);
            const uint64_t dBh = sw128_desc(bHi_s), dBl = sw128_desc(bLo_s);
#ifdef GGM_MMA_PROF
            const long long pr_i0 = clock64();
#endif
            if (issuer) {
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                const int slot = a * 4 + ks;
                const uint64_t o = (uint64_t)(2 * ks);
                const uint32_t acc = (a | ks) ? 1u : 0u;
                if (slot < p.KS) {
                  mma_f16<PAIR>(d_tmem, dAh + o, dBh + o, idesc, acc);
                  if (three) {  // the seed and screening passes use hi*hi alone
                    mma_f16<PAIR>(d_tmem, dAh + o, dBl + o, idesc, 1u);
                    mma_f16<PAIR>(d_tmem, dAl + o, dBh + o, idesc, 1u);
                  }
                } else if (slot < p.KS + p.TS) {
                  // packed tail: A's slot in the lo array [hi|hi|lo], B's in the hi array
                  // [hi|lo|hi] (3 products of the last k mod 16 elements in one K step)
                  mma_f16<PAIR>(d_tmem, dAl + o, dBh + o, idesc, acc);
                }
              }
              mma_commit_any<PAIR>(&empty[stage]);
            }
            __syncwarp();
#ifdef GGM_MMA_PROF
            pr_is += clock64() - pr_i0;
#endif
            if (++stage == NS) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (issuer) mma_commit_any<PAIR>(&tfull[buf]);
          __syncwarp();
          if (++buf == 2) {
            buf = 0;
            tphase ^= 1;
          }
        }
        if (resident) {
          if (issuer) mma_commit_any<PAIR>(aempty);
          __syncwarp();
          ++a_iter;
        }
      }
#ifdef GGM_MMA_PROF
      if (issuer && (blockIdx.x & 15) == 0)
        printf("MMAPROF cta %d tiles %lld total %lld tempty %lld full %lld afull %lld issue %lld\n",
               (int)blockIdx.x, pr_n, clock64() - pr_t0, pr_te, pr_tf, pr_ta, pr_is);
#endif
#undef PROF_W
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    if (PAIR)
      tmem_dealloc_pair(tmem_base, kTmemCols);
    else
      tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ------------------------------------------------------------------ BK3 (mode 0, C > 1)
template <int MAXT>
__global__ void merge_partials(const int32_t* __restrict__ pcol, const float* __restrict__ pval,
                               int64_t rows, int C, int t, int64_t* row_ptr, int32_t* col,
                               float* val) {
  const int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (lr >= rows) return;
  TopList<MAXT> top;
  top.init(t);
  for (int c = 0; c < C; ++c) {
    const int64_t base = ((int64_t)c * rows + lr) * t;
    for (int e = 0; e < t; ++e) {
      const int j = pcol[base + e];
      if (j < 0) continue;
      const float v = pval[base + e];
      top.merge_insert(fabsf(v), v, j);
    }
  }
  top.emit_sorted(t, col + lr * t, val + lr * t, 1.f);
  row_ptr[lr] = lr * t;
  if (lr == rows - 1) row_ptr[rows] = rows * t;
}

// ------------------------------------------------------------------ BK3 (kSym)
// Row j's final list = top-t of (its row-direction list over its own cyclic window) ∪
// (the transposed-direction candidates other blocks emitted for it; sorted by target row,
// the row's range found by binary search).
__device__ __forceinline__ int64_t lower_bound_u32(const uint32_t* a, int64_t n, uint32_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Re-evaluation of the screened candidates (pool sorted by target row): U in bound order,
// rows padded to kp = k rounded up to 4 floats (16-byte aligned float4 slices),
// kRecGroup lanes per candidate; fp32 x fp32 products are exact in fp64 and summed in a
// fixed order (lane slices, then a kRecGroup-lane butterfly), so ψ_ij and ψ_ji come out
// bit-identical.
constexpr int kRecMaxK = 128;
constexpr int kRecGroup = 8;                      // lanes per candidate
__host__ __device__ inline int rec_stride(int k) { return (k + 3) & ~3; }
// Only candidates that can still reach the row's exact top t are re-evaluated: with M_j =
// screen_margin(j) in ψ units (the screening error bound of every pair of row j) and s_t the
// t-th largest screened magnitude of the row's candidates, an exact top-t entry c has
// |ψ1(c)| >= T - M_j >= s_t - 2 M_j (T the exact t-th magnitude, s_t <= T + M_j).  The
// others get value 0 and cannot displace the re-evaluated ones in merge_sym.  On a rank's
// partial list (distributed scheme) s_t is smaller than on the full row: still conservative.
// rows' candidate ranges of the key-sorted pool: off[j] = first index with key >= j (off[n]
// = the number of real candidates; unused reservations carry key UINT32_MAX, sorted last)
__global__ void cand_row_offsets(const uint32_t* __restrict__ skey, int64_t ncand, int64_t n,
                                 int64_t* __restrict__ off) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n;
       j += (int64_t)gridDim.x * blockDim.x)
    off[j] = lower_bound_u32(skey, ncand, (uint32_t)j);
}
// cut[j] = s_t - 2 M_j, or -1 (keep all) for rows with at most t candidates: one thread per
// row, a magnitude-only top-t list over the row's screened values
template <int MAXT>
__global__ void rec_cut(const int64_t* __restrict__ off, const uint2* __restrict__ sval,
                        int64_t n, int t, int k, const float* __restrict__ rn,
                        const int32_t* __restrict__ perm,
                        const unsigned int* __restrict__ rn_max_bits,
                        const DevScalars* __restrict__ sc, float* __restrict__ cut) {
  const float umax = __uint_as_float(*rn_max_bits);
  const float sf = ldexpf(1.f, sc->exp2);  // ψ units = accumulator units / s^2
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = off[j], b1 = off[j + 1];
    if (b1 - b0 <= t) {
      cut[j] = -1.f;
      continue;
    }
    MagList<MAXT> top;
    top.init(t);
    for (int64_t e = b0; e < b1; ++e) {
      const float a = fabsf(__uint_as_float(sval[e].y));
      if (a > top.m[0]) top.insert(a);
    }
    const float mj = ldexpf(screen_margin(rn[perm[j]] * sf, umax * sf, k), -2 * sc->exp2);
    cut[j] = top.m[0] - 2.f * mj;
  }
}
// U = V diag(sqrt(λ)) in bound order (fp32, row stride rec_stride(k), zero padded), the
// re-evaluation operand: ψ_ij = Σ_r U_ir U_jr.  One warp per row (one permutation lookup),
// sqrt(λ) staged in shared memory once per block.
__global__ void gather_u_bound(const float* __restrict__ V, const double* __restrict__ lam,
                               const int32_t* __restrict__ perm, int64_t n, int k,
                               float* __restrict__ Ub) {
  __shared__ double sl[kRecMaxK];
  for (int c = threadIdx.x; c < k; c += blockDim.x) sl[c] = sqrt(lam[c]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int kp = rec_stride(k);
  const bool vec = (k & 3) == 0 && (reinterpret_cast<uintptr_t>(V) & 15) == 0;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float* v = V + (int64_t)perm[p] * k;
    if (vec) {  // k ≡ 0 (mod 4): kp = k, float4 rows
      const float4* v4 = reinterpret_cast<const float4*>(v);
      float4* u4 = reinterpret_cast<float4*>(Ub + p * kp);
      for (int j = lane; j < (k >> 2); j += 32) {
        const float4 x = __ldg(v4 + j);
        const double* l = sl + 4 * j;
        u4[j] = make_float4((float)((double)x.x * l[0]), (float)((double)x.y * l[1]),
                            (float)((double)x.z * l[2]), (float)((double)x.w * l[3]));
      }
      continue;
    }
    for (int c = lane; c < kp; c += 32) Ub[p * kp + c] = c < k ? (float)((double)v[c] * sl[c]) : 0.f;
  }
}
// Exact values of the pool candidates: candidate-parallel over the key-sorted pool (uniform
// work, no per-row chains), kRecGroup lanes per candidate, 2 x 32/kRecGroup candidates per
// warp in flight; candidates below their row's cut (nullptr: none) get 0 without loads.
// Slots at or beyond off[n] (unused reservations) are skipped.  ψ = Σ_c U_jc U_ic over the lane slices in a fixed order, then a kRecGroup-lane
// butterfly: the same products in the same order for (j, i) and (i, j).
template <int R>  // float4 slices per lane: 32 R >= kp
__global__ void __launch_bounds__(256) recompute_sorted(const uint32_t* __restrict__ skey,
                                                        uint2* __restrict__ sval,
                                                        const int64_t* __restrict__ off, int64_t n,
                                                        const float* __restrict__ Ub, int k,
                                                        const float* __restrict__ cut) {
  const int lane = threadIdx.x & 31;
  const int g = lane % kRecGroup;   // slice of the candidate's rows
  const int cs = lane / kRecGroup;  // candidate slot of this step
  constexpr int CPW = 32 / kRecGroup;
  constexpr int U = 2;
  const int kp = rec_stride(k);
  const int64_t ncand = off[n];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e0 = warp * (U * CPW); e0 < ncand; e0 += nwarps * (U * CPW)) {
    float4 xa[U][R], xb[U][R];
    bool keep[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t ei = e0 + u * CPW + cs;
      const bool ok = ei < ncand;
      const uint32_t j = ok ? skey[ei] : 0u;
      const uint2 cvv = ok ? sval[ei] : make_uint2(0u, 0u);
      const uint32_t i = cvv.x;
      GGM_DCHECK(!ok || (j < (uint32_t)n && i < (uint32_t)n));
      keep[u] = ok && (cut == nullptr || fabsf(__uint_as_float(cvv.y)) >= cut[j]);
      const float4* ua = reinterpret_cast<const float4*>(Ub + (int64_t)j * kp);
      const float4* vb = reinterpret_cast<const float4*>(Ub + (int64_t)i * kp);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int c = 32 * r + 4 * g;
        const bool in = keep[u] && c < kp;
        xa[u][r] = in ? __ldg(ua + c / 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        xb[u][r] = in ? __ldg(vb + c / 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {  // exact fp32 x fp32 products
        acc = fma((double)xa[u][r].x, (double)xb[u][r].x, acc);
        acc = fma((double)xa[u][r].y, (double)xb[u][r].y, acc);
        acc = fma((double)xa[u][r].z, (double)xb[u][r].z, acc);
        acc = fma((double)xa[u][r].w, (double)xb[u][r].w, acc);
      }
#pragma unroll
      for (int o = kRecGroup / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const int64_t ei = e0 + u * CPW + cs;
      if (g == 0 && ei < ncand) sval[ei].y = __float_as_uint(keep[u] ? (float)acc : 0.f);
    }
  }
}

// R = ceil(kp / 32) instantiations (no FMAs on padding slices); one resident wave of blocks
// (the kernel is grid-stride: later waves would each take a full stride share)
template <int R>
static void launch_recompute_r(const uint32_t* skey, uint2* sval, const int64_t* off, int64_t n,
                               const float* Ub, int k, const float* cut, int sms,
                               cudaStream_t s) {
  static int per_sm = 0;
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, recompute_sorted<R>, 256, 0) !=
            cudaSuccess || per_sm < 1)
      per_sm = 2;
  }
  recompute_sorted<R><<<sms * per_sm, 256, 0, s>>>(skey, sval, off, n, Ub, k, cut);
}
template <int MAXT>
__global__ void merge_sym(const uint32_t* __restrict__ key, const uint2* __restrict__ cv,
                          int64_t ncand, int64_t n, int t, const int32_t* __restrict__ perm,
                          int64_t row_begin, int64_t row_end, int64_t* row_id,
                          int64_t* row_ptr, int32_t* col, float* val,
                          const int64_t* __restrict__ off = nullptr) {
  // row j (bound-order index): top t of its candidates (source in bound order, value) by
  // (|ψ| desc, original column id asc), ascending columns.  row_id == nullptr: written at
  // the original row id (single GPU, full axis); else at j - row_begin, with its original id
  // in row_id (a rank's share of the distributed symmetric scheme)
  const int64_t j = row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= row_end) return;
  TopList<MAXT> top;
  top.init(t);
  // the row's bucket: from the re-evaluation's row offsets when given, else two binary searches
  const int64_t b0 = off ? off[j] : lower_bound_u32(key, ncand, (uint32_t)j);
  const int64_t b1 = off ? off[j + 1] : lower_bound_u32(key, ncand, (uint32_t)j + 1u);
  for (int64_t e = b0; e < b1; ++e) {
    const uint2 x = cv[e];
    GGM_DCHECK(x.x < (uint32_t)n);
    const float v = __uint_as_float(x.y);
    top.merge_insert(fabsf(v), v, __ldg(perm + x.x));
  }
  const int64_t o = row_id ? j - row_begin : (int64_t)perm[j];
  if (row_id) row_id[o] = perm[j];
  top.emit_sorted(t, col + o * t, val + o * t, 1.f);
  if (row_ptr) {
    row_ptr[o] = o * t;
    if (o == n - 1) row_ptr[n] = n * t;
  }
}

// per-destination counts of a key-sorted candidate list: bnd[r] = first index with key >= lo[r]
__global__ void bucket_bounds(const uint32_t* __restrict__ key, int64_t ncand,
                              const int64_t* __restrict__ lo, int nb, int64_t* __restrict__ bnd) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= nb) bnd[r] = lower_bound_u32(key, ncand, (uint32_t)lo[r]);
}

__global__ void iota_i32(int32_t* p, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

__global__ void fill_f32(float* p, int64_t count, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ------------------------------------------------------------------ BK3 (mode 1)
__global__ void coo_to_csr(const int64_t* __restrict__ key, const float* __restrict__ v,
                           int64_t count, int64_t n, int64_t rows, int64_t* row_ptr,
                           int32_t* col, float* val) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= count;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < count) {
      col[e] = (int32_t)(key[e] % n);
      val[e] = v[e];
    }
    const int64_t r = (e < count) ? key[e] / n : rows;       // first row NOT before e
    const int64_t rp = (e == 0) ? -1 : key[e - 1] / n;      // row of the previous entry
    for (int64_t rr = rp + 1; rr <= r && rr <= rows; ++rr) row_ptr[rr] = e;
  }
}

__global__ void zero_row_ptr(int64_t* row_ptr, int64_t rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= rows;
       i += (int64_t)gridDim.x * blockDim.x)
    row_ptr[i] = 0;
}

// ------------------------------------------------------------------ host plan

struct Plan {
  int64_t n, rows, row_begin;
  int k, KA, KS, TS, t, mode, resident, alias;
  int64_t RB, NT, C, TPC;
  int64_t nBblocks, nAblocks;
  int64_t capacity;
  size_t coo_temp_bytes;
  int pair;      // CTA-pair kernels (cta_group::2), A resident only
  int64_t RBu;   // units of row blocks: RB (1 CTA) or ceil(RB/2) 256-row blocks (pair)
  int64_t NBu;   // kSym/kSeed units over the axis: NB or ceil(NB/2)
  int sym;       // symmetric scheme (kSeed + kSym + merge_sym)
  int screen;    // symmetric scheme: hi*hi screening + exact re-evaluation of candidates
  int rec_cut;   // screening, mode 0: per-row re-evaluation cuts allowed (1: when the pool
                 // is candidate-heavy, 2: always — GGM_REC_CUT=1); needs the screened values
  int SS;        // seed column-tile stride
  int64_t NB;    // 128-row blocks of the axis
  int64_t cand_total;  // kSym: candidate pool capacity (entries)
  size_t sort_temp_bytes;
};

static int choose_chunks(int64_t RB, int64_t NT, int sms) {
  int best = 1;
  double best_cost = 1e300;
  const int cmax = (int)std::min<int64_t>(NT, 64);
  for (int C = 1; C <= cmax; ++C) {
    const int64_t units = RB * C;
    const int64_t tpc = (NT + C - 1) / C;
    const int64_t waves = (units + sms - 1) / sms;
    // per-CTA tiles on the critical path + a small merge penalty per extra chunk
    const double cost = (double)waves * tpc * (1.0 + 0.002 * (C - 1));
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = C;
    }
  }
  return best;
}

// seed sample fraction for the next plans on this thread (0: kSeedFrac).  The overall rules'
// top-32 lists pass on down-weighted scores sets 8: the flattened score distribution leaves
// ~t x (n / sample) candidates per row, which a 1/64 sample would overflow.
static thread_local int g_seed_frac_override = 0;
struct SeedFracScope {
  int saved;
  explicit SeedFracScope(int f) : saved(g_seed_frac_override) { g_seed_frac_override = f; }
  ~SeedFracScope() { g_seed_frac_override = saved; }
};
// extra symmetric candidate-pool entries for the next plans on this thread (the overall
// rules' global-threshold pass: every directed entry above τ on top of the top-m lists)
static thread_local int64_t g_cand_extra = 0;
struct CandExtraScope {
  int64_t saved;
  explicit CandExtraScope(int64_t e) : saved(g_cand_extra) { g_cand_extra = e; }
  ~CandExtraScope() { g_cand_extra = saved; }
};

static ggm_status make_plan(int64_t n, int k, int64_t row_begin, int64_t row_end,
                            const ggm_sparsify_opts* o, int64_t capacity, Plan* pl) {
  if (!o) return fail(GGM_ERR_INVALID_ARGUMENT, "opts is NULL");
  if (n < 2) return fail(GGM_ERR_INVALID_ARGUMENT, "n=%lld < 2", (long long)n);
  if (n > (int64_t)INT_MAX - 256) return fail(GGM_ERR_INVALID_ARGUMENT, "n too large for int32 columns");
  if (k < 1 || k > n) return fail(GGM_ERR_INVALID_ARGUMENT, "k=%d not in [1,n]", k);
  if (row_begin < 0 || row_end > n || row_begin >= row_end)
    return fail(GGM_ERR_INVALID_ARGUMENT, "row range [%lld,%lld) invalid for n=%lld",
                (long long)row_begin, (long long)row_end, (long long)n);
  if (o->mode < 0 || o->mode > 3)  // 2 (row mass), 3 (histogram): internal (overall rules)
    return fail(GGM_ERR_INVALID_ARGUMENT, "mode=%d", o->mode);
  if (o->mode == 0 && (o->topk < 1))
    return fail(GGM_ERR_INVALID_ARGUMENT, "topk=%d < 1", o->topk);
  if (o->mode == 0 && o->topk > GGM_MAX_TOPK)
    return fail(GGM_ERR_UNSUPPORTED, "topk=%d > GGM_MAX_TOPK=%d", o->topk, GGM_MAX_TOPK);
  if (o->mode == 1 && !(o->tau >= 0.f && std::isfinite(o->tau)))
    return fail(GGM_ERR_INVALID_ARGUMENT, "tau must be finite and >= 0");
  if (o->col_chunks < 0) return fail(GGM_ERR_INVALID_ARGUMENT, "col_chunks < 0");
  if (o->symmetric < 0 || o->symmetric > 2)
    return fail(GGM_ERR_INVALID_ARGUMENT, "symmetric=%d not in {0,1,2}", o->symmetric);
  pl->n = n;
  pl->k = k;
  pl->row_begin = row_begin;
  pl->rows = row_end - row_begin;
  pl->mode = o->mode;
  pl->t = (int)std::max<int64_t>(1, std::min<int64_t>(o->topk, n - 1));
  pl->KA = (k + kAtomElems - 1) / kAtomElems;
  // K slots: full 16-element slots x 3 MMAs, plus the packed tail (3 products of the last
  // k mod 16 elements in ceil(3r/16) slots) when it saves MMAs and fits the free slots of
  // the last atom: k = 100 -> 6 x 3 + 1 = 19 MMAs per K sweep instead of 7 x 3 = 21
  {
    const int m = k / 16, r = k % 16, ts = (3 * r + 15) / 16;
    const bool pack = r > 0 && ts < 3 && m + ts <= 4 * pl->KA && !getenv("GGM_NO_TAILPACK");
    pl->KS = pack ? m : (k + 15) / 16;
    pl->TS = pack ? ts : 0;
  }
  pl->resident = pl->KA <= kMaxResidentAtoms ? 1 : 0;
  pl->alias = (row_begin % kRowsPerBlock) == 0 ? 1 : 0;
  pl->NT = (n + kTileN - 1) / kTileN;
  pl->RB = (pl->rows + kRowsPerBlock - 1) / kRowsPerBlock;
  pl->NB = (n + kRowsPerBlock - 1) / kRowsPerBlock;
  // CTA pairs whenever A is resident: per-SM operand traffic halves (see num_stages)
  pl->pair = pl->resident && !getenv("GGM_NO_PAIR") ? 1 : 0;
  pl->RBu = pl->pair ? (pl->RB + 1) / 2 : pl->RB;
  pl->NBu = pl->pair ? (pl->NB + 1) / 2 : pl->NB;
  // B: all 256-row column tiles, + 2 zero blocks so a pair's second 128-row A block of an
  // aliased row range always exists; A (unaligned row ranges): whole units
  pl->nBblocks = pl->NT * 2 + 2;
  pl->nAblocks = pl->alias ? 0 : (pl->pair ? 2 * pl->RBu : pl->RB);
  const int sms = num_sms();
  const int ctas = pl->pair ? sms / 2 : sms;  // concurrent units
  const bool full_axis = row_begin == 0 && row_end == n;
  // symmetric scheme (each unordered block pair evaluated once): full axis, top-t mode, A
  // resident; automatic (0) above kSymAutoN rows, where the seed pass and the candidate
  // merge are small against the halved tensor-core work
  // symmetric scheme: per-row top-t (mode 0) or threshold (mode 1, thresholds = τ)
  const bool sym_ok = (o->mode == 0 || o->mode == 1) && full_axis && pl->resident;
  pl->sym = sym_ok && (o->symmetric == 1 || (o->symmetric == 0 && n >= kSymAutoN)) ? 1 : 0;
  pl->screen = pl->sym && k <= 128 && !getenv("GGM_NO_SCREEN") ? 1 : 0;
  // re-evaluation cuts pay only on candidate-heavy pools (the top-32 lists of the overall
  // rules, ~10t candidates per row); at top-10 (~2t per row) they keep nearly every
  // candidate, and without them the epilogue skips each candidate's screened value
  pl->rec_cut = 0;
  if (pl->screen && pl->mode == 0) {
    pl->rec_cut = pl->t >= kRecCutMinT ? 1 : 0;
    if (const char* e = getenv("GGM_REC_CUT")) pl->rec_cut = atoi(e) != 0 ? 2 : 0;  // tests: both forms
  }
  // candidates: ~ t x 16 / 2 per row expected (seed samples 1/16 of the columns, half of
  // each row's columns come from the transposed direction); regions hold 2x that on average
  // pool: 2x the expected candidates + one chunk per epilogue warp of partially used space
  // candidates: each row's entries >= its bound b_i (the t-th largest over a 1/SS column
  // sample, i.e. about the (SS t)-th largest overall): ~SS t per row, from both directions;
  // the pool holds 2x that plus the partially used reservation of every epilogue warp
  // seed sample: the n/kSeedFrac columns of largest ||U_j|| (whole 256-column tiles, at
  // least one).  |ψ_ij| <= ||U_i|| ||U_j||, so large-norm columns hold most rows' largest
  // entries: on C5 factors the t-th largest over this 1/64 sample leaves ~21 candidates per
  // row where a strided 1/8 sample left ~89 (any sample gives a valid bound).
  // Size: n/kSeedFrac columns, but at least kSeedMinTiles tiles (12,288 columns) while that
  // stays <= 1/8 of the axis; never fewer than 8 tiles.  The seed is a plain pass over
  // n x sample entries; a larger sample tightens b_i, which cuts the main kernel's rare-path
  // visits (chunks with an entry above a bound): C4 (n = 2e5, k = 64) main 4.77 -> 3.95 ms
  // for +0.23 ms of seed at 49 vs 13 tiles; C5 (n = 1e6) main 96.9 -> 93.9 ms for +2.2 ms
  // at 1/32 vs 1/64 (profiles/r02_logs/r02u_seed_sweep.log).
  {
    int64_t tiles;
    if (g_seed_frac_override > 0 || getenv("GGM_SEED_FRAC")) {
      int64_t frac = g_seed_frac_override;
      if (const char* e = getenv("GGM_SEED_FRAC")) frac = std::max(1, atoi(e));  // tuning only
      tiles = std::max<int64_t>(8, (n / frac + kTileN - 1) / kTileN);
    } else {
      tiles = (n / kSeedFrac + kTileN - 1) / kTileN;
      tiles = std::max<int64_t>(tiles, std::min<int64_t>(kSeedMinTiles, pl->NT / 8));
      tiles = std::max<int64_t>(8, tiles);
    }
    pl->SS = (int)std::max<int64_t>(1, std::min<int64_t>(pl->NT, tiles));
  }
  // pool: an uninformative sample leaves ~ t x (n / sample size) candidates per row; hold
  // twice that, capped at 32 t per row (overflow -> exact plain recomputation)
  {
    const int64_t ratio = (n + pl->SS * kTileN - 1) / (pl->SS * kTileN);
    const int64_t per_row = pl->t * std::max<int64_t>(4, std::min<int64_t>(2 * ratio, 32));
    // mode 1: every directed entry above τ (minus the screening bound) is a candidate;
    // room for the output capacity + 25 % (overflow -> exact plain recomputation)
    const int64_t want = pl->mode == 1 ? std::max<int64_t>(capacity + capacity / 4, int64_t(1) << 20)
                                       : n * per_row;
    pl->cand_total = pl->sym ? want + g_cand_extra + (int64_t)sms * 16 * kCandChunk * 2 : 0;
  }
  pl->sort_temp_bytes = 0;
  if (pl->sym) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint2*)nullptr, (uint2*)nullptr, pl->cand_total);
    size_t tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, (const float*)nullptr, (float*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, n);
    pl->sort_temp_bytes = std::max(tb, tb2);
  }
  int64_t C = o->col_chunks > 0 ? o->col_chunks
                                : (pl->mode == 0 ? choose_chunks(pl->RBu, pl->NT, ctas) : 1);
  C = std::max<int64_t>(1, std::min<int64_t>(C, pl->NT));
  pl->TPC = (pl->NT + C - 1) / C;
  pl->C = (pl->NT + pl->TPC - 1) / pl->TPC;  // no empty chunks
  pl->capacity = capacity;
  pl->coo_temp_bytes = 0;
  if (pl->mode == 1 && capacity > 0) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const int64_t*)nullptr, (int64_t*)nullptr,
                                    (const float*)nullptr, (float*)nullptr, (int64_t)capacity);
    pl->coo_temp_bytes = tb;
  }
  return GGM_OK;
}

struct Work {
  DevScalars* sc;
  uint8_t* Bop;
  uint8_t* Aop;
  int32_t* pcol;
  float* pval;
  int64_t* key_in;
  int64_t* key_out;
  float* cv_in;
  float* cv_out;
  void* cub_tmp;
  float* thr;          // kSym: seed bounds by original row [NB*128]
  float* thr_p;        // kSym: bounds in permuted (sorted) order [NB*128]
  float* thr_s;        // kSym screening: thr_p lowered by the hi*hi error bound [NB*128]
  float* thr_cmin;     // kSym: minimum of the effective bounds over each 32-column chunk
  float* thr_cmin8;    // kSym: ... over each 8-column group
  float* Ub;           // kSym screening: U = V diag(sqrt λ) in bound order (re-evaluation)
  int64_t* roff;       // kSym screening: candidate row offsets of the sorted pool [n+1]
  float* rcut;         // kSym screening: per-row re-evaluation cuts [n]
  int32_t* ids;        // kSym: 0..n-1
  int32_t* perm;       // kSym: permuted index -> original id [n]
  float* rn;           // kSym: row norms ||U_i|| [n]
  float* rn_s;         // kSym: row norms in descending order [n]
  int32_t* perm_n;     // kSym: norm order -> original id [n]
  uint32_t* ckey;      // kSym: candidate pool
  uint2* cval;
  uint32_t* skey;      // kSym: sorted by target row
  uint2* sval;
  void* sort_tmp;
};

static size_t carve(const Plan& pl, void* ws, Work* w) {
  Carve cv(ws);
  w->sc = cv.take<DevScalars>(1);
  w->Bop = cv.take<uint8_t>((size_t)pl.nBblocks * block_bytes(pl.KA));
  w->Aop = cv.take<uint8_t>((size_t)pl.nAblocks * block_bytes(pl.KA));
  size_t npart = (pl.mode == 0 && pl.C > 1) ? (size_t)pl.C * pl.rows * pl.t : 0;
  w->pcol = cv.take<int32_t>(npart);
  w->pval = cv.take<float>(npart);
  const size_t ncoo = pl.mode == 1 ? (size_t)std::max<int64_t>(pl.capacity, 0) : 0;
  w->key_in = cv.take<int64_t>(ncoo);
  w->key_out = cv.take<int64_t>(ncoo);
  w->cv_in = cv.take<float>(ncoo);
  w->cv_out = cv.take<float>(ncoo);
  w->cub_tmp = cv.take<char>(pl.coo_temp_bytes);
  const size_t nb = pl.sym ? (size_t)(2 * pl.NBu) : 0;  // 128-column blocks incl. pair padding
  const size_t ct = pl.sym ? (size_t)pl.cand_total : 0;
  w->thr = cv.take<float>(nb * kRowsPerBlock);
  w->thr_p = cv.take<float>(nb * kRowsPerBlock);
  w->thr_s = cv.take<float>(pl.screen ? nb * kRowsPerBlock : 0);
  w->thr_cmin = cv.take<float>(nb * kRowsPerBlock / 32);
  w->thr_cmin8 = cv.take<float>(nb * kRowsPerBlock / 8);
  w->Ub = cv.take<float>(pl.screen ? (size_t)pl.n * rec_stride(pl.k) : 0);
  w->roff = cv.take<int64_t>(pl.screen ? (size_t)pl.n + 1 : 0);
  w->rcut = cv.take<float>(pl.screen ? (size_t)pl.n : 0);
  w->ids = cv.take<int32_t>(pl.sym ? (size_t)pl.n : 0);
  w->perm = cv.take<int32_t>(pl.sym ? (size_t)pl.n : 0);
  w->rn = cv.take<float>(pl.sym ? (size_t)pl.n : 0);
  w->rn_s = cv.take<float>(pl.sym ? (size_t)pl.n : 0);
  w->perm_n = cv.take<int32_t>(pl.sym ? (size_t)pl.n : 0);
  w->ckey = cv.take<uint32_t>(ct);
  w->cval = cv.take<uint2>(ct);
  w->skey = cv.take<uint32_t>(ct);
  w->sval = cv.take<uint2>(ct);
  w->sort_tmp = cv.take<char>(pl.sort_temp_bytes);
  return cv.used();
}

struct EventTimer {
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool on;
  cudaStream_t s;
  EventTimer(bool enabled, cudaStream_t st) : on(enabled), s(st) {
    if (on)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark(int i) {
    if (on) cudaEventRecord(ev[i], s);
  }
  void finish() {
    if (!on) return;
    cudaEventSynchronize(ev[3]);
    for (int i = 0; i < 3; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      record_timing(i, ms);
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
};

// 2-D tensor map over a tiled operand array viewed as lines of 128 bytes (64 x uint16):
// box = 128 lines = one 16 KB (128-row block, K atom) chunk, no swizzle (the data is already
// stored in the SWIZZLE_128B canonical layout by split_tile).  Used by the CTA-pair kernels,
// whose cta_group::2 tensor copies credit the pair leader's mbarrier.
static ggm_status make_line_tmap(CUtensorMap* tm, const void* base, uint64_t lines) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(GGM_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {64, (cuuint64_t)std::max<uint64_t>(lines, 128)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides,
                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(GGM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return GGM_OK;
}

struct TMaps {
  CUtensorMap A, B;
};

template <int MAXT, int KIND, bool PAIR>
static cudaError_t launch_fused_k(const TMaps& tm, const FusedParams& fp, size_t smem, int grid,
                                  cudaStream_t st) {
  auto kern = fused_recon_topk<MAXT, KIND, PAIR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(threads_of(epw_of(KIND, MAXT)), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (PAIR) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  e = cudaLaunchKernelEx(&cfg, kern, tm.A, tm.B, fp);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}
template <int MAXT, bool PAIR>
static cudaError_t launch_fused_t(const TMaps& tm, const FusedParams& fp, size_t smem, int grid,
                                  cudaStream_t st) {
  // the candidate epilogue (kSym) keeps no per-row list: one instantiation
  return fp.kind == kPlain      ? launch_fused_k<MAXT, kPlain, PAIR>(tm, fp, smem, grid, st)
         : fp.kind == kSeed     ? launch_fused_k<MAXT, kSeed, PAIR>(tm, fp, smem, grid, st)
         : fp.kind == kSymList  ? launch_fused_k<5, kSymList, PAIR>(tm, fp, smem, grid, st)
                                : launch_fused_k<5, kSym, PAIR>(tm, fp, smem, grid, st);
}
template <bool PAIR>
static cudaError_t launch_fused_p(const TMaps& tm, const FusedParams& fp, int t, size_t smem,
                                  int grid, cudaStream_t s) {
  return t <= 5    ? launch_fused_t<5, PAIR>(tm, fp, smem, grid, s)
         : t <= 10 ? launch_fused_t<10, PAIR>(tm, fp, smem, grid, s)
         : t <= 16 ? launch_fused_t<16, PAIR>(tm, fp, smem, grid, s)
                   : launch_fused_t<32, PAIR>(tm, fp, smem, grid, s);
}

// fp.pair selects the CTA-pair kernel; its tensor maps are built over fp.A / fp.B with the
// given numbers of 128-row blocks
static ggm_status launch_fused(const FusedParams& fp_in, int t, int64_t ablocks, int64_t bblocks,
                               cudaStream_t s) {
  FusedParams fp = fp_in;
  if (fp.wsplit < 1 || !fp.pair) fp.wsplit = 1;
  if (fp.unit_hi <= 0) {  // default: all units of this kind
    fp.unit_lo = 0;
    fp.unit_hi = fp.kind == kPlain ? fp.RB * fp.C
                 : fp.kind >= kSym ? fp.RB * fp.wsplit
                                   : fp.RB;
  }
  if (fp.unit_step < 1) fp.unit_step = 1;
  if (fp.pm_n > 0 && (fp.kind != kSym || fp.wsplit % fp.pm_n != 0 || (fp.wsplit & 1) ||
                     (fp.wsplit / fp.pm_n != 1 && (fp.wsplit / fp.pm_n) % 2 != 0)))
    fp.pm_n = 0;
  if (fp.pm_n == 0 && fp.unit_hi <= fp.unit_lo) return GGM_OK;  // empty shard
  const size_t smem = fused_smem_bytes(fp.KA, fp.resident, fp.pair);
  const int units = unit_count<kSym>(fp);
  TMaps tm;
  memset(&tm, 0, sizeof(tm));
  cudaError_t ce;
  count_launches(1);
  if (fp.pair) {
    const uint64_t lpb = (uint64_t)2 * fp.KA * kRowsPerBlock;
    ggm_status st = make_line_tmap(&tm.A, fp.A, (uint64_t)ablocks * lpb);
    if (st == GGM_OK) st = make_line_tmap(&tm.B, fp.B, (uint64_t)bblocks * lpb);
    if (st != GGM_OK) return st;
    const int pairs = std::max(1, std::min(num_sms() / 2, units));
    ce = launch_fused_p<true>(tm, fp, t, smem, 2 * pairs, s);
  } else {
    const int grid = std::max(1, std::min(num_sms(), units));
    ce = launch_fused_p<false>(tm, fp, t, smem, grid, s);
  }
  if (ce != cudaSuccess) return fail(GGM_ERR_CUDA, "fused kernel launch: %s", cudaGetErrorString(ce));
  return GGM_OK;
}

template <int MAXT>
static void launch_merge_sym_t(const Work& w, const Plan& pl, int64_t ncand, int64_t* row_ptr,
                               int32_t* col, float* val, cudaStream_t s) {
  const int threads = 128;
  const int blocks = (int)((pl.n + threads - 1) / threads);
  // screening plans with candidates computed the pool's row offsets (recompute_pool)
  merge_sym<MAXT><<<blocks, threads, 0, s>>>(w.skey, w.sval, ncand, pl.n, pl.t, w.perm, 0, pl.n,
                                             nullptr, row_ptr, col, val,
                                             (pl.screen && ncand > 0) ? w.roff : nullptr);
}

static thread_local double g_stats[6] = {0, 0, 0, 0, 0, 0};

}  // namespace sp
}  // namespace ggm

using namespace ggm;
using namespace ggm::sp;

extern "C" void ggm_last_stats(double out[6]) {
  for (int i = 0; i < 6; ++i) out[i] = g_stats[i];
}

// Seed-call reuse (distributed symmetric scheme): ggm_sym_seed_shard leaves the scale, the
// row norms and the norm order in its workspace; the seeded shard call on the SAME workspace
// and inputs (its thr_all came from those seed calls) skips recomputing them.  Host-side
// stamps keyed by the workspace address; any other call on that workspace, or different
// inputs, recompute everything.
struct SeedStamp {
  const float* V;
  const double* lambda;
  int64_t n;
  int k, t, mode, nranks;
};
static std::mutex g_seed_mu;
static std::unordered_map<const void*, SeedStamp> g_seed_reg;
static void seed_stamp_set(const void* ws, const SeedStamp& st) {
  std::lock_guard<std::mutex> g(g_seed_mu);
  g_seed_reg[ws] = st;
}
static bool seed_stamp_take(const void* ws, const SeedStamp& st) {  // one-shot match
  std::lock_guard<std::mutex> g(g_seed_mu);
  auto it = g_seed_reg.find(ws);
  if (it == g_seed_reg.end()) return false;
  const SeedStamp o = it->second;
  g_seed_reg.erase(it);
  return o.V == st.V && o.lambda == st.lambda && o.n == st.n && o.k == st.k && o.t == st.t &&
         o.mode == st.mode && o.nranks == st.nranks;
}
static void seed_stamp_forget(const void* ws) {
  std::lock_guard<std::mutex> g(g_seed_mu);
  g_seed_reg.erase(ws);
}
// zero the per-call counters of a workspace whose scale and norm maximum are reused
__global__ void reset_pool_counters(DevScalars* sc) {
  sc->cand_overflow = 0;
  sc->coo_count = 0;
  sc->cand_alloc = 0;
  sc->cand_emitted = 0;
}

extern "C" ggm_status ggm_sparse_precision_workspace(int64_t n, int k, int64_t row_begin,
                                                     int64_t row_end,
                                                     const ggm_sparsify_opts* opts,
                                                     int64_t capacity, size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  if (opts && opts->mode != 0 && opts->mode != 1)
    return fail(GGM_ERR_INVALID_ARGUMENT, "mode=%d not in {0,1}", opts->mode);
  Plan pl;
  ggm_status st = make_plan(n, k, row_begin, row_end, opts, capacity, &pl);
  if (st != GGM_OK) return st;
  Work w;
  *bytes = carve(pl, nullptr, &w);
  return GGM_OK;
}

// 128-row blocks readable from fp.A (aliased into the B operand, or the separate A operand)
static int64_t a_blocks(const Plan& pl, int64_t row_begin) {
  return pl.alias ? pl.nBblocks - row_begin / kRowsPerBlock : pl.nAblocks;
}
static FusedParams base_params(const Plan& pl, const Work& w, int64_t n, int64_t row_begin) {
  FusedParams fp{};
  fp.B = w.Bop;
  fp.A = pl.alias ? w.Bop + (size_t)(row_begin / kRowsPerBlock) * block_bytes(pl.KA) : w.Aop;
  fp.KA = pl.KA;
  fp.KS = pl.KS;
  fp.TS = pl.TS;
  fp.resident = pl.resident;
  fp.n = n;
  fp.row_begin = row_begin;
  fp.rows = pl.rows;
  fp.kind = kPlain;
  fp.RB = (int)pl.RBu;
  fp.NT = (int)pl.NT;
  fp.pair = pl.pair;
  fp.C = (int)pl.C;
  fp.TPC = (int)pl.TPC;
  fp.NB = (int)pl.NBu;  // kSym window modulus (128- or 256-row blocks)
  fp.mode = pl.mode;
  fp.t = pl.t;
  fp.sc = w.sc;
  fp.pcol = w.pcol;
  fp.pval = w.pval;
#ifdef GGM_EPI_DEBUG
  const char* d = getenv("GGM_DEBUG_EPI");
  fp.dbg = d ? atoi(d) : 0;
#endif
  return fp;
}

// exact re-evaluation of a key-sorted pool of ncand slots: row offsets, per-row cuts, then
// the values.  The cuts pay only when rows hold many more candidates than t (the top-32
// lists of the overall rules: re-evaluation 133 -> 38 + 10 ms at n = 10^6); at ~2t per row
// (C4/C5 top-10) they keep nearly every candidate and cost a pass (C5: 2.09 vs 2.42 +
// 0.10 ms), so they run when the pool averages more than kRecCutRatio t per row (cut_mode
// 1, plans with t >= kRecCutMinT, whose epilogue stores the screened values; 2: always;
// 0: never).  t <= 0: every candidate (threshold mode).
static void recompute_pool(const Work& w, int64_t ncand, int64_t n, int k, int t, int cut_mode,
                           int sms, cudaStream_t s) {
  cand_row_offsets<<<(int)std::min<int64_t>((n + 256) / 256, sms * 16), 256, 0, s>>>(
      w.skey, ncand, n, w.roff);
  const float* cut = nullptr;
  const bool use_cut =
      t > 0 && (cut_mode == 2 || (cut_mode == 1 && ncand > (int64_t)kRecCutRatio * t * n));
  if (use_cut) {
    const int blocks = (int)std::min<int64_t>((n + 127) / 128, sms * 16);
    if (t <= 10)
      rec_cut<10><<<blocks, 128, 0, s>>>(w.roff, w.sval, n, t, k, w.rn, w.perm, &w.sc->rn_max_bits, w.sc, w.rcut);
    else if (t <= 16)
      rec_cut<16><<<blocks, 128, 0, s>>>(w.roff, w.sval, n, t, k, w.rn, w.perm, &w.sc->rn_max_bits, w.sc, w.rcut);
    else
      rec_cut<32><<<blocks, 128, 0, s>>>(w.roff, w.sval, n, t, k, w.rn, w.perm, &w.sc->rn_max_bits, w.sc, w.rcut);
    cut = w.rcut;
    count_launches(1);
  }
  const int R = (rec_stride(k) + 31) / 32;
  if (R <= 1)
    launch_recompute_r<1>(w.skey, w.sval, w.roff, n, w.Ub, k, cut, sms, s);
  else if (R == 2)
    launch_recompute_r<2>(w.skey, w.sval, w.roff, n, w.Ub, k, cut, sms, s);
  else if (R == 3)
    launch_recompute_r<3>(w.skey, w.sval, w.roff, n, w.Ub, k, cut, sms, s);
  else
    launch_recompute_r<4>(w.skey, w.sval, w.roff, n, w.Ub, k, cut, sms, s);
  count_launches(2);
}

// Symmetric scheme, phases 1-3 (replicated on every rank of the distributed form): rows in
// descending ||U_i|| order, seed pass over the largest-norm columns -> per-row lower bounds,
// rows re-ordered by bound (w.perm: bound order -> original id, w.thr_p: bounds), operand
// re-split in bound order.
// seed_ulo/seed_uhi >= 0: run only the seed pass over those units, leave the raw per-row seed
// values (norm order) in w.thr and return (a rank's share of a sharded seed).
// thr_all != nullptr: skip the seed pass and take the raw seed values of all rows from it.
static ggm_status sym_prepare(const Plan& pl, const Work& w, const float* V, const double* lambda,
                              int64_t n, int k, const FusedParams& fp, cudaStream_t s,
                              int seed_ulo = -1, int seed_uhi = -1,
                              const float* thr_all = nullptr, float tau_cap = 0.f,
                              bool norms_ready = false) {
  const int sms = num_sms();
  ggm_status st;
    // (1) rows in descending ||U_i|| order (CUB sort of the row norms), split in that order
    // (norms_ready: the row norms, their maximum and the norm order are already in the
    // workspace from this rank's seed-share call on the same inputs)
  const int64_t nthr = 2 * pl.NBu * kRowsPerBlock;
  fill_f32<<<(int)std::min<int64_t>((nthr + 255) / 256, sms * 8), 256, 0, s>>>(w.thr, nthr,
                                                                             INFINITY);
  if (!norms_ready) {
    row_norms<<<(int)std::min<int64_t>((n * 32 + 255) / 256, sms * 16), 256, 0, s>>>(
        V, lambda, n, k, w.rn, &w.sc->rn_max_bits);
    iota_i32<<<(int)std::min<int64_t>((n + 255) / 256, sms * 8), 256, 0, s>>>(w.ids, n);
    {
      size_t tb = pl.sort_temp_bytes;
      GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(w.sort_tmp, tb, w.rn, w.rn_s, w.ids,
                                                             w.perm_n, (int)n, 0, 32, s));
    }
    count_launches(4);
  } else {
    count_launches(1);
  }
  if (pl.mode == 1) {
    // threshold mode: every row's bound is τ itself (accumulator units); no seed pass
    fill_tau<<<(int)std::min<int64_t>((n + 255) / 256, sms * 8), 256, 0, s>>>(w.thr, n, fp.tau, w.sc);
    count_launches(1);
  } else if (thr_all) {
    GGM_CUDA_TRY(cudaMemcpyAsync(w.thr, thr_all, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
  } else {
    const int64_t nrows_pad = (int64_t)pl.nBblocks * kRowsPerBlock;
    if (seed_ulo >= 0) {
      // a rank's seed share reads only its own row units (A) and the first SS column tiles
      // (B): split just those rows (the replicated full split cost 0.24 ms per rank at C5)
      const int64_t R = pl.pair ? 2 * kRowsPerBlock : kRowsPerBlock;
      const int64_t b_hi = std::min<int64_t>(nrows_pad, (int64_t)pl.SS * kTileN);
      int64_t a_lo = std::min<int64_t>(nrows_pad, seed_ulo * R);
      const int64_t a_hi = std::min<int64_t>(nrows_pad, seed_uhi * R);
      launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, 0, b_hi, w.sc, w.Bop, w.perm_n);
      a_lo = std::max(a_lo, b_hi);
      if (a_hi > a_lo)
        launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, a_lo, a_hi - a_lo, w.sc,
                     w.Bop + (size_t)(a_lo / kRowsPerBlock) * block_bytes(pl.KA), w.perm_n);
      count_launches(2);
    } else {
      launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, 0, nrows_pad, w.sc, w.Bop,
                   w.perm_n);
      count_launches(1);
    }
    // (2) seed: per row, the t-th largest hi·hi chunk maximum over the first SS column
    // tiles (the largest-norm columns), minus the hi·hi rounding bound -> lower bound b_i
    FusedParams sp = fp;
    sp.kind = kSeed;
    sp.RB = (int)pl.NBu;
    sp.SS = pl.SS;
    sp.thr_out = w.thr;
    if (seed_ulo >= 0) {
      sp.unit_lo = seed_ulo;
      sp.unit_hi = seed_uhi;
    }
    st = launch_fused(sp, pl.t, a_blocks(pl, 0), pl.nBblocks, s);
    if (st != GGM_OK) return st;
    if (seed_ulo >= 0) return GGM_OK;
  }
  if (pl.mode != 1) {
    seed_bounds<<<(int)std::min<int64_t>((n + 255) / 256, sms * 8), 256, 0, s>>>(
        w.thr, w.rn_s, &w.sc->rn_max_bits, n, k, w.sc);
    count_launches(1);
    if (tau_cap > 0.f) {  // bound_i = min(top-t bound_i, τ): also every entry above τ
      cap_tau<<<(int)std::min<int64_t>((n + 255) / 256, sms * 8), 256, 0, s>>>(w.thr, n, tau_cap, w.sc);
      count_launches(1);
    }
  }
  // (3) order rows (= columns) by their bound: sort (bound, original id) -> the final
  // permutation and the permuted bounds; re-split in that order, so the 32 columns of
  // every epilogue chunk carry nearly equal bounds
  {
    size_t tb = pl.sort_temp_bytes;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, tb, w.thr, w.thr_p, w.perm_n, w.perm,
                                                 (int)n, 0, 32, s));
  }
  fill_f32<<<(int)std::min<int64_t>((nthr - n + 255) / 256 + 1, sms * 8), 256, 0, s>>>(
      w.thr_p + n, nthr - n, INFINITY);
  if (pl.screen) {
    screen_bounds<<<(int)std::min<int64_t>((nthr + 255) / 256, sms * 8), 256, 0, s>>>(
        w.thr_p, w.rn, w.perm, &w.sc->rn_max_bits, n, k, nthr, w.sc, w.thr_s);
    count_launches(1);
  }
  chunk_min32<<<(int)std::min<int64_t>((nthr / 32 + 255) / 256, sms * 8), 256, 0, s>>>(
      pl.screen ? w.thr_s : w.thr_p, nthr / 32, w.thr_cmin);
  chunk_min32<<<(int)std::min<int64_t>((nthr / 8 + 255) / 256, sms * 8), 256, 0, s>>>(
      pl.screen ? w.thr_s : w.thr_p, nthr / 8, w.thr_cmin8, 8);
  count_launches(1);
  count_launches(1);
  if (pl.screen) {
    gather_u_bound<<<(int)std::min<int64_t>((n * 32 + 255) / 256, sms * 16), 256, 0, s>>>(
        V, lambda, w.perm, n, k, w.Ub);
    count_launches(1);
  }
  {
    launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, 0, (int64_t)pl.nBblocks * kRowsPerBlock, w.sc, w.Bop,
        w.perm);
  }
  count_launches(3);
  GGM_CUDA_TRY(cudaGetLastError());
  return GGM_OK;
}

// Phase 4: the symmetric main kernel over units unit_lo, unit_lo + unit_step, ... < unit_hi
// (all units on one GPU; rank r of N takes units r, r + N, ... in the distributed form, so
// every rank gets the same mix of bound levels — contiguous shares left the last ranks with
// most of the candidate emission, tools/sim_ranks.py); candidates -> w.ckey / w.cval.
static ggm_status sym_main(const Plan& pl, const Work& w, FusedParams fp, int unit_lo,
                           int unit_hi, cudaStream_t s, int unit_step = 1, int pm_n = 0) {
  fp.kind = kSym;
  fp.RB = (int)pl.NBu;
  fp.thr = pl.screen ? w.thr_s : w.thr_p;
  fp.thr_min = w.thr_cmin;
  fp.thr_min8 = w.thr_cmin8;
  fp.screen = pl.screen;
  fp.cand_vals = (!pl.screen || pl.rec_cut) ? 1 : 0;
  fp.perm = w.perm;
  fp.cand_key = w.ckey;
  fp.cand_val = w.cval;
  fp.cand_total = pl.cand_total;
  fp.wsplit = pl.pair ? kWindowSplit : 1;
  fp.unit_lo = unit_lo;
  fp.unit_hi = unit_hi * fp.wsplit;  // unit_hi counts row blocks; units = sub-windows
  fp.unit_step = unit_step;
  fp.pm_n = pm_n;
  fp.pm_r = unit_lo;
  if (pm_n == 0 && fp.unit_hi <= unit_lo) return GGM_OK;
  return launch_fused(fp, pl.t, a_blocks(pl, 0), pl.nBblocks, s);
}

extern "C" ggm_status ggm_sparse_precision(int64_t n, int k, const float* V, const double* lambda,
                                           int64_t row_begin, int64_t row_end,
                                           const ggm_sparsify_opts* opts, int64_t* row_ptr,
                                           int32_t* col, float* val, int64_t capacity,
                                           int64_t* nnz_out, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  seed_stamp_forget(workspace);
  if (!V || !lambda || !row_ptr || !nnz_out || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (opts && opts->mode != 0 && opts->mode != 1)
    return fail(GGM_ERR_INVALID_ARGUMENT, "mode=%d not in {0,1}", opts->mode);
  Plan pl;
  ggm_status st = make_plan(n, k, row_begin, row_end, opts, capacity, &pl);
  if (st != GGM_OK) return st;
  if (pl.mode == 0 && capacity < pl.rows * pl.t)
    return fail(GGM_ERR_INVALID_ARGUMENT, "capacity %lld < rows*t_eff = %lld",
                (long long)capacity, (long long)(pl.rows * pl.t));
  if ((pl.mode == 0 || capacity > 0) && (!col || !val))
    return fail(GGM_ERR_INVALID_ARGUMENT, "col/val NULL");
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  Work w;
  const size_t need = carve(pl, workspace, &w);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  if (!ggm_device_supported())
    return fail(GGM_ERR_CUDA, "current device is not compute capability 10.0 (sm_100a)");

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  reset_launches();
  for (double& x : g_stats) x = 0.0;
  g_stats[4] = 16.0 * ((pl.screen ? 1 : 3) * pl.KS + pl.TS);  // MMA K elements issued per evaluated entry
  g_stats[5] = pl.pair;
  EventTimer tm(timing_enabled(), s);
  tm.mark(0);
  GGM_CUDA_TRY(cudaMemsetAsync(w.sc, 0, sizeof(DevScalars), s));
  const int sms = num_sms();
  {
    const int64_t total = n * (int64_t)k;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, sms * 8));
    absmax_check<<<grid, 256, 0, s>>>(V, lambda, n, k, w.sc);
    scale_finalize<<<1, 1, 0, s>>>(w.sc);
    if (!pl.sym) {  // (the symmetric scheme splits in norm order below)
      launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, 0, (int64_t)pl.nBblocks * kRowsPerBlock, w.sc,
          w.Bop);
      count_launches(1);
    }
    count_launches(2);
    if (!pl.alias) {
      launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, row_begin, (int64_t)pl.nAblocks * kRowsPerBlock,
          w.sc, w.Aop);
      count_launches(1);
    }
    GGM_CUDA_TRY(cudaGetLastError());
  }
  // mode 1 tail (plain scheme, and the symmetric scheme after its candidates became COO):
  // count, capacity check, sort COO by (row, col), assemble CSR
  auto mode1_tail = [&]() -> ggm_status {
    DevScalars hs;
    GGM_CUDA_TRY(cudaMemcpyAsync(&hs, w.sc, sizeof(hs), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    if (hs.flags & 1) return fail(GGM_ERR_DOMAIN, "V contains non-finite values");
    if (hs.flags & 2) return fail(GGM_ERR_DOMAIN, "lambda must be finite and > 0 (P:65)");
    const int64_t count = (int64_t)hs.coo_count;
    *nnz_out = count;
    if (count > capacity) {
      tm.mark(3);
      tm.finish();
      return fail(GGM_ERR_CAPACITY, "threshold mode: %lld entries > capacity %lld",
                  (long long)count, (long long)capacity);
    }
    if (count > 0) {
      size_t tb = pl.coo_temp_bytes;
      GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, w.key_in, w.key_out, w.cv_in,
                                                   w.cv_out, count, 0, 64, s));
      const int blocks = (int)std::min<int64_t>((count + 256) / 256 + 1, sms * 8);
      coo_to_csr<<<blocks, 256, 0, s>>>(w.key_out, w.cv_out, count, n, pl.rows, row_ptr, col, val);
      count_launches(1);
    } else {
      zero_row_ptr<<<(int)std::min<int64_t>((pl.rows + 256) / 256 + 1, sms * 8), 256, 0, s>>>(
          row_ptr, pl.rows);
      count_launches(1);
    }
    GGM_CUDA_TRY(cudaGetLastError());
    tm.mark(3);
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    tm.finish();
    return GGM_OK;
  };
  FusedParams fp = base_params(pl, w, n, row_begin);
  if (pl.sym) {
    fp.tau = pl.mode == 1 ? opts->tau : 0.f;
    st = sym_prepare(pl, w, V, lambda, n, k, fp, s);
    if (st != GGM_OK) return st;
    tm.mark(1);
    st = sym_main(pl, w, fp, 0, (int)pl.NBu, s);
    if (st != GGM_OK) return st;
    tm.mark(2);
    // sort the candidate pool by target row (unused slots carry UINT32_MAX -> sorted last)
    DevScalars hs;
    GGM_CUDA_TRY(cudaMemcpyAsync(&hs, w.sc, sizeof(hs), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    if (hs.flags & 1) return fail(GGM_ERR_DOMAIN, "V contains non-finite values");
    if (hs.flags & 2) return fail(GGM_ERR_DOMAIN, "lambda must be finite and > 0 (P:65)");
    const int hovf = hs.cand_overflow;
    if (pl.mode == 1) {
      if (hovf) {
        // pool exhausted: the plain threshold pass (exact) from an un-permuted split
        launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, 0, (int64_t)pl.nBblocks * kRowsPerBlock, w.sc, w.Bop);
        count_launches(1);
        Plan bp = pl;
        bp.sym = 0;
        FusedParams op = base_params(bp, w, n, 0);
        op.row_ptr = row_ptr;
        op.tau = opts->tau;
        op.coo_key = w.key_in;
        op.coo_val = w.cv_in;
        op.coo_count = &w.sc->coo_count;
        op.capacity = capacity;
        st = launch_fused(op, pl.t, a_blocks(pl, 0), pl.nBblocks, s);
        if (st != GGM_OK) return st;
        g_stats[0] = 0;
        g_stats[3] = 1;
        return mode1_tail();
      }
      const int64_t ncand = (int64_t)std::min<unsigned long long>(hs.cand_alloc, pl.cand_total);
      if (ncand > 0) {
        size_t tb = pl.sort_temp_bytes;
        int ebits = 1;
        while ((int64_t(1) << ebits) <= n) ++ebits;
        GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, tb, w.ckey, w.skey, w.cval,
                                                     w.sval, ncand, 0, ebits, s));
        if (pl.screen) {  // exact values of every screened candidate (no top-t filter)
          recompute_pool(w, ncand, n, k, 0, 0, sms, s);
        }
        sym_threshold_coo<<<(int)std::min<int64_t>((ncand + 255) / 256, sms * 16), 256, 0, s>>>(
            w.skey, w.sval, ncand, n, w.perm, opts->tau, capacity, &w.sc->coo_count, w.key_in,
            w.cv_in);
        count_launches(1);
      }
      g_stats[0] = 2;
      g_stats[2] = (double)hs.cand_emitted;
      return mode1_tail();
    }
    if (hovf) {
      // the candidate pool filled up: recompute the whole axis with the plain scheme (exact)
      // from an un-permuted split
      {
        launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, 0, (int64_t)pl.nBblocks * kRowsPerBlock, w.sc, w.Bop);
        count_launches(1);
      }
      Plan bp = pl;
      bp.sym = 0;
      FusedParams op = base_params(bp, w, n, 0);
      op.row_ptr = row_ptr;
      if (pl.C == 1) {
        op.col = col;
        op.val = val;
      }
      st = launch_fused(op, pl.t, a_blocks(pl, 0), pl.nBblocks, s);
      if (st != GGM_OK) return st;
      if (pl.C > 1) {
        const int blocks = (int)((pl.rows + 127) / 128);
        if (pl.t <= 5)
          merge_partials<5><<<blocks, 128, 0, s>>>(w.pcol, w.pval, pl.rows, (int)pl.C, pl.t, row_ptr, col, val);
        else if (pl.t <= 10)
          merge_partials<10><<<blocks, 128, 0, s>>>(w.pcol, w.pval, pl.rows, (int)pl.C, pl.t, row_ptr, col, val);
        else if (pl.t <= 16)
          merge_partials<16><<<blocks, 128, 0, s>>>(w.pcol, w.pval, pl.rows, (int)pl.C, pl.t, row_ptr, col, val);
        else
          merge_partials<32><<<blocks, 128, 0, s>>>(w.pcol, w.pval, pl.rows, (int)pl.C, pl.t, row_ptr, col, val);
        count_launches(1);
      }
      tm.mark(3);
      GGM_CUDA_TRY(cudaStreamSynchronize(s));
      tm.finish();
      g_stats[0] = 0;
      g_stats[1] = (double)(pl.pair ? 2 * pl.RBu : pl.RB) * kRowsPerBlock * pl.NT * kTileN;
      g_stats[3] = 1;
      *nnz_out = pl.rows * pl.t;
      return GGM_OK;
    }
    const int64_t ncand = (int64_t)std::min<unsigned long long>(hs.cand_alloc, pl.cand_total);
    if (ncand > 0) {
      size_t tb = pl.sort_temp_bytes;
      // keys are permuted row ids < n; unused slots (UINT32_MAX) keep all low bits set, so
      // sorting on the low ebits bits (2^ebits > n) still places them last
      int ebits = 1;
      while ((int64_t(1) << ebits) <= n) ++ebits;
      GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, tb, w.ckey, w.skey, w.cval, w.sval,
                                                   ncand, 0, ebits, s));
      if (pl.screen) {  // exact values of the screened candidates
        recompute_pool(w, ncand, n, k, pl.t, pl.rec_cut, sms, s);
      }
    }
    if (pl.t <= 5)
      launch_merge_sym_t<5>(w, pl, ncand, row_ptr, col, val, s);
    else if (pl.t <= 10)
      launch_merge_sym_t<10>(w, pl, ncand, row_ptr, col, val, s);
    else if (pl.t <= 16)
      launch_merge_sym_t<16>(w, pl, ncand, row_ptr, col, val, s);
    else
      launch_merge_sym_t<32>(w, pl, ncand, row_ptr, col, val, s);
    count_launches(1);
    GGM_CUDA_TRY(cudaGetLastError());
    tm.mark(3);
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    tm.finish();
    double evaluated = 0.0;  // entries evaluated by the symmetric pass (incl. masked halves)
    for (int64_t b = 0; b < pl.NBu; ++b) {
      const int64_t NBu = pl.NBu;
      const int64_t W = (NBu & 1) ? (NBu + 1) / 2 : NBu / 2 + (b < NBu / 2 ? 1 : 0);
      evaluated += pl.pair ? (double)W * 2 * kRowsPerBlock * kTileN
                           : (double)((W + 1) / 2) * kRowsPerBlock * kTileN;
    }
    g_stats[0] = 2;
    g_stats[1] = evaluated;
    g_stats[2] = (double)hs.cand_emitted;  // written; the sort above covers ncand reserved slots
    g_stats[3] = 0;
    *nnz_out = pl.rows * pl.t;
    return GGM_OK;
  }
  fp.row_ptr = row_ptr;
  fp.col = (pl.mode == 0 && pl.C == 1) ? col : nullptr;
  fp.val = (pl.mode == 0 && pl.C == 1) ? val : nullptr;
  fp.tau = pl.mode == 1 ? opts->tau : 0.f;
  fp.coo_key = w.key_in;
  fp.coo_val = w.cv_in;
  fp.coo_count = &w.sc->coo_count;
  fp.capacity = pl.mode == 1 ? capacity : 0;
  tm.mark(1);
  st = launch_fused(fp, pl.t, a_blocks(pl, row_begin), pl.nBblocks, s);
  if (st != GGM_OK) return st;
  tm.mark(2);
  g_stats[0] = 0;
  g_stats[1] = (double)(pl.pair ? 2 * pl.RBu : pl.RB) * kRowsPerBlock * pl.NT * kTileN;

  DevScalars hs;
  if (pl.mode == 0) {
    if (pl.C > 1) {
      const int threads = 128;
      const int blocks = (int)((pl.rows + threads - 1) / threads);
      if (pl.t <= 5)
        merge_partials<5><<<blocks, threads, 0, s>>>(w.pcol, w.pval, pl.rows, (int)pl.C, pl.t,
                                                     row_ptr, col, val);
      else if (pl.t <= 10)
        merge_partials<10><<<blocks, threads, 0, s>>>(w.pcol, w.pval, pl.rows, (int)pl.C, pl.t,
                                                      row_ptr, col, val);
      else if (pl.t <= 16)
        merge_partials<16><<<blocks, threads, 0, s>>>(w.pcol, w.pval, pl.rows, (int)pl.C, pl.t,
                                                      row_ptr, col, val);
      else
        merge_partials<32><<<blocks, threads, 0, s>>>(w.pcol, w.pval, pl.rows, (int)pl.C, pl.t,
                                                      row_ptr, col, val);
      GGM_CUDA_TRY(cudaGetLastError());
      count_launches(1);
    }
    tm.mark(3);
    GGM_CUDA_TRY(cudaMemcpyAsync(&hs, w.sc, sizeof(hs), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    tm.finish();
    if (hs.flags & 1) return fail(GGM_ERR_DOMAIN, "V contains non-finite values");
    if (hs.flags & 2) return fail(GGM_ERR_DOMAIN, "lambda must be finite and > 0 (P:65)");
    *nnz_out = pl.rows * pl.t;
    return GGM_OK;
  }
  // mode 1: count, capacity check, sort COO by (row, col), assemble CSR
  return mode1_tail();
}

// ------------------------------------------------------------------ distributed symmetric scheme
// (DESIGN.md §5): every rank runs the replicated phases 1-3 and its contiguous share of the
// symmetric units, buckets its candidates by the rank that owns their target row, the caller
// exchanges the buckets (all-to-all), and each rank merges the candidates of its own rows.

static ggm_status sym_shard_plan(int64_t n, int k, const ggm_sparsify_opts* opts, Plan* pl) {
  if (!opts) return fail(GGM_ERR_INVALID_ARGUMENT, "opts is NULL");
  ggm_sparsify_opts o = *opts;
  o.symmetric = 1;
  ggm_status st = make_plan(n, k, 0, n, &o, n * (int64_t)std::max(1, std::min<int>(o.topk, (int)(n - 1))), pl);
  if (st != GGM_OK) return st;
  if (!pl->sym)
    return fail(GGM_ERR_UNSUPPORTED, "distributed symmetric scheme needs mode 0 and k <= 128");
  return GGM_OK;
}

// Part-major share of the distributed symmetric units (0: rank-strided); GGM_SYM_ASSIGN=strided
// forces the rank-strided form (A/B, tests).
static int sym_part_major(const Plan& pl, int nranks) {
  const char* e = getenv("GGM_SYM_ASSIGN");
  if (e && strcmp(e, "strided") == 0) return 0;
  const int q = nranks > 0 ? kWindowSplit / nranks : 0;
  return (nranks > 1 && pl.pair && kWindowSplit % 2 == 0 && kWindowSplit % nranks == 0 &&
          (q == 1 || q % 2 == 0)) ? nranks : 0;
}
// owner rank of unit (sub-window part, row block b) under the folded part-major share
static int sym_pm_owner(int part, int64_t b, int nranks) {
  const int j = std::min(part, kWindowSplit - 1 - part);
  if (kWindowSplit / nranks == 1) return (b & 1) ? kWindowSplit - 1 - part : part;
  return j % nranks;
}
static int64_t sym_unit_rows(const Plan& pl) { return pl.pair ? 2 * kRowsPerBlock : kRowsPerBlock; }
static int64_t sym_unit_lo(const Plan& pl, int rank, int nranks) {
  return pl.NBu * (int64_t)rank / nranks;
}

extern "C" int64_t ggm_sym_rows_begin(int64_t n, int k, const ggm_sparsify_opts* opts, int rank,
                                      int nranks) {
  Plan pl;
  if (nranks < 1 || rank < 0 || rank > nranks) return -1;
  if (sym_shard_plan(n, k, opts, &pl) != GGM_OK) return -1;
  return std::min<int64_t>(n, sym_unit_lo(pl, rank, nranks) * sym_unit_rows(pl));
}

extern "C" ggm_status ggm_sparse_precision_sym_shard_workspace(int64_t n, int k,
                                                                const ggm_sparsify_opts* opts,
                                                                size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  Plan pl;
  ggm_status st = sym_shard_plan(n, k, opts, &pl);
  if (st != GGM_OK) return st;
  Work w;
  *bytes = carve(pl, nullptr, &w) + 256 + sizeof(int64_t) * 2 * (GGM_MAX_RANKS + 1);
  return GGM_OK;
}

static ggm_status sym_shard_impl(
    int64_t n, int k, const float* V, const double* lambda, const ggm_sparsify_opts* opts,
    int rank, int nranks, uint32_t* cand_key, uint32_t* cand_val, int64_t cand_capacity,
    int64_t* counts, int32_t* perm, void* workspace, size_t workspace_bytes, void* stream,
    const float* thr_all);

extern "C" ggm_status ggm_sparse_precision_sym_shard(
    int64_t n, int k, const float* V, const double* lambda, const ggm_sparsify_opts* opts,
    int rank, int nranks, uint32_t* cand_key, uint32_t* cand_val, int64_t cand_capacity,
    int64_t* counts, int32_t* perm, void* workspace, size_t workspace_bytes, void* stream) {
  return sym_shard_impl(n, k, V, lambda, opts, rank, nranks, cand_key, cand_val, cand_capacity,
                        counts, perm, workspace, workspace_bytes, stream, nullptr);
}

extern "C" ggm_status ggm_sparse_precision_sym_shard_seeded(
    int64_t n, int k, const float* V, const double* lambda, const ggm_sparsify_opts* opts,
    int rank, int nranks, const float* thr_all, uint32_t* cand_key, uint32_t* cand_val,
    int64_t cand_capacity, int64_t* counts, int32_t* perm, void* workspace,
    size_t workspace_bytes, void* stream) {
  if (!thr_all) return fail(GGM_ERR_INVALID_ARGUMENT, "thr_all is NULL");
  return sym_shard_impl(n, k, V, lambda, opts, rank, nranks, cand_key, cand_val, cand_capacity,
                        counts, perm, workspace, workspace_bytes, stream, thr_all);
}

extern "C" ggm_status ggm_sym_seed_shard(int64_t n, int k, const float* V, const double* lambda,
                                         const ggm_sparsify_opts* opts, int rank, int nranks,
                                         float* thr_out, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (!V || !lambda || !thr_out || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (nranks < 1 || nranks > GGM_MAX_RANKS || rank < 0 || rank >= nranks)
    return fail(GGM_ERR_INVALID_ARGUMENT, "rank %d / nranks %d invalid", rank, nranks);
  seed_stamp_forget(workspace);
  Plan pl;
  ggm_status st = sym_shard_plan(n, k, opts, &pl);
  if (st != GGM_OK) return st;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  Work w;
  const size_t need = carve(pl, workspace, &w);
  if (workspace_bytes < need) return fail(GGM_ERR_INVALID_ARGUMENT, "workspace too small");
  if (!ggm_device_supported())
    return fail(GGM_ERR_CUDA, "current device is not compute capability 10.0 (sm_100a)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  reset_launches();
  const int sms = num_sms();
  GGM_CUDA_TRY(cudaMemsetAsync(w.sc, 0, sizeof(DevScalars), s));
  {
    const int64_t total = n * (int64_t)k;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, sms * 8));
    absmax_check<<<grid, 256, 0, s>>>(V, lambda, n, k, w.sc);
    scale_finalize<<<1, 1, 0, s>>>(w.sc);
    count_launches(2);
  }
  FusedParams fp = base_params(pl, w, n, 0);
  // seed units (row blocks, equal work each): an even split
  const int ulo = (int)(pl.NBu * rank / nranks), uhi = (int)(pl.NBu * (rank + 1) / nranks);
  st = sym_prepare(pl, w, V, lambda, n, k, fp, s, ulo, uhi);
  if (st != GGM_OK) return st;
  GGM_CUDA_TRY(cudaMemcpyAsync(thr_out, w.thr, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  DevScalars hs;
  GGM_CUDA_TRY(cudaMemcpy(&hs, w.sc, sizeof(hs), cudaMemcpyDeviceToHost));
  if (hs.flags & 1) return fail(GGM_ERR_DOMAIN, "V contains non-finite values");
  if (hs.flags & 2) return fail(GGM_ERR_DOMAIN, "lambda must be finite and > 0 (P:65)");
  seed_stamp_set(workspace, SeedStamp{V, lambda, n, k, opts->topk, opts->mode, nranks});
  return GGM_OK;
}

static ggm_status sym_shard_impl(
    int64_t n, int k, const float* V, const double* lambda, const ggm_sparsify_opts* opts,
    int rank, int nranks, uint32_t* cand_key, uint32_t* cand_val, int64_t cand_capacity,
    int64_t* counts, int32_t* perm, void* workspace, size_t workspace_bytes, void* stream,
    const float* thr_all) {
  if (!V || !lambda || !cand_key || !cand_val || !counts || !perm || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (nranks < 1 || nranks > GGM_MAX_RANKS || rank < 0 || rank >= nranks)
    return fail(GGM_ERR_INVALID_ARGUMENT, "rank %d / nranks %d invalid", rank, nranks);
  Plan pl;
  ggm_status st = sym_shard_plan(n, k, opts, &pl);
  if (st != GGM_OK) return st;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  Work w;
  const size_t need = carve(pl, workspace, &w);
  const size_t extra = 256 + sizeof(int64_t) * 2 * (GGM_MAX_RANKS + 1);
  if (workspace_bytes < need + extra)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes,
                need + extra);
  if (!ggm_device_supported())
    return fail(GGM_ERR_CUDA, "current device is not compute capability 10.0 (sm_100a)");
  int64_t* d_lo = reinterpret_cast<int64_t*>(static_cast<uint8_t*>(workspace) + ((need + 255) & ~size_t(255)));
  int64_t* d_bnd = d_lo + (GGM_MAX_RANKS + 1);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  reset_launches();
  for (double& x : g_stats) x = 0.0;
  EventTimer tm(timing_enabled(), s);
  tm.mark(0);
  const int sms = num_sms();
  // seeded call on the workspace of this rank's seed share with the same inputs: the scale,
  // the domain flags, the row norms and the norm order are reused (seed_stamp_take)
  const bool reuse =
      thr_all && seed_stamp_take(workspace, SeedStamp{V, lambda, n, k, opts->topk, opts->mode, nranks});
  if (!thr_all) seed_stamp_forget(workspace);
  if (reuse) {
    reset_pool_counters<<<1, 1, 0, s>>>(w.sc);
    count_launches(1);
  } else {
    GGM_CUDA_TRY(cudaMemsetAsync(w.sc, 0, sizeof(DevScalars), s));
    const int64_t total = n * (int64_t)k;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, sms * 8));
    absmax_check<<<grid, 256, 0, s>>>(V, lambda, n, k, w.sc);
    scale_finalize<<<1, 1, 0, s>>>(w.sc);
    count_launches(2);
  }
  FusedParams fp = base_params(pl, w, n, 0);
  st = sym_prepare(pl, w, V, lambda, n, k, fp, s, -1, -1, thr_all, 0.f, reuse);
  if (st != GGM_OK) return st;
  tm.mark(1);
  // this rank's block pairs (the merge ownership of rows below stays the contiguous
  // bound-order ranges): folded part-major when nranks divides the sub-window count (a
  // rank owns sub-windows j and wsplit-1-j of EVERY row block, row blocks in order, so the
  // CTAs of a wave stream overlapping column windows through L2 as at N = 1; unit_of), else
  // rank-strided units rank, rank + nranks, ...; both give every rank the same mix of bound
  // levels (C5, N = 8 per-rank main 11.9-13.3 ms strided, 11.3-12.8 unfolded part-major)
  const int pm = sym_part_major(pl, nranks);
  st = sym_main(pl, w, fp, rank, (int)pl.NBu, s, nranks, pm);
  if (st != GGM_OK) return st;
  tm.mark(2);
  DevScalars hs;
  GGM_CUDA_TRY(cudaMemcpyAsync(&hs, w.sc, sizeof(hs), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hs.flags & 1) return fail(GGM_ERR_DOMAIN, "V contains non-finite values");
  if (hs.flags & 2) return fail(GGM_ERR_DOMAIN, "lambda must be finite and > 0 (P:65)");
  if (hs.cand_overflow)
    return fail(GGM_ERR_CAPACITY, "symmetric candidate pool overflow (use the row-sharded plain scheme)");
  const int64_t ncand = (int64_t)std::min<unsigned long long>(hs.cand_alloc, pl.cand_total);
  int ebits = 1;
  while ((int64_t(1) << ebits) <= n) ++ebits;
  if (ncand > 0) {
    size_t tb = pl.sort_temp_bytes;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, tb, w.ckey, w.skey, w.cval, w.sval,
                                                 ncand, 0, ebits, s));
    if (pl.screen) {  // exact values before the buckets leave this rank
      recompute_pool(w, ncand, n, k, pl.t, pl.rec_cut, sms, s);
    }
  }
  // destination buckets: rank r owns bound-order rows [lo_r, lo_{r+1}); unused pool slots
  // (key UINT32_MAX) sort after every real key
  std::vector<int64_t> lo(nranks + 1);
  for (int r = 0; r <= nranks; ++r)
    lo[r] = std::min<int64_t>(n, sym_unit_lo(pl, r, nranks) * sym_unit_rows(pl));
  GGM_CUDA_TRY(cudaMemcpyAsync(d_lo, lo.data(), sizeof(int64_t) * (nranks + 1),
                               cudaMemcpyHostToDevice, s));
  bucket_bounds<<<1, 64, 0, s>>>(w.skey, ncand, d_lo, nranks, d_bnd);
  count_launches(1);
  std::vector<int64_t> bnd(nranks + 1);
  GGM_CUDA_TRY(cudaMemcpyAsync(bnd.data(), d_bnd, sizeof(int64_t) * (nranks + 1),
                               cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t total = bnd[nranks] - bnd[0];
  for (int r = 0; r < nranks; ++r) counts[r] = bnd[r + 1] - bnd[r];
  if (total > cand_capacity)
    return fail(GGM_ERR_CAPACITY, "%lld candidates > capacity %lld", (long long)total,
                (long long)cand_capacity);
  if (total > 0) {
    GGM_CUDA_TRY(cudaMemcpyAsync(cand_key, w.skey + bnd[0], sizeof(uint32_t) * total,
                                 cudaMemcpyDeviceToDevice, s));
    GGM_CUDA_TRY(cudaMemcpyAsync(cand_val, w.sval + bnd[0], sizeof(uint2) * total,
                                 cudaMemcpyDeviceToDevice, s));
  }
  GGM_CUDA_TRY(cudaMemcpyAsync(perm, w.perm, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  tm.mark(3);
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  tm.finish();
  double evaluated = 0.0;  // entries evaluated by this rank's units
  const int64_t ws = pl.pair ? kWindowSplit : 1;
  for (int64_t u = 0; u < pl.NBu * ws; ++u) {  // this rank's units
    const int64_t NBu = pl.NBu, part = u / NBu, b = u % NBu;
    if (pm ? (sym_pm_owner((int)part, b, nranks) != rank) : (u % nranks != rank)) continue;
    const int64_t W = (NBu & 1) ? (NBu + 1) / 2 : NBu / 2 + (b < NBu / 2 ? 1 : 0);
    evaluated += pl.pair ? (double)((part + 1) * W / ws - part * W / ws) * 2 * kRowsPerBlock * kTileN
                         : (double)((W + 1) / 2) * kRowsPerBlock * kTileN;
  }
  g_stats[0] = 2;
  g_stats[1] = evaluated;
  g_stats[2] = (double)total;
  g_stats[4] = 16.0 * ((pl.screen ? 1 : 3) * pl.KS + pl.TS);
  g_stats[5] = pl.pair;
  return GGM_OK;
}

extern "C" ggm_status ggm_sym_merge_workspace(int64_t ncand, size_t* bytes) {
  if (!bytes || ncand < 0) return fail(GGM_ERR_INVALID_ARGUMENT, "bad argument");
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint2*)nullptr, (uint2*)nullptr, std::max<int64_t>(ncand, 1));
  const size_t a = ((size_t)std::max<int64_t>(ncand, 1) * sizeof(uint32_t) + 255) & ~size_t(255);
  const size_t b = ((size_t)std::max<int64_t>(ncand, 1) * sizeof(uint2) + 255) & ~size_t(255);
  *bytes = a + b + tb + 256;
  return GGM_OK;
}

extern "C" ggm_status ggm_sym_merge(int64_t n, int t, const uint32_t* cand_key,
                                    const uint32_t* cand_val, int64_t ncand, const int32_t* perm,
                                    int64_t row_begin, int64_t row_end, int64_t* row_id,
                                    int32_t* col, float* val, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  seed_stamp_forget(workspace);
  if (!perm || !row_id || !col || !val || (ncand > 0 && (!cand_key || !cand_val)) || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (n < 2 || row_begin < 0 || row_end > n || row_begin > row_end || ncand < 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "row range / n / ncand invalid");
  if (t < 1 || t > GGM_MAX_TOPK) return fail(GGM_ERR_INVALID_ARGUMENT, "t=%d invalid", t);
  const int te = (int)std::min<int64_t>(t, n - 1);
  size_t need = 0;
  ggm_sym_merge_workspace(ncand, &need);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  reset_launches();
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const size_t a = ((size_t)std::max<int64_t>(ncand, 1) * sizeof(uint32_t) + 255) & ~size_t(255);
  const size_t b = ((size_t)std::max<int64_t>(ncand, 1) * sizeof(uint2) + 255) & ~size_t(255);
  uint32_t* skey = reinterpret_cast<uint32_t*>(ws);
  uint2* sval = reinterpret_cast<uint2*>(ws + a);
  void* tmp = ws + a + b;
  if (ncand > 0) {
    int ebits = 1;
    while ((int64_t(1) << ebits) <= n) ++ebits;
    size_t tb = need - a - b - 256;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, cand_key, skey,
                                                 reinterpret_cast<const uint2*>(cand_val), sval,
                                                 ncand, 0, ebits, s));
  }
  const int64_t rows = row_end - row_begin;
  if (rows > 0) {
    const int threads = 128;
    const int blocks = (int)((rows + threads - 1) / threads);
    if (te <= 5)
      merge_sym<5><<<blocks, threads, 0, s>>>(skey, sval, ncand, n, te, perm, row_begin, row_end, row_id, nullptr, col, val);
    else if (te <= 10)
      merge_sym<10><<<blocks, threads, 0, s>>>(skey, sval, ncand, n, te, perm, row_begin, row_end, row_id, nullptr, col, val);
    else if (te <= 16)
      merge_sym<16><<<blocks, threads, 0, s>>>(skey, sval, ncand, n, te, perm, row_begin, row_end, row_id, nullptr, col, val);
    else
      merge_sym<32><<<blocks, threads, 0, s>>>(skey, sval, ncand, n, te, perm, row_begin, row_end, row_id, nullptr, col, val);
    count_launches(1);
    GGM_CUDA_TRY(cudaGetLastError());
  }
  return GGM_OK;
}

// ------------------------------------------------------------------ whole-graph edge rules
// (DESIGN.md §4 "overall"): keep the N largest edges overall by
// score |ψ_ij| (or |ψ_ij| / sqrt(w_i w_j) with w_i = Σ_{k≠i}|ψ_ik|, down-weighting high-degree
// vertices), plus each vertex's m best edges.  Down-weighting is a diagonal similarity:
// score_ij = |ψ'_ij| for Ψ' = D^-1/2 Ψ D^-1/2 = U' U'^T with U' = D^-1/2 U, so every pass runs
// on the row-scaled factors V' = V ⊙ w^-1/2.  Steps: (1) row masses (plain tiles, mode 2);
// (2) per-row top-t1 of Ψ' (t1 >= max(m, ceil(2N/n))) -> a lower bound L of the N-th largest
// score (the smallest row t1-th value, and the 2N-th largest listed value: both are scores of
// >= N distinct pairs); (3) every directed entry with score >= L (threshold mode); (4) keep
// i < j, rank (score desc, i, j) with two stable radix sorts, take N, add the min-edges from
// (2), de-duplicate; (5) symmetric CSR with ψ_ij = ψ'_ij · sqrt(w_i w_j).

namespace ggm {
namespace sp {

// x *= 2^-2e (the row masses from accumulator units to ψ units; a power of two: exact)
__global__ void scale_pow2(double* __restrict__ x, int64_t n, const DevScalars* __restrict__ sc) {
  const double f = ldexp(1.0, -2 * sc->exp2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= f;
}
__global__ void scale_rows(const float* __restrict__ V, const double* __restrict__ w, int64_t n,
                           int k, float* __restrict__ Vs, double* __restrict__ sq) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * (int64_t)k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / k;
    const double wr = w ? w[r] : 1.0;
    const double rs = wr > 0.0 ? 1.0 / sqrt(wr) : 0.0;
    Vs[i] = (float)((double)V[i] * rs);
    if (i % k == 0) sq[r] = wr > 0.0 ? sqrt(wr) : 0.0;
  }
}

// abs values of the pass-1 list entries; per-row t1-th largest |value| (lists hold exactly t1
// entries per row) -> atomic min
__global__ void list_stats(const float* __restrict__ val, int64_t n, int t1,
                           float* __restrict__ rowmin, unsigned int* __restrict__ max_bits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float mn = INFINITY, mx = 0.f;
    for (int e = 0; e < t1; ++e) {
      const float a = fabsf(val[i * t1 + e]);
      mn = fminf(mn, a);
      mx = fmaxf(mx, a);
    }
    rowmin[i] = mn;
    atomicMax(max_bits, __float_as_uint(mx));  // non-negative floats order as uints
  }
}

// rows whose t1-th listed score is >= x (saturated)
__global__ void count_ge(const float* __restrict__ rowmin, int64_t n, float x,
                         unsigned int* __restrict__ cnt) {
  unsigned int c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += rowmin[i] >= x ? 1u : 0u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// listed entries -> (pair key min*n+max, signed ψ') in slot i*t1 + e; zero entries -> ~0
__global__ void list_pairs(const int32_t* __restrict__ col, const float* __restrict__ val,
                           int64_t n, int t1, uint64_t* __restrict__ pkey,
                           float* __restrict__ score) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * t1;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)(q / t1), j = (uint64_t)col[q];
    const float v = val[q];
    pkey[q] = fabsf(v) > 0.f ? (i < j ? i * (uint64_t)n + j : j * (uint64_t)n + i) : ~0ull;
    score[q] = v;
  }
}

// pass-3 COO (row, col, value') -> upper-triangle candidate arrays (pair key i*n+j, score)
__global__ void upper_pairs(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const float* __restrict__ val, int64_t n,
                            unsigned long long* __restrict__ cnt, uint64_t* __restrict__ pkey,
                            float* __restrict__ score) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int64_t j = col[e];
      if (j <= i) continue;
      const unsigned long long at = atomicAdd(cnt, 1ull);
      pkey[at] = (uint64_t)i * (uint64_t)n + (uint64_t)j;
      score[at] = val[e];  // signed ψ'; ranked by |.|
    }
  }
}

__global__ void abs_copy(const float* __restrict__ x, int64_t cnt, float* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fabsf(x[i]);
}
__global__ void gather_rows(const float* __restrict__ V, const int32_t* __restrict__ ids,
                            int64_t rows, int k, float* __restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < rows * k;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = V[(int64_t)ids[q / k] * k + q % k];
}
__global__ void mark_rows(const int32_t* __restrict__ ids, int64_t rows, uint8_t* __restrict__ in) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < rows;
       a += (int64_t)gridDim.x * blockDim.x)
    in[ids[a]] = 1;
}
// listed pairs with an endpoint outside S -> the overall histogram (same buckets as mode 3)
__global__ void list_hist(const uint64_t* __restrict__ pk, const float* __restrict__ sc,
                          int64_t cnt, int64_t n, const uint8_t* __restrict__ inS, float x0,
                          int hs, unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0u;
  __syncthreads();
  const uint32_t bx0 = __float_as_uint(x0);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = pk[q];
    const int64_t i = (int64_t)(key / (uint64_t)n), j = (int64_t)(key % (uint64_t)n);
    const float a = fabsf(sc[q]);
    if (a > x0 && !(inS[i] && inS[j]))
      atomicAdd(&h[min(255u, (__float_as_uint(a) - bx0) >> hs)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (h[b]) atomicAdd(hist + b, (unsigned long long)h[b]);
}

// block threshold output (local rows a < b of S) -> global pair keys appended at *cnt
__global__ void block_pairs(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const float* __restrict__ val, int64_t rows,
                            const int32_t* __restrict__ ids, int64_t n,
                            unsigned long long* __restrict__ cnt, uint64_t* __restrict__ pkey,
                            float* __restrict__ score) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < rows;
       a += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t gi = (uint64_t)ids[a];
    for (int64_t e = rp[a]; e < rp[a + 1]; ++e) {
      const int64_t b = col[e];
      if (b <= a) continue;
      const uint64_t gj = (uint64_t)ids[b];
      const unsigned long long at = atomicAdd(cnt, 1ull);
      pkey[at] = gi < gj ? gi * (uint64_t)n + gj : gj * (uint64_t)n + gi;
      score[at] = val[e];
    }
  }
}

// min-edges: each row's m best list entries (score desc, column asc) -> pair keys (i<j order)
__global__ void min_edge_pairs(const int32_t* __restrict__ col, const float* __restrict__ val,
                               int64_t n, int t1, int m, uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < m; ++a) {  // a-th best: rank among the row's t1 entries
      int best = -1;
      for (int e = 0; e < t1; ++e) {
        int rank = 0;
        const float ae = fabsf(val[i * t1 + e]);
        const int ce = col[i * t1 + e];
        for (int f = 0; f < t1; ++f) {
          const float af = fabsf(val[i * t1 + f]);
          if (af > ae || (af == ae && col[i * t1 + f] < ce)) ++rank;
        }
        if (rank == a) best = e;
      }
      const int64_t j = best >= 0 ? col[i * t1 + best] : i;
      const int64_t lo = j < i ? j : i, hi = j < i ? i : j;
      // an exactly-zero ψ'_ij is no edge (Q17)
      const bool ok = best >= 0 && fabsf(val[i * t1 + best]) > 0.f;
      out[i * m + a] = ok ? (uint64_t)lo * (uint64_t)n + (uint64_t)hi : ~0ull;
    }
  }
}

// final edges (sorted unique pair keys) -> both directions (row key = r*n + c) with ψ values
__global__ void expand_edges(const uint64_t* __restrict__ pk, int64_t ne, int64_t n,
                             const float* __restrict__ sval, const double* __restrict__ sq,
                             uint64_t* __restrict__ dkey, float* __restrict__ dval) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = pk[e] / (uint64_t)n, j = pk[e] % (uint64_t)n;
    const float v = (float)((double)sval[e] * sq[i] * sq[j]);
    dkey[2 * e] = i * (uint64_t)n + j;
    dkey[2 * e + 1] = j * (uint64_t)n + i;
    dval[2 * e] = v;
    dval[2 * e + 1] = v;
  }
}

__global__ void dir_to_csr(const uint64_t* __restrict__ key, const float* __restrict__ v,
                           int64_t count, int64_t n, int64_t* row_ptr, int32_t* col, float* val) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= count;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < count) {
      col[e] = (int32_t)(key[e] % (uint64_t)n);
      val[e] = v[e];
    }
    const int64_t r = (e < count) ? (int64_t)(key[e] / (uint64_t)n) : n;
    const int64_t rp = (e == 0) ? -1 : (int64_t)(key[e - 1] / (uint64_t)n);
    for (int64_t rr = rp + 1; rr <= r && rr <= n; ++rr) row_ptr[rr] = e;
  }
}

}  // namespace sp
}  // namespace ggm

using namespace ggm;
using namespace ggm::sp;

namespace {

// Overall rules, path 3 (one symmetric pass for the whole candidate set): per-row bounds
// min(top-m seed bound, τ), so the pool holds every directed entry above τ and each row's
// top-m candidates.  After the exact re-evaluation: the pairs (i < j) with |ψ| > τ ->
// pkey/score (all counted in *d_count, the first cap written) and each row's exact top m ->
// row_ptr/col/val (stride m).  GGM_ERR_CAPACITY: the pool overflowed (the caller falls back).
static ggm_status sym_tau_topm(int64_t n, int k, const float* V, const double* lambda, int m,
                               float tau, int64_t extra, void* ws, size_t ws_bytes,
                               uint64_t* pkey, float* score, int64_t cap,
                               unsigned long long* d_count, int64_t* npairs, int64_t* row_ptr,
                               int32_t* col, float* val, cudaStream_t s) {
  ggm_sparsify_opts so{};
  so.mode = 0;
  so.topk = m;
  so.symmetric = 1;
  Plan pl;
  ggm_status st;
  {
    CandExtraScope ce(extra);
    st = make_plan(n, k, 0, n, &so, n * (int64_t)m, &pl);
  }
  if (st != GGM_OK) return st;
  if (!pl.sym) return fail(GGM_ERR_UNSUPPORTED, "overall path 3 needs the symmetric scheme");
  reset_launches();
  Work w;
  if (ws_bytes < carve(pl, ws, &w)) return fail(GGM_ERR_INVALID_ARGUMENT, "overall path 3 workspace");
  const int sms = num_sms();
  GGM_CUDA_TRY(cudaMemsetAsync(w.sc, 0, sizeof(DevScalars), s));
  absmax_check<<<(int)std::max<int64_t>(1, std::min<int64_t>((n * k + 255) / 256, sms * 8)), 256, 0, s>>>(
      V, lambda, n, k, w.sc);
  scale_finalize<<<1, 1, 0, s>>>(w.sc);
  count_launches(2);
  FusedParams fp = base_params(pl, w, n, 0);
  fp.tau = 0.f;
  st = sym_prepare(pl, w, V, lambda, n, k, fp, s, -1, -1, nullptr, tau);
  if (st != GGM_OK) return st;
  st = sym_main(pl, w, fp, 0, (int)pl.NBu, s);
  if (st != GGM_OK) return st;
  DevScalars hs;
  GGM_CUDA_TRY(cudaMemcpyAsync(&hs, w.sc, sizeof(hs), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hs.flags & 1) return fail(GGM_ERR_DOMAIN, "V contains non-finite values");
  if (hs.flags & 2) return fail(GGM_ERR_DOMAIN, "lambda must be finite and > 0 (P:65)");
  if (hs.cand_overflow) return fail(GGM_ERR_CAPACITY, "overall path 3: candidate pool overflow");
  const int64_t ncand = (int64_t)std::min<unsigned long long>(hs.cand_alloc, pl.cand_total);
  GGM_CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s));
  if (ncand > 0) {
    size_t tb = pl.sort_temp_bytes;
    int ebits = 1;
    while ((int64_t(1) << ebits) <= n) ++ebits;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, tb, w.ckey, w.skey, w.cval, w.sval,
                                                 ncand, 0, ebits, s));
    if (pl.screen) recompute_pool(w, ncand, n, k, 0, 0, sms, s);  // every candidate exact
    sym_upper_pairs<<<(int)std::min<int64_t>((ncand + 255) / 256, sms * 16), 256, 0, s>>>(
        w.skey, w.sval, ncand, n, w.perm, tau, cap, d_count, pkey, score);
    count_launches(1);
  }
  if (m <= 5)
    launch_merge_sym_t<5>(w, pl, ncand, row_ptr, col, val, s);
  else if (m <= 10)
    launch_merge_sym_t<10>(w, pl, ncand, row_ptr, col, val, s);
  else if (m <= 16)
    launch_merge_sym_t<16>(w, pl, ncand, row_ptr, col, val, s);
  else
    launch_merge_sym_t<32>(w, pl, ncand, row_ptr, col, val, s);
  count_launches(1);
  unsigned long long hc = 0;
  GGM_CUDA_TRY(cudaMemcpyAsync(&hc, d_count, sizeof(hc), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  GGM_CUDA_TRY(cudaGetLastError());
  *npairs = (int64_t)hc;
  return GGM_OK;
}

// path 3 sample: rows (s n)/R + n/(2R), s < R (a stratified sample of the axis)
__global__ void sample_rows(int32_t* __restrict__ ids, int64_t R, int64_t n) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < R;
       q += (int64_t)gridDim.x * blockDim.x)
    ids[q] = (int32_t)(q * n / R + n / (2 * R) < n ? q * n / R + n / (2 * R) : n - 1);
}
constexpr int64_t kOverallSampleRows = 16384;  // path 3: rows of the pair sample
constexpr int64_t kOverallPath3MinN = 65536;   // path 3 by default from this axis length
constexpr double kOverallTauMargin = 1.25;      // τ: sampled rank of 1.25 N pairs (2.5 N directed)
static int64_t overall_path3_extra(int64_t N) { return 4 * N; }

constexpr int kOverallSeedFrac = 8;  // seed sample of the top-t1 lists pass (see make_plan)
thread_local int g_overall_path = -1;  // 0: lists only, 1: histogram + threshold, 2: block
thread_local int64_t g_overall_sat = 0;  // saturated rows at L3
thread_local float g_overall_ms[5] = {0.f, 0.f, 0.f, 0.f, 0.f};

// phase marks of the overall driver (CUDA events on its stream, when ggm_set_timing(1))
struct PhaseTimer {
  cudaEvent_t ev[6] = {};
  bool on;
  cudaStream_t s;
  int last = -1;
  PhaseTimer(bool enabled, cudaStream_t st) : on(enabled), s(st) {
    if (on)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark(int i) {
    if (on) {
      cudaEventRecord(ev[i], s);
      last = i;
    }
  }
  ~PhaseTimer() {
    if (!on) return;
    if (last == 5) {
      cudaEventSynchronize(ev[5]);
      for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&g_overall_ms[i], ev[i], ev[i + 1]);
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
};

struct OverallPlan {
  int64_t n, N, cand_cap, E_max;
  int k, t1, m, downweight;
  size_t ws_sub;   // max sub-call workspace (mass / top-t1 / threshold)
  size_t cub_tmp;  // max CUB temp
};

ggm_status overall_plan(int64_t n, int k, const ggm_overall_opts* o, int64_t cand_capacity,
                        OverallPlan* op) {
  if (!o) return fail(GGM_ERR_INVALID_ARGUMENT, "opts is NULL");
  if (n < 3 || k < 1 || k > n) return fail(GGM_ERR_INVALID_ARGUMENT, "n >= 3, 1 <= k <= n");
  const int64_t pairs = n * (n - 1) / 2;
  if (o->n_edges < 1 || o->n_edges > pairs)
    return fail(GGM_ERR_INVALID_ARGUMENT, "n_edges=%lld not in [1, n(n-1)/2]", (long long)o->n_edges);
  if (o->min_edges < 0 || o->min_edges > GGM_MAX_TOPK)
    return fail(GGM_ERR_INVALID_ARGUMENT, "min_edges not in [0, %d]", GGM_MAX_TOPK);
  if (cand_capacity < 1) return fail(GGM_ERR_INVALID_ARGUMENT, "cand_capacity < 1");
  op->n = n;
  op->k = k;
  op->N = o->n_edges;
  op->m = (int)std::min<int64_t>(o->min_edges, n - 1);
  op->downweight = o->downweight ? 1 : 0;
  // n·t1 >= 4N listed entries when possible: the 2N-th largest listed value is then a tight
  // lower bound (exact unless a row holds more than t1 of the top 2N directed entries)
  const int64_t need_t = 2 * ((2 * op->N + n - 1) / n);
  op->t1 = (int)std::min<int64_t>(n - 1, std::min<int64_t>(GGM_MAX_TOPK, std::max<int64_t>(
                                                                std::max<int64_t>(op->m, need_t), 1)));
  op->cand_cap = cand_capacity;
  op->E_max = op->N + n * op->m;
  size_t b = 0, mx = 0;
  ggm_sparsify_opts so{};
  so.mode = 2;
  so.topk = 1;
  {  // internal passes (row mass, histogram): plain plan, no output capacity
    Plan pl;
    Work wk;
    ggm_status st2 = make_plan(n, k, 0, n, &so, 0, &pl);
    if (st2 != GGM_OK) return st2;
    mx = std::max(mx, carve(pl, nullptr, &wk));
  }
  ggm_status st = GGM_OK;
  so.mode = 0;
  so.topk = op->t1;
  {
    SeedFracScope sf(kOverallSeedFrac);
    st = ggm_sparse_precision_workspace(n, k, 0, n, &so, n * op->t1, &b);
  }
  if (st != GGM_OK) return st;
  mx = std::max(mx, b);
  so.mode = 1;
  so.topk = 1;
  so.tau = 0.f;
  st = ggm_sparse_precision_workspace(n, k, 0, n, &so, cand_capacity, &b);
  if (st != GGM_OK) return st;
  mx = std::max(mx, b);
  {  // path 3: the sample's top-T lists and the global-threshold pass (if it applies)
    const int64_t R = std::min<int64_t>(n, kOverallSampleRows);
    if (R >= 3) {
      ggm_sparsify_opts s3{};
      s3.mode = 0;
      s3.topk = (int)std::min<int64_t>(GGM_MAX_TOPK, R - 1);
      if (ggm_sparse_precision_workspace(R, k, 0, R, &s3, R * s3.topk, &b) == GGM_OK)
        mx = std::max(mx, b);
    }
    ggm_sparsify_opts s4{};
    s4.mode = 0;
    s4.topk = std::max(op->m, 1);
    s4.symmetric = 1;
    Plan pl;
    Work wk;
    CandExtraScope ce(overall_path3_extra(op->N));
    if (make_plan(n, k, 0, n, &s4, n * (int64_t)s4.topk, &pl) == GGM_OK && pl.sym)
      mx = std::max(mx, carve(pl, nullptr, &wk));
  }
  op->ws_sub = mx;
  size_t c = 0, t = 0;
  const int64_t L = op->n * op->t1 + cand_capacity + 2 * op->E_max;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, t, (const float*)nullptr, (float*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, L);
  c = std::max(c, t);
  cub::DeviceRadixSort::SortKeysDescending(nullptr, t, (const float*)nullptr, (float*)nullptr, L);
  c = std::max(c, t);
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int64_t*)nullptr, (int64_t*)nullptr, L);
  c = std::max(c, t);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, t, (const float*)nullptr, (float*)nullptr,
                                            (const int64_t*)nullptr, (int64_t*)nullptr, L);
  c = std::max(c, t);
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const float*)nullptr, (float*)nullptr, L);
  c = std::max(c, t);
  cub::DeviceSelect::UniqueByKey(nullptr, t, (const uint64_t*)nullptr, (const float*)nullptr,
                                 (uint64_t*)nullptr, (float*)nullptr, (int64_t*)nullptr, L);
  c = std::max(c, t);
  op->cub_tmp = c;
  return GGM_OK;
}

struct OverallWork {
  float* Vs;
  double *w, *sq;
  void* sub;
  int64_t *rp1, *rp3;
  int32_t *col1, *col3;
  float *val1, *val3, *rowmin, *Vsub;
  int32_t *rid, *rid_s;
  uint8_t* inS;
  unsigned int* min_bits;  // [0] saturated-row count, [1] max listed score bits
  unsigned long long* hist;
  unsigned long long* cnt;
  uint64_t *pk, *pk_s, *uk, *uk_s;
  float *sc, *ak, *ak_s, *uv, *uv_s;
  int64_t *idx, *idx1, *idx2, *nsel;
  void* cub;
};

size_t overall_carve(const OverallPlan& op, void* ws, OverallWork* w) {
  Carve c(ws);
  const int64_t n = op.n, E = op.E_max, L = n * op.t1, C = op.cand_cap + L;
  w->Vs = c.take<float>((size_t)n * op.k);
  w->w = c.take<double>(n);
  w->sq = c.take<double>(n);
  w->sub = c.take<char>(op.ws_sub);
  w->rp1 = c.take<int64_t>(n + 1);
  w->col1 = c.take<int32_t>(L);
  w->val1 = c.take<float>(L);
  w->rowmin = c.take<float>(n);
  w->Vsub = c.take<float>((size_t)n * op.k);
  w->rid = c.take<int32_t>(n);
  w->rid_s = c.take<int32_t>(n);
  w->inS = c.take<uint8_t>(n);
  w->min_bits = c.take<unsigned int>(2);
  w->hist = c.take<unsigned long long>(256);
  w->cnt = c.take<unsigned long long>(1);
  w->rp3 = c.take<int64_t>(n + 1);
  w->col3 = c.take<int32_t>(op.cand_cap);
  w->val3 = c.take<float>(op.cand_cap);
  w->pk = c.take<uint64_t>(C);
  w->pk_s = c.take<uint64_t>(C);
  w->sc = c.take<float>(C);
  w->ak = c.take<float>(C);
  w->ak_s = c.take<float>(C);
  w->idx = c.take<int64_t>(C);
  w->idx1 = c.take<int64_t>(C);
  w->idx2 = c.take<int64_t>(C);
  w->uk = c.take<uint64_t>(2 * E);    // union keys, then directed keys
  w->uk_s = c.take<uint64_t>(2 * E);
  w->uv = c.take<float>(2 * E);
  w->uv_s = c.take<float>(2 * E);
  w->nsel = c.take<int64_t>(1);
  w->cub = c.take<char>(op.cub_tmp);
  return c.used();
}

__global__ void iota_i64(int64_t* p, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = i;
}
__global__ void gather_abs(const float* __restrict__ sc, const int64_t* __restrict__ idx,
                           int64_t count, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fabsf(sc[idx[i]]);
}
// top N (by idx2 order) -> union arrays [0, N): pair key, signed value'
__global__ void take_top(const int64_t* __restrict__ idx2, int64_t N,
                         const uint64_t* __restrict__ pk, const float* __restrict__ sc,
                         uint64_t* __restrict__ uk, float* __restrict__ uv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    uk[i] = pk[idx2[i]];
    uv[i] = sc[idx2[i]];
  }
}
// min-edge values from the pass-1 lists (signed ψ'), keyed like min_edge_pairs
__global__ void min_edge_vals(const int32_t* __restrict__ col, const float* __restrict__ val,
                              const uint64_t* __restrict__ keys, int64_t n, int t1, int m,
                              float* __restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * m;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / m;
    const uint64_t key = keys[q];
    float v = 0.f;
    if (key != ~0ull) {
      const uint64_t lo = key / (uint64_t)n, hi = key % (uint64_t)n;
      const int64_t j = (int64_t)(lo == (uint64_t)i ? hi : lo);
      for (int e = 0; e < t1; ++e)
        if (col[i * t1 + e] == j) v = val[i * t1 + e];
    }
    out[q] = v;
  }
}

}  // namespace

extern "C" ggm_status ggm_sparse_precision_overall_workspace(int64_t n, int k,
                                                            const ggm_overall_opts* opts,
                                                            int64_t cand_capacity, size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  OverallPlan op;
  ggm_status st = overall_plan(n, k, opts, cand_capacity, &op);
  if (st != GGM_OK) return st;
  OverallWork w;
  *bytes = overall_carve(op, nullptr, &w);
  return GGM_OK;
}

extern "C" ggm_status ggm_sparse_precision_overall(
    int64_t n, int k, const float* V, const double* lambda, const ggm_overall_opts* opts,
    int64_t cand_capacity, int64_t* row_ptr, int32_t* col, float* val, int64_t capacity,
    int64_t* nnz_out, void* workspace, size_t workspace_bytes, void* stream) {
  seed_stamp_forget(workspace);
  if (!V || !lambda || !row_ptr || !nnz_out || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer argument");
  OverallPlan op;
  ggm_status st = overall_plan(n, k, opts, cand_capacity, &op);
  if (st != GGM_OK) return st;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  OverallWork w;
  const size_t need = overall_carve(op, workspace, &w);
  if (workspace_bytes < need)
    return fail(GGM_ERR_INVALID_ARGUMENT, "workspace %zu < required %zu", workspace_bytes, need);
  if (!ggm_device_supported())
    return fail(GGM_ERR_CUDA, "current device is not compute capability 10.0 (sm_100a)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int sms = num_sms();
  const int g = sms * 8;
  auto blocks = [&](int64_t cnt) { return (int)std::max<int64_t>(1, std::min<int64_t>((cnt + 255) / 256, g)); };
  int launches = 0;
  PhaseTimer ph(timing_enabled(), s);
  ph.mark(0);
  // (1) row masses of Ψ (plain tiles, mode 2), then V' = V ⊙ w^-1/2
  if (op.downweight) {
    Plan pl;
    ggm_sparsify_opts so{};
    so.mode = 2;
    so.topk = 1;
    st = make_plan(n, k, 0, n, &so, 0, &pl);
    if (st != GGM_OK) return st;
    Work sw;
    carve(pl, w.sub, &sw);
    GGM_CUDA_TRY(cudaMemsetAsync(sw.sc, 0, sizeof(DevScalars), s));
    GGM_CUDA_TRY(cudaMemsetAsync(w.w, 0, sizeof(double) * n, s));
    absmax_check<<<blocks(n * (int64_t)k), 256, 0, s>>>(V, lambda, n, k, sw.sc);
    scale_finalize<<<1, 1, 0, s>>>(sw.sc);
    launch_split(s, sms, V, lambda, n, k, pl.KA, pl.KS, pl.TS, 0, (int64_t)pl.nBblocks * kRowsPerBlock, sw.sc, sw.Bop);
    FusedParams fp = base_params(pl, sw, n, 0);
    fp.mass_out = w.w;
    if (pl.resident && !std::getenv("GGM_OVERALL_PLAIN_MASS")) {
      // each unordered block pair once: row sums + column sums (half the plain MMA work)
      fp.kind = kSymList;
      fp.RB = (int)pl.NBu;
      fp.wsplit = kWindowSplit;  // (only CTA pairs split windows)
    }
    st = launch_fused(fp, pl.t, a_blocks(pl, 0), pl.nBblocks, s);
    if (st != GGM_OK) return st;
    scale_pow2<<<blocks(n), 256, 0, s>>>(w.w, n, sw.sc);  // accumulator -> ψ units (exact)
    launches += 5;
  }
  scale_rows<<<blocks(n * (int64_t)k), 256, 0, s>>>(V, op.downweight ? w.w : nullptr, n, k, w.Vs, w.sq);
  GGM_CUDA_TRY(cudaGetLastError());
  ++launches;
  // (2) per-row top-t1 of Ψ'
  ph.mark(1);
  // Path 3 (default from kOverallPath3MinN rows; GGM_OVERALL_PATH=3 forces it): a global
  // threshold τ from a uniform pair sample (the top-T lists of R stratified sample rows
  // among themselves: (R(R-1))/(n(n-1)) of all pairs; directed counts / 2 never exceed the
  // sample's pair counts, so τ errs low), set at the sampled rank of 2.5 N directed entries
  // (~1.25 N pairs above it); then ONE symmetric pass with bounds min(top-m bound, τ) gives
  // every pair above τ and each row's top m.  Exact when >= N pairs exceed τ (checked);
  // otherwise, or when the sample / pool / capacities do not fit, the lists path below runs.
  const char* force = std::getenv("GGM_OVERALL_PATH");  // test hook: "1" hist, "2" block, "3"
  int lst = op.t1;  // stride of the per-row lists used by the min-edges rule
  int64_t nc = 0;
  bool done3 = false;
  if (force ? force[0] == '3' : n >= kOverallPath3MinN) {
    const int64_t C = op.cand_cap + n * op.t1;  // pair-candidate arrays
    const int64_t R = std::min<int64_t>(n, kOverallSampleRows);
    const int T = (int)std::min<int64_t>(GGM_MAX_TOPK, R - 1);
    float tau = 0.f;
    if (R >= 3 && R * T <= op.cand_cap) {
      const float* F = w.Vs;
      if (R < n) {
        sample_rows<<<blocks(R), 256, 0, s>>>(w.rid, R, n);
        gather_rows<<<blocks(R * k), 256, 0, s>>>(w.Vs, w.rid, R, k, w.Vsub);
        F = w.Vsub;
        launches += 2;
      }
      ggm_sparsify_opts so{};
      so.mode = 0;
      so.topk = T;
      int64_t nnz = 0;
      if (ggm_sparse_precision(R, k, F, lambda, 0, R, &so, w.rp3, w.col3, w.val3, op.cand_cap,
                               &nnz, w.sub, op.ws_sub, stream) == GGM_OK) {
        launches += ggm_last_launches();
        const double pr = (double)R * (double)(R - 1) / ((double)n * (double)(n - 1));
        // directed entries of the sample: 2 x its pairs above the level
        const int64_t K = (int64_t)std::ceil(2.0 * kOverallTauMargin * (double)op.N * pr);
        if (K >= 64 && K <= R * T) {
          abs_copy<<<blocks(R * T), 256, 0, s>>>(w.val3, R * T, w.ak);
          size_t tb = op.cub_tmp;
          GGM_CUDA_TRY(cub::DeviceRadixSort::SortKeysDescending(w.cub, tb, w.ak, w.ak_s, R * T, 0, 32, s));
          GGM_CUDA_TRY(cudaMemcpyAsync(&tau, w.ak_s + K - 1, sizeof(float), cudaMemcpyDeviceToHost, s));
          GGM_CUDA_TRY(cudaStreamSynchronize(s));
          launches += 2;
        }
      }
    }
    if (std::getenv("GGM_DEBUG_OVERALL"))
      fprintf(stderr, "overall path 3: sample R=%lld T=%d cand_cap %lld -> tau %g\n", (long long)R, T,
              (long long)op.cand_cap, (double)tau);
    if (tau > 0.f) {
      int64_t np = 0;
      const ggm_status st3 = sym_tau_topm(n, k, w.Vs, lambda, std::max(op.m, 1), tau,
                                          overall_path3_extra(op.N), w.sub, op.ws_sub, w.pk,
                                          w.sc, C, w.cnt, &np, w.rp1, w.col1, w.val1, s);
      launches += ggm_last_launches();
      if (std::getenv("GGM_DEBUG_OVERALL"))
        fprintf(stderr, "overall path 3: R=%lld T=%d tau=%g status=%d pairs=%lld (N=%lld, cap %lld)\n",
                (long long)R, T, (double)tau, (int)st3, (long long)np, (long long)op.N, (long long)C);
      if (st3 == GGM_ERR_DOMAIN) return st3;
      if (st3 == GGM_OK && np >= op.N && np <= C) {
        done3 = true;
        nc = np;
        lst = std::max(op.m, 1);
        g_overall_path = 3;
        g_overall_sat = 0;
        ph.mark(2);
        ph.mark(3);
      }
    }
  }
  if (!done3) {
  {
    ggm_sparsify_opts so{};
    so.mode = 0;
    so.topk = op.t1;
    int64_t nnz = 0;
    SeedFracScope sf(kOverallSeedFrac);
    st = ggm_sparse_precision(n, k, w.Vs, lambda, 0, n, &so, w.rp1, w.col1, w.val1, n * op.t1,
                              &nnz, w.sub, op.ws_sub, stream);
    if (st != GGM_OK) return st;
    if (std::getenv("GGM_DEBUG_OVERALL"))
      fprintf(stderr, "overall lists t1=%d: scheme %.0f entries %.3g cand %.3g recomputed %.0f\n",
              op.t1, g_stats[0], g_stats[1], g_stats[2], g_stats[3]);
    launches += ggm_last_launches();
  }
  // (3) candidates.  The listed pairs (either direction, de-duplicated) give L3 = the N-th
  // largest listed pair score, a lower bound of the N-th largest pair score (N real pairs
  // reach it).  Row i is saturated when its t1-th listed score is >= L3 (it may hold
  // unlisted entries >= L3).  A pair (i, j) with score >= L3 is missing from the lists only
  // if both i and j are saturated, so: no saturated row -> the lists hold the top N pairs
  // (path 0); a few -> add the saturated rows' block S x S by a threshold pass on their
  // gathered factor rows (path 2); many -> histogram + full threshold pass (path 1).
  auto dedupe = [&](int64_t cnt, int64_t* out) -> ggm_status {
    size_t tb = op.cub_tmp;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.pk, w.pk_s, w.sc, w.ak_s, cnt, 0, 64, s));
    tb = op.cub_tmp;
    GGM_CUDA_TRY(cub::DeviceSelect::UniqueByKey(w.cub, tb, w.pk_s, w.ak_s, w.pk, w.sc, w.nsel, cnt, s));
    int64_t u = 0;
    GGM_CUDA_TRY(cudaMemcpyAsync(&u, w.nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    if (u > 0) {  // drop the ~0 sentinel (zero entries)
      uint64_t lastk = 0;
      GGM_CUDA_TRY(cudaMemcpyAsync(&lastk, w.pk + u - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      GGM_CUDA_TRY(cudaStreamSynchronize(s));
      if (lastk == ~0ull) --u;
    }
    *out = u;
    return GGM_OK;
  };
  ph.mark(2);
  GGM_CUDA_TRY(cudaMemsetAsync(w.min_bits, 0, 2 * sizeof(unsigned int), s));
  list_stats<<<blocks(n), 256, 0, s>>>(w.val1, n, op.t1, w.rowmin, w.min_bits + 1);
  // deterministic slots i*t1 + e: duplicates keep the entry of the smaller row (stable sort)
  list_pairs<<<blocks(n * op.t1), 256, 0, s>>>(w.col1, w.val1, n, op.t1, w.pk, w.sc);
  int64_t nu1 = 0;
  st = dedupe(n * op.t1, &nu1);
  if (st != GGM_OK) return st;
  float L3 = 0.f, gmax = 0.f;
  {
    unsigned int mb = 0;
    GGM_CUDA_TRY(cudaMemcpyAsync(&mb, w.min_bits + 1, sizeof(mb), cudaMemcpyDeviceToHost, s));
    if (nu1 >= op.N) {
      abs_copy<<<blocks(nu1), 256, 0, s>>>(w.sc, nu1, w.ak);
      size_t tb = op.cub_tmp;
      GGM_CUDA_TRY(cub::DeviceRadixSort::SortKeysDescending(w.cub, tb, w.ak, w.ak_s, nu1, 0, 32, s));
      GGM_CUDA_TRY(cudaMemcpyAsync(&L3, w.ak_s + op.N - 1, sizeof(float), cudaMemcpyDeviceToHost, s));
      launches += 1;
    }
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    std::memcpy(&gmax, &mb, 4);
  }
  count_ge<<<blocks(n), 256, 0, s>>>(w.rowmin, n, L3, w.min_bits);
  launches += 3;
  unsigned int nsat = 0;
  GGM_CUDA_TRY(cudaMemcpyAsync(&nsat, w.min_bits, sizeof(nsat), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  nc = nu1;
  g_overall_path = L3 <= 0.f ? 1 : (nsat == 0 ? 0 : (2 * (int64_t)nsat <= n ? 2 : 1));
  if (force && L3 > 0.f && (force[0] == '1' || force[0] == '2')) g_overall_path = force[0] - '0';
  g_overall_sat = nsat;
  ph.mark(3);
  if (g_overall_path != 0) {
    // Path 2: S = the s_eff rows with the largest t1-th listed score (all saturated rows,
    // at least k rows so the block is a valid factor), gathered into V_S; path 1: S = all
    // rows.  (a) histogram, in 256 log buckets above x0 ~ L3, of the pair scores: the
    // block's upper triangle (plain tiles, mode 3) plus, on path 2, the listed pairs with
    // an endpoint outside S (complete above L3: such a row is not saturated) -> the exact
    // count of pairs above each bucket edge >= L3; (b) the bucket edge where that count
    // reaches N (<= the N-th largest score) is the threshold of one pass over the block
    // (threshold mode; the histogram used the same kernel arithmetic, so the candidate
    // count is known before the pass).
    const float* F = w.Vs;
    int64_t rows = n;
    if (g_overall_path == 2) {
      rows = std::min<int64_t>(n, std::max<int64_t>({(int64_t)nsat, (int64_t)k, 2}));
      iota_i32<<<blocks(n), 256, 0, s>>>(w.rid, n);
      {
        size_t tb = op.cub_tmp;
        GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(w.cub, tb, w.rowmin, w.ak_s, w.rid, w.rid_s, n, 0, 32, s));
      }
      gather_rows<<<blocks(rows * k), 256, 0, s>>>(w.Vs, w.rid_s, rows, k, w.Vsub);
      GGM_CUDA_TRY(cudaMemsetAsync(w.inS, 0, n, s));
      mark_rows<<<blocks(rows), 256, 0, s>>>(w.rid_s, rows, w.inS);
      F = w.Vsub;
      launches += 3;
    }
    // x0 > 0 keeps bucket offsets invariant under the kernel's power-of-two operand scale
    // (bits(x·2^s) - bits(x0·2^s) = bits(x) - bits(x0) for normal floats); with no bound
    // from the lists, x0 = 2^-60 max|ψ'| (smaller entries are below the fp32 accuracy of
    // the products and count as zero, Q17)
    const float x0 = L3 > 0.f ? L3 * (1.f - 1e-5f) : std::ldexp(gmax, -60);
    uint32_t bx0, bmax;
    std::memcpy(&bx0, &x0, 4);
    std::memcpy(&bmax, &gmax, 4);
    const uint64_t range = (uint64_t)(bmax > bx0 ? bmax - bx0 : 0) + 64;  // ulp slack
    int hs = 0;
    while ((range >> hs) > 255) ++hs;
    {
      Plan pl;
      ggm_sparsify_opts so{};
      so.mode = 3;
      so.topk = 1;
      st = make_plan(rows, k, 0, rows, &so, 0, &pl);
      if (st != GGM_OK) return st;
      Work sw;
      carve(pl, w.sub, &sw);
      GGM_CUDA_TRY(cudaMemsetAsync(sw.sc, 0, sizeof(DevScalars), s));
      GGM_CUDA_TRY(cudaMemsetAsync(w.hist, 0, 256 * sizeof(unsigned long long), s));
      absmax_check<<<blocks(rows * (int64_t)k), 256, 0, s>>>(F, lambda, rows, k, sw.sc);
      scale_finalize<<<1, 1, 0, s>>>(sw.sc);
      launch_split(s, sms, F, lambda, rows, k, pl.KA, pl.KS, pl.TS, 0, (int64_t)pl.nBblocks * kRowsPerBlock, sw.sc, sw.Bop);
      FusedParams fp = base_params(pl, sw, rows, 0);
      fp.tau = x0;
      fp.hist_out = w.hist;
      fp.hshift = hs;
      st = launch_fused(fp, pl.t, a_blocks(pl, 0), pl.nBblocks, s);
      if (st != GGM_OK) return st;
      launches += 3;
      if (g_overall_path == 2) {
        list_hist<<<std::max(1, std::min(sms * 4, (int)((nu1 + 1023) / 1024))), 256, 0, s>>>(
            w.pk, w.sc, nu1, n, w.inS, x0, hs, w.hist);
        launches += 1;
      }
    }
    unsigned long long hh[256];
    GGM_CUDA_TRY(cudaMemcpyAsync(hh, w.hist, sizeof(hh), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    unsigned long long cum = 0;
    int bstar = 0;
    for (int bb = 255; bb >= 0; --bb) {
      cum += hh[bb];
      if (cum >= (unsigned long long)op.N) { bstar = bb; break; }
    }
    // threshold just below the bucket's lower edge: |ψ'| > tau <=> bits >= edge
    const uint32_t edge = bx0 + ((uint32_t)bstar << hs);
    const uint32_t tb3 = edge > 0 ? edge - 1 : 0;
    float tau3;
    std::memcpy(&tau3, &tb3, 4);
    // directed candidates <= 2 x the pairs counted (+ slack for ulp asymmetry ψ_ij / ψ_ji)
    const int64_t need = 2 * (int64_t)cum + 2 * (int64_t)(cum / 1000) + 4096;
    if (need > op.cand_cap) {
      *nnz_out = -need;
      return fail(GGM_ERR_CAPACITY, "overall: ~%lld candidates > cand_capacity %lld",
                  (long long)need, (long long)op.cand_cap);
    }
    int64_t ncoo = 0;
    ggm_sparsify_opts so3{};
    so3.mode = 1;
    so3.topk = 1;
    so3.tau = edge > 0 ? tau3 : 0.f;
    st = ggm_sparse_precision(rows, k, F, lambda, 0, rows, &so3, w.rp3, w.col3, w.val3,
                              op.cand_cap, &ncoo, w.sub, op.ws_sub, stream);
    if (st == GGM_ERR_CAPACITY) {
      *nnz_out = -ncoo;
      return fail(GGM_ERR_CAPACITY, "overall: %lld candidates > cand_capacity %lld",
                  (long long)ncoo, (long long)op.cand_cap);
    }
    if (st != GGM_OK) return st;
    launches += ggm_last_launches() + 1;
    if (g_overall_path == 1) {
      GGM_CUDA_TRY(cudaMemsetAsync(w.cnt, 0, sizeof(unsigned long long), s));
      upper_pairs<<<blocks(n), 256, 0, s>>>(w.rp3, w.col3, w.val3, n, w.cnt, w.pk, w.sc);
      unsigned long long hc = 0;
      GGM_CUDA_TRY(cudaMemcpyAsync(&hc, w.cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
      GGM_CUDA_TRY(cudaStreamSynchronize(s));
      nc = (int64_t)hc;
    } else {
      GGM_CUDA_TRY(cudaMemcpyAsync(w.cnt, &nu1, sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
      block_pairs<<<blocks(rows), 256, 0, s>>>(w.rp3, w.col3, w.val3, rows, w.rid_s, n, w.cnt, w.pk, w.sc);
      unsigned long long hc = 0;
      GGM_CUDA_TRY(cudaMemcpyAsync(&hc, w.cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
      GGM_CUDA_TRY(cudaStreamSynchronize(s));
      st = dedupe((int64_t)hc, &nc);
      if (st != GGM_OK) return st;
      launches += 1;
    }
  }
  }  // lists path
  // (4) candidates ranked by (score desc, i, j): stable sorts by pair key, then by |score|
  ph.mark(4);
  const int64_t Ntop = std::min<int64_t>(op.N, nc);
  iota_i64<<<blocks(nc), 256, 0, s>>>(w.idx, nc);
  {
    size_t tb = op.cub_tmp;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.pk, w.pk_s, w.idx, w.idx1, nc, 0, 64, s));
  }
  gather_abs<<<blocks(nc), 256, 0, s>>>(w.sc, w.idx1, nc, w.ak);
  {
    // stable descending sort by |score| keeps (i, j) order among ties
    size_t tb = op.cub_tmp;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(w.cub, tb, w.ak, w.ak_s, w.idx1, w.idx2,
                                                           nc, 0, 32, s));
  }
  take_top<<<blocks(Ntop), 256, 0, s>>>(w.idx2, Ntop, w.pk, w.sc, w.uk, w.uv);
  int64_t nu = Ntop;
  if (op.m > 0) {
    min_edge_pairs<<<blocks(n), 256, 0, s>>>(w.col1, w.val1, n, lst, op.m, w.uk + Ntop);
    min_edge_vals<<<blocks(n * op.m), 256, 0, s>>>(w.col1, w.val1, w.uk + Ntop, n, lst, op.m, w.uv + Ntop);
    nu += n * op.m;
  }
  launches += 5 + (op.m > 0 ? 2 : 0);
  {
    size_t tb = op.cub_tmp;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.uk, w.uk_s, w.uv, w.uv_s, nu, 0, 64, s));
    tb = op.cub_tmp;
    GGM_CUDA_TRY(cub::DeviceSelect::UniqueByKey(w.cub, tb, w.uk_s, w.uv_s, w.uk, w.uv, w.nsel, nu, s));
  }
  int64_t ne = 0;
  GGM_CUDA_TRY(cudaMemcpyAsync(&ne, w.nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  uint64_t last = 0;
  if (ne > 0) {  // drop the ~0 sentinel (min-edge slots of rows with fewer entries)
    GGM_CUDA_TRY(cudaMemcpyAsync(&last, w.uk + ne - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    GGM_CUDA_TRY(cudaStreamSynchronize(s));
    if (last == ~0ull) --ne;
  }
  // (5) both directions, ψ = ψ'·sqrt(w_i w_j), sorted by (row, col) -> CSR
  *nnz_out = 2 * ne;
  if (2 * ne > capacity)
    return fail(GGM_ERR_CAPACITY, "overall: %lld entries > capacity %lld", (long long)(2 * ne),
                (long long)capacity);
  if (ne > 0 && (!col || !val)) return fail(GGM_ERR_INVALID_ARGUMENT, "col/val NULL");
  expand_edges<<<blocks(ne), 256, 0, s>>>(w.uk, ne, n, w.uv, w.sq, w.uk_s, w.uv_s);
  {
    size_t tb = op.cub_tmp;
    GGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.uk_s, w.uk, w.uv_s, w.uv, 2 * ne, 0, 64, s));
  }
  dir_to_csr<<<blocks(2 * ne + 1), 256, 0, s>>>(w.uk, w.uv, 2 * ne, n, row_ptr, col, val);
  GGM_CUDA_TRY(cudaGetLastError());
  ph.mark(5);
  GGM_CUDA_TRY(cudaStreamSynchronize(s));
  reset_launches();
  count_launches(launches + 3);
  return GGM_OK;
}

extern "C" int ggm_overall_last_path(int64_t* saturated, float ms[5]) {
  if (saturated) *saturated = g_overall_sat;
  if (ms)
    for (int i = 0; i < 5; ++i) ms[i] = g_overall_ms[i];
  return g_overall_path;
}
