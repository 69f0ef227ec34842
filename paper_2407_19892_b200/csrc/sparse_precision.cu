// sparse_precision.cu — fused recomposition + per-row sparsification of
//   Ψ = V diag(λ) V^T   (Cor. of Thm 2; Alg. 1 lines 18-20)
// evaluated in 128 x 256 tiles on sm_100a tensor cores (tcgen05.mma, fp32 accumulators in
// TMEM), with the per-row top-t / threshold selection fused into the epilogue so that the
// n x n matrix is never written ("we eigen-recompose and threshold simultaneously").
//
// Kernels (DESIGN.md §"Kernels"):
//   BK1a absmax_check   max_{i,r} |V_ir|·sqrt(λ_r), finiteness / λ>0 flags
//   BK1b scale_finalize power-of-two scale s = 2^e with max|U|·s <= 2^14
//   BK1c split_tile     U·s = hi + lo (two fp16 terms) written in the pre-swizzled
//                       (SWIZZLE_128B, K-major) 128-row block layout the MMA reads
//   BK2  fused_recon_topk  persistent, warp-specialised: 1 producer warp (bulk async
//                       copies), 1 MMA-issuer warp (3 MMAs / K-step: hi·hi, hi·lo, lo·hi),
//                       4 epilogue warps (tcgen05.ld thread = row, register top-t)
//   BK3  merge_partials / coo_to_csr  column-chunk merge (mode 0) and CSR assembly (mode 1)
#include <cub/device/device_radix_sort.cuh>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <vector>

#include "ggm_internal.h"
#include "ptx_sm100.cuh"

namespace ggm {
namespace sp {

constexpr int kRowsPerBlock = 128;        // M (rows of Ψ per CTA tile; TMEM lanes)
constexpr int kTileN = 256;               // N (columns of Ψ per tile; 2 operand blocks)
constexpr int kAtomElems = 64;            // fp16 elements per 128-byte swizzle row
constexpr int kAtomBytes = kRowsPerBlock * 128;  // one (128-row block, K atom) = 16 KB
constexpr int kStages = 2;
constexpr int kThreads = 384;             // 12 warps: 4 role warps + 8 epilogue warps
constexpr int kTmemCols = 512;            // 2 accumulator buffers x 256 columns
constexpr int kMaxResidentAtoms = 2;
constexpr int kEpiWarps = 8;              // epilogue warps (2 per TMEM lane quadrant)
constexpr int kScratchFloats = 32 * 32;   // per epilogue warp: [32 values][32 lanes]      // A (128 rows x KA atoms x hi/lo) resident if KA<=2

__host__ __device__ inline size_t block_bytes(int KA) { return (size_t)2 * KA * kAtomBytes; }

struct DevScalars {
  unsigned int absmax_bits;  // float bits of max |U|
  int flags;                 // 1 = non-finite V, 2 = lambda <= 0 or non-finite
  int exp2;                  // e: s = 2^e
  int pad;
  unsigned long long coo_count;
};

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
  float m = 0.f;
  int bad = 0;
  const int64_t total = n * (int64_t)k;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    float v = V[idx];
    int c = (int)(idx % k);
    if (!isfinite(v)) bad = 1;
    double l = lam[c];
    float u = (float)(fabs((double)v) * sqrt(l > 0.0 ? l : 0.0));
    m = fmaxf(m, u);
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
__global__ void split_tile(const float* __restrict__ V, const double* __restrict__ lam,
                           int64_t n, int k, int KA, int64_t row0, int64_t nrows_pad,
                           const DevScalars* __restrict__ sc, uint8_t* __restrict__ dst) {
  const int chunks_per_row = KA * 8;
  const int64_t total = nrows_pad * chunks_per_row;
  const double s = ldexp(1.0, sc->exp2);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / chunks_per_row;
    const int ch = (int)(idx % chunks_per_row);
    const int64_t g = row0 + row;
    __align__(16) __half hi[8];
    __align__(16) __half lo[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = ch * 8 + e;
      double x = 0.0;
      if (g < n && c < k) x = (double)V[g * k + c] * sqrt(lam[c]) * s;
      __half h = __double2half(x);
      hi[e] = h;
      lo[e] = __double2half(x - (double)__half2float(h));
    }
    const int64_t b = row / kRowsPerBlock;
    const int r = (int)(row % kRowsPerBlock);
    const int a = ch >> 3, c8 = ch & 7;
    const size_t off = (size_t)b * block_bytes(KA) + (size_t)a * kAtomBytes + (size_t)r * 128 +
                       (size_t)((c8 ^ (r & 7)) * 16);
    *reinterpret_cast<uint4*>(dst + off) = *reinterpret_cast<const uint4*>(hi);
    *reinterpret_cast<uint4*>(dst + off + (size_t)KA * kAtomBytes) =
        *reinterpret_cast<const uint4*>(lo);
  }
}

// ------------------------------------------------------------------ BK2
struct FusedParams {
  const uint8_t* A;  // row-block operand (rows [row_begin,row_end)), tiled layout
  const uint8_t* B;  // column operand (all n rows, padded to 256), tiled layout
  int KA;            // K atoms of 64
  int KS;            // K steps of 16 actually issued (ceil(k/16))
  int resident;      // 1: A kept in shared memory for a whole row block
  int64_t n, row_begin, rows;
  int RB, NT, C, TPC;
  int mode, t;
  float tau;
  const DevScalars* sc;
  int64_t* row_ptr;
  int32_t* col;
  float* val;
  int32_t* pcol;
  float* pval;
  int64_t* coo_key;
  float* coo_val;
  unsigned long long* coo_count;
  int64_t capacity;
  int dbg;  // timing experiments only (GGM_DEBUG_EPI): 1 = TMEM loads only, 2 = no epilogue work
};

__host__ __device__ inline size_t stage_bytes(int resident) {
  return (resident ? 0 : (size_t)2 * kAtomBytes) + (size_t)4 * kAtomBytes;
}
__host__ inline size_t fused_smem_bytes(int KA, int resident) {
  size_t a = resident ? block_bytes(KA) : 0;
  return 1024 /*align slack*/ + a + kStages * stage_bytes(resident) + 256 /*barriers*/ +
         kEpiWarps * kScratchFloats * sizeof(float);
}

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
};

// Epilogue role (warps 4-11): TMEM -> registers, fused per-row top-t / threshold.
// Warp w handles TMEM lane quadrant q = w & 3 (thread = row) and column half h = (w-4) >> 2
// of every 256-column tile (4 x tcgen05.ld.32x32b.x32 per tile, the next chunk's load in
// flight while the current chunk is reduced).  Two warps share each row; their partial
// lists are merged through shared memory at the end of a unit.  Fast path per 32 values:
// 4 independent FMNMX3 chains of |v| against the row's current t-th magnitude; the rare
// path stages the chunk in the warp's shared scratch and inserts candidates in column order.

__device__ __forceinline__ float max32_abs(const float (&v)[32]) {
  float m0 = fabsf(v[0]), m1 = fabsf(v[1]), m2 = fabsf(v[2]), m3 = fabsf(v[3]);
#pragma unroll
  for (int e = 4; e < 32; e += 8) {
    m0 = fmaxf(m0, fmaxf(fabsf(v[e + 0]), fabsf(v[e + 4])));
    m1 = fmaxf(m1, fmaxf(fabsf(v[e + 1]), fabsf(v[e + 5])));
    m2 = fmaxf(m2, fmaxf(fabsf(v[e + 2]), fabsf(v[e + 6])));
    m3 = fmaxf(m3, fmaxf(fabsf(v[e + 3]), fabsf(v[e + 7])));
  }
  return fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
}

template <int MAXT>
__device__ __forceinline__ void epilogue_role(const FusedParams& p, uint32_t tmem_base,
                                              uint64_t* tfull, uint64_t* tempty, int unit0,
                                              int ustride, int units, int rows_per_unit,
                                              int row_off, bool remote_arrive, int warp,
                                              int lane, float* scratch_all) {
  const int ew = warp - 4;
  const int q = warp & 3;   // TMEM lane quadrant accessible to this warp
  const int h = ew >> 2;    // column half of each tile
  const int r = q * 32 + lane;
  float* scratch = scratch_all + ew * kScratchFloats;
  const float scale_down = ldexpf(1.f, -p.sc->exp2);  // ψ = acc · 2^-e · 2^-e
  const float tau_s = ldexpf(ldexpf(p.tau, p.sc->exp2), p.sc->exp2);
  const float qnan = __int_as_float(0x7fc00000);
  const int t = p.t;
  int buf = 0;
  uint32_t tphase = 0;
  TopList<MAXT> top;
  for (int u = unit0; u < units; u += ustride) {
    const int rb = u / p.C, cc = u % p.C;
    const int j0 = cc * p.TPC, j1 = min(p.NT, j0 + p.TPC);
    const int64_t lr = (int64_t)rb * rows_per_unit + row_off + r;
    const bool valid = lr < p.rows;
    const int64_t gi = p.row_begin + lr;
    top.init(t);
    for (int j = j0; j < j1; ++j) {
      mbar_wait(&tfull[buf], tphase);
      tc_fence_after();
      const uint32_t taddr =
          tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kTileN + h * (kTileN / 2));
      const int nchunks = p.dbg == 2 ? 0 : (kTileN / 2) / 32;
      uint32_t vn[32];
      if (nchunks) tmem_ld32_nowait(taddr, vn);
#pragma unroll 1
      for (int c = 0; c < nchunks; ++c) {
        float v[32];
        tmem_wait_ld(vn);
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(vn[e]);
        if (c + 1 < nchunks) tmem_ld32_nowait(taddr + (c + 1) * 32, vn);
        if (p.dbg == 1) {
          if (v[0] == 12345.f && v[31] == 54321.f) p.row_ptr[0] = (int64_t)v[7];
          continue;
        }
        const int64_t col0 = (int64_t)j * kTileN + h * (kTileN / 2) + c * 32;
        if (((uint64_t)(gi - col0) < 32ull) || (col0 + 32 > p.n)) {
          // diagonal (j == i: not an edge, Q8) and padding columns (j >= n): NaN, ignored
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int64_t jj = col0 + e;
            if (jj == gi || jj >= p.n) v[e] = qnan;
          }
        }
        const float m = max32_abs(v);
        const float thr = p.mode == 0 ? top.thr() : tau_s;
        if (__any_sync(0xffffffffu, m > thr)) {
          // rare path: stage the chunk, then visit this thread's candidates in column order
          uint32_t mask = 0;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            scratch[e * 32 + lane] = v[e];
            mask |= (fabsf(v[e]) > thr ? 1u : 0u) << e;
          }
          __syncwarp();
          if (p.mode == 0) {
            while (mask) {
              const int e = __ffs(mask) - 1;
              mask &= mask - 1;
              const float x = scratch[e * 32 + lane];
              const float a = fabsf(x);
              if (a > top.thr()) top.insert(a, x, (int)(col0 + e));
            }
          } else if (valid && mask) {
            unsigned long long base =
                atomicAdd(p.coo_count, (unsigned long long)__popc(mask));
            while (mask) {
              const int e = __ffs(mask) - 1;
              mask &= mask - 1;
              if ((int64_t)base < p.capacity) {
                p.coo_key[base] = lr * p.n + col0 + e;
                p.coo_val[base] = scratch[e * 32 + lane] * scale_down * scale_down;
              }
              ++base;
            }
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (remote_arrive)
          mbar_arrive_cluster(&tempty[buf], 0);
        else
          mbar_arrive(&tempty[buf]);
      }
      if (++buf == 2) {
        buf = 0;
        tphase ^= 1;
      }
    }
    if (p.mode != 0) continue;
    // merge the two column halves of each row: half 1 publishes (values into its own
    // scratch, columns into the half-0 warp's), half 0 merges and emits.
    float* pv = scratch_all + (4 + q) * kScratchFloats;
    float* pc = scratch_all + q * kScratchFloats;
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
        if (p.C == 1) {
          // the list is full (t <= n-1 real columns scanned); emit in ascending column
          const int64_t base = lr * t;
#pragma unroll
          for (int a = 0; a < MAXT; ++a) {
            if (a < t) {
              int rank = 0;
#pragma unroll
              for (int b = 0; b < MAXT; ++b)
                if (b < t && top.idx[b] < top.idx[a]) ++rank;
              p.col[base + rank] = top.idx[a];
              p.val[base + rank] = top.sval[a] * scale_down * scale_down;
            }
          }
          p.row_ptr[lr] = base;
          if (lr == p.rows - 1) p.row_ptr[p.rows] = base + t;
        } else {
          const int64_t base = ((int64_t)cc * p.rows + lr) * t;
#pragma unroll
          for (int a = 0; a < MAXT; ++a) {
            if (a < t) {
              p.pcol[base + a] = top.idx[a];
              p.pval[base + a] = top.sval[a] * scale_down * scale_down;
            }
          }
        }
      }
    }
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
  }
}

template <int MAXT>
__global__ void __launch_bounds__(kThreads, 1) fused_recon_topk(const FusedParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int KA = p.KA;
  const int resident = p.resident;
  const size_t a_bytes = resident ? block_bytes(KA) : 0;
  const size_t st_bytes = stage_bytes(resident);
  uint8_t* sA = smem;
  uint8_t* sStage = smem + a_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + kStages * st_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tempty + 2;
  uint64_t* aempty = afull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);
  float* scratch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int units = p.RB * p.C;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (p.sc->flags != 0) {
    // invalid input: skip all work (status reported by the host after synchronising)
  } else if (warp == 0) {
    // ===================== producer: bulk async copies global -> shared ==============
    if (lane == 0) {
      const uint64_t pol_b = policy_evict_last();
      const uint64_t pol_a = policy_evict_first();
      const size_t bb = block_bytes(KA);
      int stage = 0;
      uint32_t phase = 0;
      int a_iter = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int rb = u / p.C, cc = u % p.C;
        const int j0 = cc * p.TPC, j1 = min(p.NT, j0 + p.TPC);
        const uint8_t* Ablk = p.A + (size_t)rb * bb;
        if (resident) {
          if (a_iter > 0) mbar_wait(aempty, (a_iter - 1) & 1);
          mbar_arrive_expect_tx(afull, (uint32_t)bb);
          bulk_g2s(sA, Ablk, (uint32_t)bb, afull, pol_a);
          ++a_iter;
        }
        for (int j = j0; j < j1; ++j) {
          const uint8_t* B0 = p.B + (size_t)(2 * j) * bb;
          const uint8_t* B1 = B0 + bb;
          for (int a = 0; a < KA; ++a) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = sStage + stage * st_bytes;
            mbar_arrive_expect_tx(&full[stage], (uint32_t)st_bytes);
            uint8_t* sb = st;
            if (!resident) {
              bulk_g2s(st, Ablk + (size_t)a * kAtomBytes, kAtomBytes, &full[stage], pol_a);
              bulk_g2s(st + kAtomBytes, Ablk + (size_t)(KA + a) * kAtomBytes, kAtomBytes,
                       &full[stage], pol_a);
              sb = st + 2 * kAtomBytes;
            }
            // B hi (rows 0-127 | 128-255), then B lo: 256 rows per atom, uniform 1 KB SBO
            bulk_g2s(sb, B0 + (size_t)a * kAtomBytes, kAtomBytes, &full[stage], pol_b);
            bulk_g2s(sb + kAtomBytes, B1 + (size_t)a * kAtomBytes, kAtomBytes, &full[stage],
                     pol_b);
            bulk_g2s(sb + 2 * kAtomBytes, B0 + (size_t)(KA + a) * kAtomBytes, kAtomBytes,
                     &full[stage], pol_b);
            bulk_g2s(sb + 3 * kAtomBytes, B1 + (size_t)(KA + a) * kAtomBytes, kAtomBytes,
                     &full[stage], pol_b);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer: one thread drives the tensor cores ==============
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(kRowsPerBlock, kTileN);
      int stage = 0;
      uint32_t phase = 0;
      int buf = 0;
      uint32_t tphase = 0;
      int a_iter = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int cc = u % p.C;
        const int j0 = cc * p.TPC, j1 = min(p.NT, j0 + p.TPC);
        if (resident) {
          mbar_wait(afull, a_iter & 1);
          tc_fence_after();
        }
        for (int j = j0; j < j1; ++j) {
          mbar_wait(&tempty[buf], tphase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(buf * kTileN);
          for (int a = 0; a < KA; ++a) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            uint8_t* st = sStage + stage * st_bytes;
            const uint8_t* aHi = resident ? sA + (size_t)a * kAtomBytes : st;
            const uint8_t* aLo = resident ? sA + (size_t)(KA + a) * kAtomBytes : st + kAtomBytes;
            const uint8_t* bHi = resident ? st : st + 2 * kAtomBytes;
            const uint8_t* bLo = bHi + 2 * kAtomBytes;
            const uint32_t aHi_s = smem_u32(aHi), aLo_s = smem_u32(aLo);
            const uint32_t bHi_s = smem_u32(bHi), bLo_s = smem_u32(bLo);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              if (a * 4 + ks < p.KS) {
                const uint32_t off = ks * 32;
                const uint32_t acc = (a | ks) ? 1u : 0u;
                mma_f16_ss(d_tmem, sw128_desc(aHi_s + off), sw128_desc(bHi_s + off), idesc, acc);
                mma_f16_ss(d_tmem, sw128_desc(aHi_s + off), sw128_desc(bLo_s + off), idesc, 1u);
                mma_f16_ss(d_tmem, sw128_desc(aLo_s + off), sw128_desc(bHi_s + off), idesc, 1u);
              }
            }
            mma_commit(&empty[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mma_commit(&tfull[buf]);
          if (++buf == 2) {
            buf = 0;
            tphase ^= 1;
          }
        }
        if (resident) {
          mma_commit(aempty);
          ++a_iter;
        }
      }
    }
  } else if (warp >= 4) {
    epilogue_role<MAXT>(p, tmem_base, tfull, tempty, blockIdx.x, gridDim.x, units,
                        kRowsPerBlock, 0, false, warp, lane, scratch);
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}


// ------------------------------------------------------------------ BK2, CTA-pair variant
// Two CTAs of a cluster (one TPC) run one tcgen05.mma.cta_group::2 pipeline: M = 256 rows
// (128 per CTA, accumulators in each CTA's TMEM), N = 256 columns with each CTA holding HALF
// of the B tile (128 rows) in its shared memory, so per-CTA operand traffic and smem
// footprint halve and the pipeline can be 4 stages deep.  The leader (cluster rank 0) issues
// the MMAs; both CTAs' producers load with tensor-map TMA crediting the leader's full
// barriers; tcgen05.commit multicasts stage/accumulator releases to both CTAs; the peer's
// epilogue releases TMEM buffers by remote mbarrier arrival on the leader.
constexpr int kPairStagesResident = 4;
constexpr int kPairStagesStreaming = 3;

__host__ __device__ inline size_t pair_stage_bytes(int resident) {
  return (resident ? 0 : (size_t)2 * kAtomBytes) + (size_t)2 * kAtomBytes;
}
__host__ __device__ inline int pair_stages(int resident) {
  return resident ? kPairStagesResident : kPairStagesStreaming;
}
__host__ inline size_t pair_smem_bytes(int KA, int resident) {
  size_t a = resident ? block_bytes(KA) : 0;
  return 1024 + a + pair_stages(resident) * pair_stage_bytes(resident) + 256 +
         kEpiWarps * kScratchFloats * sizeof(float);
}

template <int MAXT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    fused_recon_topk_pair(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmB, const FusedParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int KA = p.KA;
  const int resident = p.resident;
  const int S = pair_stages(resident);
  const size_t a_bytes = resident ? block_bytes(KA) : 0;
  const size_t st_bytes = pair_stage_bytes(resident);
  uint8_t* sA = smem;
  uint8_t* sStage = smem + a_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + S * st_bytes);
  uint64_t* full = bars;            // [S]  (leader's are used)
  uint64_t* empty = bars + 4;       // [S]  (both CTAs)
  uint64_t* tfull = bars + 8;       // [2]  (both CTAs)
  uint64_t* tempty = bars + 10;     // [2]  (leader's are used; 8 arrivals)
  uint64_t* afull = bars + 12;      // leader's used
  uint64_t* aempty = bars + 13;     // both
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  float* scratch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int units = p.RB * p.C;  // RB counts 256-row pair blocks here

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kEpiWarps);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const bool skip = p.sc->flags != 0;

  if (!skip && warp == 0) {
    // ===================== producers (both CTAs): tensor-map TMA into own smem =========
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      const uint64_t pol_b = policy_evict_last();
      const uint64_t pol_a = policy_evict_first();
      const int lines_per_block = 2 * KA * kRowsPerBlock;  // 128-byte lines per 128-row block
      int stage = 0;
      uint32_t phase = 0;
      int a_iter = 0;
      for (int u = pair; u < units; u += npairs) {
        const int rb2 = u / p.C, cc = u % p.C;
        const int j0 = cc * p.TPC, j1 = min(p.NT, j0 + p.TPC);
        const int ablk = rb2 * 2 + (int)rank;  // this CTA's 128 rows of the pair block
        const int aline = ablk * lines_per_block;
        if (resident) {
          if (a_iter > 0) mbar_wait(aempty, (a_iter - 1) & 1);
          if (rank == 0) mbar_arrive_expect_tx(afull, (uint32_t)(2 * block_bytes(KA)));
          for (int a = 0; a < 2 * KA; ++a)
            tma_load_2d_pair(sA + (size_t)a * kAtomBytes, &tmA, 0, aline + a * kRowsPerBlock,
                             afull, pol_a);
          ++a_iter;
        }
        for (int j = j0; j < j1; ++j) {
          const int bline = (2 * j + (int)rank) * lines_per_block;  // this CTA's half of B
          for (int a = 0; a < KA; ++a) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], (uint32_t)(2 * st_bytes));
            uint8_t* st = sStage + stage * st_bytes;
            uint8_t* sb = st;
            if (!resident) {
              tma_load_2d_pair(st, &tmA, 0, aline + a * kRowsPerBlock, &full[stage], pol_a);
              tma_load_2d_pair(st + kAtomBytes, &tmA, 0, aline + (KA + a) * kRowsPerBlock,
                               &full[stage], pol_a);
              sb = st + 2 * kAtomBytes;
            }
            tma_load_2d_pair(sb, &tmB, 0, bline + a * kRowsPerBlock, &full[stage], pol_b);
            tma_load_2d_pair(sb + kAtomBytes, &tmB, 0, bline + (KA + a) * kRowsPerBlock,
                             &full[stage], pol_b);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (!skip && warp == 1) {
    // ===================== MMA issuer (leader CTA only) ================================
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(2 * kRowsPerBlock, kTileN);
      int stage = 0;
      uint32_t phase = 0;
      int buf = 0;
      uint32_t tphase = 0;
      int a_iter = 0;
      for (int u = pair; u < units; u += npairs) {
        const int cc = u % p.C;
        const int j0 = cc * p.TPC, j1 = min(p.NT, j0 + p.TPC);
        if (resident) {
          mbar_wait(afull, a_iter & 1);
          tc_fence_after();
        }
        for (int j = j0; j < j1; ++j) {
          mbar_wait(&tempty[buf], tphase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(buf * kTileN);
          for (int a = 0; a < KA; ++a) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            uint8_t* st = sStage + stage * st_bytes;
            const uint8_t* aHi = resident ? sA + (size_t)a * kAtomBytes : st;
            const uint8_t* aLo = resident ? sA + (size_t)(KA + a) * kAtomBytes : st + kAtomBytes;
            const uint8_t* bHi = resident ? st : st + 2 * kAtomBytes;
            const uint8_t* bLo = bHi + kAtomBytes;
            const uint32_t aHi_s = smem_u32(aHi), aLo_s = smem_u32(aLo);
            const uint32_t bHi_s = smem_u32(bHi), bLo_s = smem_u32(bLo);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              if (a * 4 + ks < p.KS) {
                const uint32_t off = ks * 32;
                const uint32_t acc = (a | ks) ? 1u : 0u;
                mma_f16_ss_pair(d_tmem, sw128_desc(aHi_s + off), sw128_desc(bHi_s + off), idesc,
                                acc);
                mma_f16_ss_pair(d_tmem, sw128_desc(aHi_s + off), sw128_desc(bLo_s + off), idesc,
                                1u);
                mma_f16_ss_pair(d_tmem, sw128_desc(aLo_s + off), sw128_desc(bHi_s + off), idesc,
                                1u);
              }
            }
            mma_commit_pair(&empty[stage]);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
          mma_commit_pair(&tfull[buf]);
          if (++buf == 2) {
            buf = 0;
            tphase ^= 1;
          }
        }
        if (resident) {
          mma_commit_pair(aempty);
          ++a_iter;
        }
      }
    }
  } else if (!skip && warp >= 4) {
    epilogue_role<MAXT>(p, tmem_base, tfull, tempty, pair, npairs, units, 2 * kRowsPerBlock,
                        (int)rank * kRowsPerBlock, rank != 0, warp, lane, scratch);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
}

// ------------------------------------------------------------------ BK3 (mode 0, C > 1)
template <int MAXT>
__global__ void merge_partials(const int32_t* __restrict__ pcol, const float* __restrict__ pval,
                               int64_t rows, int C, int t, int64_t* row_ptr, int32_t* col,
                               float* val) {
  const int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (lr >= rows) return;
  float mag[MAXT], sv[MAXT];
  int id[MAXT];
#pragma unroll
  for (int a = 0; a < MAXT; ++a) {
    mag[a] = -1.f;
    sv[a] = 0.f;
    id[a] = INT_MAX;
  }
  for (int c = 0; c < C; ++c) {
    const int64_t base = ((int64_t)c * rows + lr) * t;
    for (int e = 0; e < t; ++e) {
      const int j = pcol[base + e];
      if (j < 0) continue;
      const float v = pval[base + e];
      const float a = fabsf(v);
      // insert by (|v| desc, j asc)
#pragma unroll
      for (int s = MAXT - 1; s >= 1; --s) {
        if (s < t) {
          const bool before_prev = a > mag[s - 1] || (a == mag[s - 1] && j < id[s - 1]);
          const bool before_cur = a > mag[s] || (a == mag[s] && j < id[s]);
          if (before_prev) {
            mag[s] = mag[s - 1];
            sv[s] = sv[s - 1];
            id[s] = id[s - 1];
          } else if (before_cur) {
            mag[s] = a;
            sv[s] = v;
            id[s] = j;
          }
        }
      }
      if (a > mag[0] || (a == mag[0] && j < id[0])) {
        mag[0] = a;
        sv[0] = v;
        id[0] = j;
      }
    }
  }
  const int64_t base = lr * t;
#pragma unroll
  for (int a = 0; a < MAXT; ++a) {
    if (a < t) {
      int rank = 0;
#pragma unroll
      for (int b = 0; b < MAXT; ++b)
        if (b < t && id[b] < id[a]) ++rank;
      col[base + rank] = id[a];
      val[base + rank] = sv[a];
    }
  }
  row_ptr[lr] = base;
  if (lr == rows - 1) row_ptr[rows] = base + t;
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
  int k, KA, KS, t, mode, resident, alias, pair;
  int64_t RB, NT, C, TPC;
  int64_t nBblocks, nAblocks;
  int64_t capacity;
  size_t coo_temp_bytes;
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

static ggm_status make_plan(int64_t n, int k, int64_t row_begin, int64_t row_end,
                            const ggm_sparsify_opts* o, int64_t capacity, Plan* pl) {
  if (!o) return fail(GGM_ERR_INVALID_ARGUMENT, "opts is NULL");
  if (n < 2) return fail(GGM_ERR_INVALID_ARGUMENT, "n=%lld < 2", (long long)n);
  if (n > (int64_t)INT_MAX - 256) return fail(GGM_ERR_INVALID_ARGUMENT, "n too large for int32 columns");
  if (k < 1 || k > n) return fail(GGM_ERR_INVALID_ARGUMENT, "k=%d not in [1,n]", k);
  if (row_begin < 0 || row_end > n || row_begin >= row_end)
    return fail(GGM_ERR_INVALID_ARGUMENT, "row range [%lld,%lld) invalid for n=%lld",
                (long long)row_begin, (long long)row_end, (long long)n);
  if (o->mode != 0 && o->mode != 1) return fail(GGM_ERR_INVALID_ARGUMENT, "mode=%d", o->mode);
  if (o->mode == 0 && (o->topk < 1))
    return fail(GGM_ERR_INVALID_ARGUMENT, "topk=%d < 1", o->topk);
  if (o->mode == 0 && o->topk > GGM_MAX_TOPK)
    return fail(GGM_ERR_UNSUPPORTED, "topk=%d > GGM_MAX_TOPK=%d", o->topk, GGM_MAX_TOPK);
  if (o->mode == 1 && !(o->tau >= 0.f && std::isfinite(o->tau)))
    return fail(GGM_ERR_INVALID_ARGUMENT, "tau must be finite and >= 0");
  if (o->col_chunks < 0) return fail(GGM_ERR_INVALID_ARGUMENT, "col_chunks < 0");
  pl->n = n;
  pl->k = k;
  pl->row_begin = row_begin;
  pl->rows = row_end - row_begin;
  pl->mode = o->mode;
  pl->t = (int)std::min<int64_t>(o->topk, n - 1);
  pl->KA = (k + kAtomElems - 1) / kAtomElems;
  pl->KS = (k + 15) / 16;
  pl->resident = pl->KA <= kMaxResidentAtoms ? 1 : 0;
  // 1-CTA kernel by default (faster end to end); GGM_PAIR=1 selects the
  // CTA-pair (cta_group::2) kernel, which has the faster MMA pipeline but couples the two
  // CTAs' epilogues.
  const char* env = getenv("GGM_PAIR");
  pl->pair = (env && env[0] == '1') ? 1 : 0;
  const int rows_per_unit = pl->pair ? 2 * kRowsPerBlock : kRowsPerBlock;
  pl->alias = (row_begin % rows_per_unit) == 0 ? 1 : 0;
  pl->NT = (n + kTileN - 1) / kTileN;
  pl->RB = (pl->rows + rows_per_unit - 1) / rows_per_unit;
  pl->nBblocks = pl->NT * 2;
  pl->nAblocks = pl->alias ? 0 : pl->RB * (rows_per_unit / kRowsPerBlock);
  const int sms = pl->pair ? num_sms() / 2 : num_sms();
  int64_t C = o->col_chunks > 0 ? o->col_chunks : (pl->mode == 0 ? choose_chunks(pl->RB, pl->NT, sms) : 1);
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
};

static size_t carve(const Plan& pl, void* ws, Work* w) {
  Carve cv(ws);
  w->sc = cv.take<DevScalars>(1);
  w->Bop = cv.take<uint8_t>((size_t)pl.nBblocks * block_bytes(pl.KA));
  w->Aop = cv.take<uint8_t>((size_t)pl.nAblocks * block_bytes(pl.KA));
  const size_t npart = (pl.mode == 0 && pl.C > 1) ? (size_t)pl.C * pl.rows * pl.t : 0;
  w->pcol = cv.take<int32_t>(npart);
  w->pval = cv.take<float>(npart);
  const size_t ncoo = pl.mode == 1 ? (size_t)std::max<int64_t>(pl.capacity, 0) : 0;
  w->key_in = cv.take<int64_t>(ncoo);
  w->key_out = cv.take<int64_t>(ncoo);
  w->cv_in = cv.take<float>(ncoo);
  w->cv_out = cv.take<float>(ncoo);
  w->cub_tmp = cv.take<char>(pl.coo_temp_bytes);
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

template <int MAXT>
static cudaError_t launch_fused(const FusedParams& fp, size_t smem, int grid, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(fused_recon_topk<MAXT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fused_recon_topk<MAXT><<<grid, kThreads, smem, st>>>(fp);
  return cudaGetLastError();
}


// 2-D tensor map over a tiled operand array viewed as lines of 128 bytes (64 x uint16):
// box = 128 lines = one 16 KB (128-row block, K atom) chunk, no swizzle (the data is already
// stored in the SWIZZLE_128B canonical layout by split_tile).
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

template <int MAXT>
static cudaError_t launch_pair(const CUtensorMap& tmA, const CUtensorMap& tmB,
                               const FusedParams& fp, size_t smem, int grid, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(fused_recon_topk_pair<MAXT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fused_recon_topk_pair<MAXT><<<grid, kThreads, smem, st>>>(tmA, tmB, fp);
  return cudaGetLastError();
}

}  // namespace sp
}  // namespace ggm

using namespace ggm;
using namespace ggm::sp;

extern "C" ggm_status ggm_sparse_precision_workspace(int64_t n, int k, int64_t row_begin,
                                                     int64_t row_end,
                                                     const ggm_sparsify_opts* opts,
                                                     int64_t capacity, size_t* bytes) {
  if (!bytes) return fail(GGM_ERR_INVALID_ARGUMENT, "bytes is NULL");
  Plan pl;
  ggm_status st = make_plan(n, k, row_begin, row_end, opts, capacity, &pl);
  if (st != GGM_OK) return st;
  Work w;
  *bytes = carve(pl, nullptr, &w);
  return GGM_OK;
}

extern "C" ggm_status ggm_sparse_precision(int64_t n, int k, const float* V, const double* lambda,
                                           int64_t row_begin, int64_t row_end,
                                           const ggm_sparsify_opts* opts, int64_t* row_ptr,
                                           int32_t* col, float* val, int64_t capacity,
                                           int64_t* nnz_out, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  if (!V || !lambda || !row_ptr || !nnz_out || !workspace)
    return fail(GGM_ERR_INVALID_ARGUMENT, "null pointer argument");
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
  EventTimer tm(timing_enabled(), s);
  tm.mark(0);
  GGM_CUDA_TRY(cudaMemsetAsync(w.sc, 0, sizeof(DevScalars), s));
  const int sms = num_sms();
  {
    const int64_t total = n * (int64_t)k;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, sms * 8));
    absmax_check<<<grid, 256, 0, s>>>(V, lambda, n, k, w.sc);
    scale_finalize<<<1, 1, 0, s>>>(w.sc);
    count_launches(pl.alias ? 3 : 4);
    const int64_t totB = (int64_t)pl.nBblocks * kRowsPerBlock * pl.KA * 8;
    split_tile<<<(int)std::min<int64_t>((totB + 255) / 256, sms * 16), 256, 0, s>>>(
        V, lambda, n, k, pl.KA, 0, (int64_t)pl.nBblocks * kRowsPerBlock, w.sc, w.Bop);
    if (!pl.alias) {
      const int64_t totA = (int64_t)pl.nAblocks * kRowsPerBlock * pl.KA * 8;  // rows padded
      split_tile<<<(int)std::min<int64_t>((totA + 255) / 256, sms * 16), 256, 0, s>>>(
          V, lambda, n, k, pl.KA, row_begin, (int64_t)pl.nAblocks * kRowsPerBlock, w.sc, w.Aop);
    }
    GGM_CUDA_TRY(cudaGetLastError());
  }
  tm.mark(1);
  FusedParams fp{};
  fp.B = w.Bop;
  fp.A = pl.alias ? w.Bop + (size_t)(row_begin / kRowsPerBlock) * block_bytes(pl.KA) : w.Aop;
  fp.KA = pl.KA;
  fp.KS = pl.KS;
  fp.resident = pl.resident;
  fp.n = n;
  fp.row_begin = row_begin;
  fp.rows = pl.rows;
  fp.RB = (int)pl.RB;
  fp.NT = (int)pl.NT;
  fp.C = (int)pl.C;
  fp.TPC = (int)pl.TPC;
  fp.mode = pl.mode;
  fp.t = pl.t;
  fp.tau = pl.mode == 1 ? opts->tau : 0.f;
  fp.sc = w.sc;
  fp.row_ptr = row_ptr;
  fp.col = (pl.mode == 0 && pl.C == 1) ? col : nullptr;
  fp.val = (pl.mode == 0 && pl.C == 1) ? val : nullptr;
  fp.pcol = w.pcol;
  fp.pval = w.pval;
  fp.coo_key = w.key_in;
  fp.coo_val = w.cv_in;
  fp.coo_count = &w.sc->coo_count;
  fp.capacity = pl.mode == 1 ? capacity : 0;
  {
    const char* d = getenv("GGM_DEBUG_EPI");
    fp.dbg = d ? atoi(d) : 0;
  }
  cudaError_t ce;
  if (pl.pair) {
    const int lines_per_block = 2 * pl.KA * kRowsPerBlock;
    CUtensorMap tmA, tmB;
    const uint64_t linesB = (uint64_t)pl.nBblocks * lines_per_block;
    const uint64_t linesA = pl.alias ? linesB - (uint64_t)(row_begin / kRowsPerBlock) * lines_per_block
                                     : (uint64_t)pl.nAblocks * lines_per_block;
    ggm_status ts = make_line_tmap(&tmB, w.Bop, linesB);
    if (ts == GGM_OK) ts = make_line_tmap(&tmA, fp.A, linesA);
    if (ts != GGM_OK) return ts;
    const size_t smem = pair_smem_bytes(pl.KA, pl.resident);
    const int pairs = (int)std::min<int64_t>(sms / 2, pl.RB * pl.C);
    const int g2 = 2 * pairs;
    ce = pl.t <= 5    ? launch_pair<5>(tmA, tmB, fp, smem, g2, s)
         : pl.t <= 10 ? launch_pair<10>(tmA, tmB, fp, smem, g2, s)
         : pl.t <= 16 ? launch_pair<16>(tmA, tmB, fp, smem, g2, s)
                      : launch_pair<32>(tmA, tmB, fp, smem, g2, s);
  } else {
    const size_t smem = fused_smem_bytes(pl.KA, pl.resident);
    const int grid = (int)std::min<int64_t>(sms, pl.RB * pl.C);
    ce = pl.t <= 5    ? launch_fused<5>(fp, smem, grid, s)
         : pl.t <= 10 ? launch_fused<10>(fp, smem, grid, s)
         : pl.t <= 16 ? launch_fused<16>(fp, smem, grid, s)
                      : launch_fused<32>(fp, smem, grid, s);
  }
  if (ce != cudaSuccess)
    return fail(GGM_ERR_CUDA, "fused_recon_topk launch: %s", cudaGetErrorString(ce));
  count_launches(1);
  tm.mark(2);

  DevScalars hs;
  if (pl.mode == 0) {
    if (pl.C > 1) {
      const int threads = 128;
      const int blocks = (int)((pl.rows + threads - 1) / threads);
      if (pl.t <= 16)
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
}
