// gram_tc.cu — fp32-accurate tensor-core Gram G += Cᵀ C for the chunked exact Gram of sparse
// (or COCA-transformed) unfoldings (ggm_gram_eig_csr; Alg. 1 lines 2-4,
// P:909-912; Thm 1).  C is a dense chunk of the unfolding, samples x dim, element
// (sample c, column g) at C[c·rs + g·cs]: the samples are entries of the long side, the
// columns the side whose Gram is formed (genes for a cell axis, etc.).
//
// Split: C·2^e = hi + lo with hi = fp16(x), lo = fp16(x - hi) and one power-of-two scale e
// (max|C|·2^e < 2^14, the BK1 rule), so Cᵀ C · 2^2e ≈ hiᵀhi + hiᵀlo + loᵀhi (the dropped loᵀlo
// is 2^-22 relative); the products run on tcgen05 (kind::f16, M = 128, N = 256, K = 16),
// accumulate in fp32 in TMEM over one k-slice of kSliceAtoms x 64 samples, and the slice
// results are added into G in fp64 (red), so the fp32 accumulation error is that of a
// 4,096-term sum.  DESIGN.md BK5c (tools/gram_precision_probe.py: an fp32-accurate Gram
// keeps the selected ψ within 1e-5 of the fp64 pipeline at C2, 10x under the 1e-4 gate).
//
// Operand layout (split_T): [128-column block b][atom a][hi | lo][128 rows x 128 B], the
// SWIZZLE_128B K-major canonical layout of BK1 (16-B chunk q of row r at chunk q ^ (r & 7)),
// K = samples: one atom = 128 Gram-side columns x 64 samples.
//
// Work unit = (upper tile (I, J2): rows of block I, columns of the 256-wide super block J2,
// k-slice); units are slice-major so the concurrently running ones share their atoms in L2.
// Roles (192 threads): warp 0 producer (bulk copies, 2 stages x 96 KB), warp 1 MMA issuer
// (12 MMAs per atom), warps 2-5 epilogue (TMEM lane quadrants 2, 3, 0, 1: fp64 red of the
// upper-triangle entries into G, row-major upper = column-major lower for cuSOLVER).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "ggm_internal.h"
#include "ptx_sm100.cuh"

namespace ggm {
namespace gt {

constexpr int kAtomBytes = 128 * 128;        // 128 rows x 64 fp16
constexpr int kStages = 2;
constexpr int kStageBytes = 6 * kAtomBytes;  // A hi | A lo | B hi (2 blocks) | B lo (2 blocks)
constexpr int kThreads = 192;
constexpr int kTileN = 256;
constexpr int kDefaultSliceAtoms = 16;

struct Scal {
  unsigned int absmax_bits;
  int exp2;
};

__global__ void chunk_absmax(const double* __restrict__ C, int64_t count, Scal* sc) {
  float m = 0.f;  // the chunk is one dense block of `count` doubles
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, (float)fabs(C[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&sc->absmax_bits, __float_as_uint(m));
}

__global__ void chunk_scale(Scal* sc) {
  const float m = __uint_as_float(sc->absmax_bits);
  int e = 0;
  if (m > 0.f && isfinite(m)) {
    int ex;
    frexpf(m * 1.0001f, &ex);  // m < 2^ex (margin for the fp32 rounding of the max)
    e = max(-100, min(100, 14 - ex));
  }
  sc->exp2 = e;
}

// One CTA per (128-column block b, atom a): the 64 x 128 sub-block of C through shared
// memory (coalesced along columns), then 16-byte chunks of 8 samples per output row.
__global__ void __launch_bounds__(256) split_T(const double* __restrict__ C, int64_t rows,
                                               int64_t dim, int64_t rs, int64_t cs, int natoms,
                                               const Scal* __restrict__ sc,
                                               uint8_t* __restrict__ op) {
  __shared__ float tile[64][129];
  const int b = blockIdx.y, a = blockIdx.x;
  const int64_t c0 = (int64_t)a * 64, g0 = (int64_t)b * 128;
  const double s = ldexp(1.0, sc->exp2);
  const bool samples_fast = rs == 1;  // coalesce along whichever index is contiguous
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) {
    const int cr = samples_fast ? (i & 63) : (i >> 7);
    const int gc = samples_fast ? (i >> 6) : (i & 127);
    const int64_t c = c0 + cr, g = g0 + gc;
    tile[cr][gc] = (c < rows && g < dim) ? (float)(C[c * rs + g * cs] * s) : 0.f;
  }
  __syncthreads();
  uint8_t* atom = op + ((size_t)b * natoms + a) * 2 * kAtomBytes;
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    const int r = i >> 3, q = i & 7;  // output row (column of C), 16-B chunk (8 samples)
    __align__(16) __half hv[8], lv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float x = tile[q * 8 + e][r];
      const __half h = __float2half_rn(x);
      hv[e] = h;
      lv[e] = __float2half_rn(x - __half2float(h));
    }
    const size_t off = (size_t)r * 128 + (size_t)((q ^ (r & 7)) * 16);
    *reinterpret_cast<uint4*>(atom + off) = *reinterpret_cast<const uint4*>(hv);
    *reinterpret_cast<uint4*>(atom + kAtomBytes + off) = *reinterpret_cast<const uint4*>(lv);
  }
}

struct GtParams {
  const uint8_t* op;
  int slice_atoms;   // fp32 TMEM accumulation over slice_atoms x 64 samples
  int natoms, nblk;  // atoms of this chunk; 128-column blocks (even)
  int ntiles, nslices;
  int64_t dim;
  double* G;  // dim x dim row-major, upper triangle accumulated
  const Scal* sc;
};

// tile t -> (I, J2) over the upper super-tiles: for I = 0.., J2 from I/2 to nblk/2 - 1
__device__ __forceinline__ void tile_of(int t, int nblk, int& I, int& J2) {
  const int ns = nblk / 2;
  I = 0;
  for (;;) {
    const int cnt = ns - I / 2;
    if (t < cnt) break;
    t -= cnt;
    ++I;
  }
  J2 = I / 2 + t;
}

__global__ void __launch_bounds__(kThreads, 1) gram_tc_kernel(const GtParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nunits = p.ntiles * p.nslices;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // the four epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const size_t bstride = (size_t)p.natoms * 2 * kAtomBytes;  // one 128-column block

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer
      const uint64_t pol = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int slice = u / p.ntiles;
        int I, J2;
        tile_of(u % p.ntiles, p.nblk, I, J2);
        const int a0 = slice * p.slice_atoms, a1 = min(p.natoms, a0 + p.slice_atoms);
        for (int a = a0; a < a1; ++a) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * kStageBytes;
          mbar_arrive_expect_tx(&full[stage], (uint32_t)kStageBytes);
          const uint8_t* A = p.op + (size_t)I * bstride + (size_t)a * 2 * kAtomBytes;
          const uint8_t* B0 = p.op + (size_t)(2 * J2) * bstride + (size_t)a * 2 * kAtomBytes;
          const uint8_t* B1 = B0 + bstride;
          bulk_g2s(st, A, 2 * kAtomBytes, &full[stage], pol);                    // A hi, lo
          bulk_g2s(st + 2 * kAtomBytes, B0, kAtomBytes, &full[stage], pol);       // B hi rows 0-127
          bulk_g2s(st + 3 * kAtomBytes, B1, kAtomBytes, &full[stage], pol);       // B hi rows 128-255
          bulk_g2s(st + 4 * kAtomBytes, B0 + kAtomBytes, kAtomBytes, &full[stage], pol);  // B lo
          bulk_g2s(st + 5 * kAtomBytes, B1 + kAtomBytes, kAtomBytes, &full[stage], pol);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer
    constexpr uint32_t idesc = idesc_f16_f32(128, kTileN);
    const bool issuer = elect_one();
    int stage = 0, buf = 0;
    uint32_t phase = 0, tphase = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int slice = u / p.ntiles;
      const int a0 = slice * p.slice_atoms, a1 = min(p.natoms, a0 + p.slice_atoms);
      mbar_wait(&tempty[buf], tphase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + (uint32_t)(buf * kTileN);
      for (int a = a0; a < a1; ++a) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + stage * kStageBytes);
        const uint64_t dAh = sw128_desc(st), dAl = sw128_desc(st + kAtomBytes);
        const uint64_t dBh = sw128_desc(st + 2 * kAtomBytes), dBl = sw128_desc(st + 4 * kAtomBytes);
        if (issuer) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t o = (uint64_t)(2 * ks);
            mma_f16_ss(d, dAh + o, dBh + o, idesc, (a > a0 || ks > 0) ? 1u : 0u);
            mma_f16_ss(d, dAh + o, dBl + o, idesc, 1u);
            mma_f16_ss(d, dAl + o, dBh + o, idesc, 1u);
          }
          mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (issuer) mma_commit(&tfull[buf]);
      __syncwarp();
      if (++buf == 2) {
        buf = 0;
        tphase ^= 1;
      }
    }
  } else {  // ---------------- epilogue: warps 2..5 = TMEM lane quadrants 2, 3, 0, 1
    const int q = warp & 3;
    const double inv = ldexp(1.0, -2 * p.sc->exp2);
    int buf = 0;
    uint32_t tphase = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      int I, J2;
      tile_of(u % p.ntiles, p.nblk, I, J2);
      mbar_wait(&tfull[buf], tphase);
      tc_fence_after();
      const int64_t i = (int64_t)I * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kTileN);
#pragma unroll 1
      for (int c = 0; c < kTileN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32_nowait(taddr + c * 32, v);
        tmem_wait_ld(v);
        const int64_t j0 = (int64_t)J2 * kTileN + c * 32;
        if (i < p.dim && j0 + 31 >= i) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int64_t j = j0 + e;
            if (j >= i && j < p.dim)
              atomicAdd(p.G + i * p.dim + j, (double)__uint_as_float(v[e]) * inv);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (++buf == 2) {
        buf = 0;
        tphase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// ---------------------------------------------------------------- CSR operands (no dense chunk)
// The unfolding is A = S + z 1ᵀ (S sparse on the data's pattern, z the value of a row's zeros:
// 0 for raw data, the COCA image of 0 for the nonparanormal skeptic; the sparse rank-one form
// of P:1003-1012).  The tensor cores form only the Gram of S (operand: zero fill + scatter of
// the stored entries, straight from the CSR); the rank-one terms are added exactly in fp64
// afterwards (gram_tc_csr_rank1) — they carry the large common offset of COCA data, whose
// share of the fp32 accumulation bias would otherwise land on the small eigenvalues.
// rows_side: samples = CSR rows [r0, r1), Gram side = the m CSR columns; else samples = CSR
// columns [r0, r1), Gram side = the d CSR rows.
__device__ __forceinline__ void split16(float x, __half& h, __half& l) {
  h = __float2half_rn(x);
  l = __float2half_rn(x - __half2float(h));
}
__device__ __forceinline__ size_t op_off(int64_t b, int64_t a, int r, int e, int natoms) {
  return ((size_t)b * natoms + a) * 2 * kAtomBytes + (size_t)r * 128 +
         (size_t)((((e >> 3) ^ (r & 7)) << 4) + ((e & 7) << 1));
}

__global__ void csr_absmax(const int64_t* __restrict__ rp, const double* __restrict__ sval,
                           int64_t nrows, Scal* sc) {
  float m = 0.f;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nrows;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    for (int64_t q = rp[i] + (threadIdx.x & 31); q < rp[i + 1]; q += 32)
      m = fmaxf(m, (float)fabs(sval[q]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&sc->absmax_bits, __float_as_uint(m));
}

// scatter: one warp per CSR row; rows_side: CSR row = sample, col = Gram row; else CSR row =
// Gram row, col = sample (only columns in [r0, r1), columns ascending within a row)
__global__ void csr_scatter(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const double* __restrict__ sval, bool rows_side, int64_t r0, int64_t r1, int64_t nrows, int natoms,
                            const Scal* __restrict__ sc, uint8_t* __restrict__ op) {
  const double s = ldexp(1.0, sc->exp2);
  const int lane = threadIdx.x & 31;
  const int64_t ibeg = rows_side ? r0 : 0, iend = rows_side ? r1 : nrows;
  for (int64_t i = ibeg + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < iend;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t lo = rp[i];
    const int64_t hi = rp[i + 1];
    if (!rows_side) {  // first stored entry with col >= r0
      int64_t a0 = lo, b0 = hi;
      while (a0 < b0) {
        const int64_t mid = (a0 + b0) >> 1;
        if (col[mid] < r0) a0 = mid + 1; else b0 = mid;
      }
      lo = a0;
    }
    for (int64_t q = lo + lane; q < hi; q += 32) {
      const int64_t c = col[q];
      if (!rows_side && c >= r1) break;
      const int64_t smp = rows_side ? i - r0 : c - r0;  // sample index within the chunk
      const int64_t g = rows_side ? c : i;              // Gram-side index
      __half h, l;
      split16((float)(sval[q] * s), h, l);
      const size_t off = op_off(g >> 7, smp >> 6, (int)(g & 127), (int)(smp & 63), natoms);
      *reinterpret_cast<__half*>(op + off) = h;
      *reinterpret_cast<__half*>(op + kAtomBytes + off) = l;
    }
  }
}

// rank-one terms: rows_side (A = S + z 1ᵀ, rows = samples): AᵀA = SᵀS + u1ᵀ + 1uᵀ + (zᵀz)11ᵀ,
// u = Sᵀz; else (rows = Gram side): AAᵀ = SSᵀ + r zᵀ + z rᵀ + n zzᵀ, r = S1, n = #columns.
__global__ void rank1_vec(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                          const double* __restrict__ sval, const double* __restrict__ z,
                          int64_t d, bool rows_side, double* __restrict__ u, double* __restrict__ zz) {
  const int lane = threadIdx.x & 31;
  double zacc = 0.0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < d;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double zi = z[i];
    if (lane == 0) zacc += zi * zi;
    double rs = 0.0;
    for (int64_t q = rp[i] + lane; q < rp[i + 1]; q += 32) {
      if (rows_side)
        atomicAdd(&u[col[q]], sval[q] * zi);
      else
        rs += sval[q];
    }
    if (!rows_side) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
      if (lane == 0) u[i] = rs;
    }
  }
  if (lane == 0) atomicAdd(zz, zacc);
}
__global__ void rank1_apply(double* __restrict__ G, int64_t dim, const double* __restrict__ u,
                            const double* __restrict__ z, const double* __restrict__ zz,
                            bool rows_side, double ncols) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < dim * dim;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / dim, j = t - i * dim;
    if (j < i) continue;  // row-major upper triangle (column-major lower)
    G[t] += rows_side ? u[i] + u[j] + *zz : u[i] * z[j] + z[i] * u[j] + ncols * z[i] * z[j];
  }
}

}  // namespace gt

namespace {
size_t tc_ws(int64_t max_rows, int64_t dim) {
  const int64_t natoms = (max_rows + 63) / 64;
  int64_t nblk = (dim + 127) / 128;
  nblk += nblk & 1;
  return align_up(sizeof(gt::Scal), 256) + (size_t)nblk * natoms * 2 * gt::kAtomBytes + 1024;
}
uint8_t* tc_op(void* ws) {
  uint8_t* op = static_cast<uint8_t*>(ws) + align_up(sizeof(gt::Scal), 256);
  return op + ((1024u - (reinterpret_cast<uintptr_t>(op) & 1023u)) & 1023u);
}
// the Gram kernel over an operand of `rows` samples already in ws
ggm_status tc_run(int64_t rows, int64_t dim, double* G, void* ws, cudaStream_t s) {
  using namespace gt;
  const int natoms = (int)((rows + 63) / 64);
  int nblk = (int)((dim + 127) / 128);
  nblk += nblk & 1;
  GtParams p;
  p.op = tc_op(ws);
  p.natoms = natoms;
  p.nblk = nblk;
  p.ntiles = 0;
  for (int I = 0; I < nblk; ++I) p.ntiles += nblk / 2 - I / 2;
  static const int slice = [] {
    const char* e = getenv("GGM_GRAM_TC_SLICE");  // A/B hook: atoms per fp32 slice
    return e ? std::max(1, atoi(e)) : kDefaultSliceAtoms;
  }();
  p.slice_atoms = slice;
  p.nslices = (natoms + slice - 1) / slice;
  p.dim = dim;
  p.G = G;
  p.sc = static_cast<const Scal*>(ws);
  const size_t smem = (size_t)kStages * kStageBytes + 1024 + 256;
  static bool attr = false;
  if (!attr) {
    GGM_CUDA_TRY(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    attr = true;
  }
  const int units = p.ntiles * p.nslices;
  gram_tc_kernel<<<std::max(1, std::min(units, num_sms())), kThreads, smem, s>>>(p);
  GGM_CUDA_TRY(cudaGetLastError());
  return GGM_OK;
}
}  // namespace

// Workspace bytes of gram_tc_accumulate / gram_tc_accumulate_csr for chunks of up to
// max_rows samples.
size_t gram_tc_workspace(int64_t max_rows, int64_t dim) { return tc_ws(max_rows, dim); }

// G (dim x dim, fp64, row-major upper triangle) += Cᵀ C for the chunk C (rows samples x dim
// columns, element (c, g) at C[c·rs + g·cs], one dense block of rows·dim doubles) on `s`.
// ws: gram_tc_workspace(rows, dim) bytes.
ggm_status gram_tc_accumulate(const double* C, int64_t rows, int64_t dim, int64_t rs, int64_t cs,
                              double* G, void* ws, cudaStream_t s) {
  using namespace gt;
  if (rows <= 0) return GGM_OK;
  Scal* sc = static_cast<Scal*>(ws);
  const int natoms = (int)((rows + 63) / 64);
  int nblk = (int)((dim + 127) / 128);
  nblk += nblk & 1;
  const int sms = num_sms();
  GGM_CUDA_TRY(cudaMemsetAsync(sc, 0, sizeof(Scal), s));
  chunk_absmax<<<(int)std::min<int64_t>((rows * dim + 255) / 256, sms * 8), 256, 0, s>>>(
      C, rows * dim, sc);
  chunk_scale<<<1, 1, 0, s>>>(sc);
  split_T<<<dim3(natoms, nblk), 256, 0, s>>>(C, rows, dim, rs, cs, natoms, sc, tc_op(ws));
  GGM_CUDA_TRY(cudaGetLastError());
  count_launches(4);
  return tc_run(rows, dim, G, ws, s);
}

// The scale of a whole CSR unfolding (values sval + z at stored entries, z elsewhere), once
// per call before the chunk loop of gram_tc_accumulate_csr.
ggm_status gram_tc_csr_scale(const int64_t* rp, const double* sval, int64_t nrows, void* ws,
                             cudaStream_t s) {
  using namespace gt;
  Scal* sc = static_cast<Scal*>(ws);
  GGM_CUDA_TRY(cudaMemsetAsync(sc, 0, sizeof(Scal), s));
  csr_absmax<<<(int)std::max<int64_t>(1, std::min<int64_t>((nrows * 32 + 255) / 256, num_sms() * 8)),
               256, 0, s>>>(rp, sval, nrows, sc);
  chunk_scale<<<1, 1, 0, s>>>(sc);
  GGM_CUDA_TRY(cudaGetLastError());
  count_launches(2);
  return GGM_OK;
}

// G += Cᵀ C for the samples [r0, r1) of a CSR unfolding (d rows, values sval + z, zeros z),
// operand written straight from the CSR (no dense chunk).  rows_side: samples = rows, the
// Gram side = the dim = m columns; else samples = columns, the Gram side = the dim = d rows.
ggm_status gram_tc_accumulate_csr(const int64_t* rp, const int32_t* col, const double* sval,
                                  int64_t d, bool rows_side, int64_t r0, int64_t r1, int64_t dim,
                                  double* G, void* ws, cudaStream_t s) {
  using namespace gt;
  const int64_t rows = r1 - r0;
  if (rows <= 0) return GGM_OK;
  const int natoms = (int)((rows + 63) / 64);
  int nblk = (int)((dim + 127) / 128);
  nblk += nblk & 1;
  const int sms = num_sms();
  const Scal* sc = static_cast<const Scal*>(ws);
  uint8_t* op = tc_op(ws);
  GGM_CUDA_TRY(cudaMemsetAsync(op, 0, (size_t)nblk * natoms * 2 * kAtomBytes, s));
  const int64_t nr = rows_side ? rows : d;
  csr_scatter<<<(int)std::max<int64_t>(1, std::min<int64_t>((nr * 32 + 255) / 256, sms * 16)), 256, 0,
                s>>>(rp, col, sval, rows_side, r0, r1, d, natoms, sc, op);
  GGM_CUDA_TRY(cudaGetLastError());
  count_launches(3);
  return tc_run(rows, dim, G, ws, s);
}

// After the chunk loop: the exact rank-one terms of A = S + z 1ᵀ (fp64).  scratch: dim + 1
// doubles.  ncols: the number of CSR columns (samples) when !rows_side.
ggm_status gram_tc_csr_rank1(const int64_t* rp, const int32_t* col, const double* sval,
                             const double* z, int64_t d, bool rows_side, int64_t dim,
                             int64_t ncols, double* G, double* scratch, cudaStream_t s) {
  using namespace gt;
  const int sms = num_sms();
  GGM_CUDA_TRY(cudaMemsetAsync(scratch, 0, sizeof(double) * (dim + 1), s));
  rank1_vec<<<(int)std::max<int64_t>(1, std::min<int64_t>((d * 32 + 255) / 256, sms * 16)), 256, 0,
              s>>>(rp, col, sval, z, d, rows_side, scratch, scratch + dim);
  rank1_apply<<<(int)std::max<int64_t>(1, std::min<int64_t>((dim * dim + 255) / 256, sms * 16)), 256, 0,
                s>>>(G, dim, scratch, z, scratch + dim, rows_side, (double)ncols);
  GGM_CUDA_TRY(cudaGetLastError());
  count_launches(2);
  return GGM_OK;
}

}  // namespace ggm
