// Probe: the TMEM layout of a tcgen05.mma kind::f16 accumulator with D = f16 (one CTA,
// M = 128, N = 256, K = 16).  A[r][k] = (k == 0), B[c][k] = (k == 0) * c, so D[r][c] = c.
// The 32-bit TMEM columns 0..255 of lane r are dumped raw: packed layout <=> column j holds
// the f16 values (2j, 2j+1); unpacked <=> column j holds f16(j) in its low half.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_f16_probe tmem_f16_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "../../paper_2407_19892_b200/csrc/ptx_sm100.cuh"
using namespace ggm;

__global__ void probe(uint32_t* out, int f16acc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* A = smem;            // 128 rows x 128 B (one SW128 atom)
  uint8_t* B = smem + 16384;    // 256 rows x 128 B
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  for (int i = t; i < (16384 + 32768) / 2; i += blockDim.x) reinterpret_cast<__half*>(smem)[i] = __float2half(0.f);
  __syncthreads();
  // element (row r, k) of a SW128 K-major atom: chunk (k/8) ^ (r & 7), offset (k%8)*2
  for (int r = t; r < 128; r += blockDim.x)
    *reinterpret_cast<__half*>(A + r * 128 + (((0) ^ (r & 7)) << 4)) = __float2half(1.f);
  for (int c = t; c < 256; c += blockDim.x)
    *reinterpret_cast<__half*>(B + c * 128 + (((0) ^ (c & 7)) << 4)) = __float2half((float)c);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (t < 32) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (t == 0) {
    uint32_t idesc = idesc_f16_f32(128, 256);
    if (f16acc) idesc &= ~(3u << 4);  // D format 0 = f16
    mma_f16_ss(tb, sw128_desc(smem_u32(A)), sw128_desc(smem_u32(B)), idesc, 0u);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int q = t >> 5, lane = t & 31;
  for (int c = 0; c < 8; ++c) {
    uint32_t v[32];
    tmem_ld32_nowait(tb + ((uint32_t)(q * 32) << 16) + c * 32, v);
    tmem_wait_ld(v);
    for (int e = 0; e < 32; ++e) out[(q * 32 + lane) * 256 + c * 32 + e] = v[e];
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

int main() {
  uint32_t* d; cudaMalloc(&d, 128 * 256 * 4);
  uint32_t* h = (uint32_t*)malloc(128 * 256 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 52000);
  for (int f16 = 0; f16 < 2; ++f16) {
    cudaMemset(d, 0, 128 * 256 * 4);
    probe<<<1, 128, 49152 + 2048>>>(d, f16);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 128 * 256 * 4, cudaMemcpyDeviceToHost);
    printf("D=%s err=%s\n", f16 ? "f16" : "f32", cudaGetErrorString(e));
    for (int r : {0, 5, 127}) {
      printf(" lane %3d:", r);
      for (int j : {0, 1, 2, 3, 64, 127, 128, 255}) {
        uint32_t x = h[r * 256 + j];
        __half lo = __ushort_as_half((unsigned short)(x & 0xffff)), hi = __ushort_as_half((unsigned short)(x >> 16));
        float xf; memcpy(&xf, &x, 4);
        printf(" [%d]=%08x(f32 %.1f | f16 lo %.1f hi %.1f)", j, x, xf, __half2float(lo), __half2float(hi));
      }
      printf("\n");
    }
  }
  return 0;
}
