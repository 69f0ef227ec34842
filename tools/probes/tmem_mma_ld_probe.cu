// Do TMEM loads overlap tcgen05.mma into another TMEM buffer?  (sm_100a, 1 CTA per SM)
// warp 0 (one thread) issues NM back-to-back kind::f16 M=128 N=256 K=16 MMAs into columns
// 256..511; warps 4..19 (4 per lane quadrant, as the BK2 epilogue) each read 32 lanes x 64
// columns of columns 0..255 NL times (tcgen05.ld.32x32b.x64 + wait::ld).  Modes: MMA only,
// loads only, both concurrently; prints cycles of each side.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/tmem_mma_ld_probe tools/probes/tmem_mma_ld_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_19892_b200/csrc/ptx_sm100.cuh"
using namespace ggm;
__global__ void __launch_bounds__(640, 1) probe(int mode, int NM, int NL, unsigned long long* out,
                                                uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u * (i & 1);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  unsigned long long c_mma = 0, c_ld = 0;
  if (warp == 0) {
    if (mode != 1 && lane == 0) {
      const uint64_t dA = sw128_desc(smem_u32(smem));
      const uint64_t dB = sw128_desc(smem_u32(smem + 16384));
      constexpr uint32_t idesc = idesc_f16_f32(128, 256);
      const long long c0 = clock64();
      for (int i = 0; i < NM; ++i) mma_f16_ss(t + 256, dA + 2 * (i & 3), dB + 2 * (i & 3), idesc, i > 0);
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      c_mma = clock64() - c0;
      out[blockIdx.x * 2 + 0] = c_mma;
    }
  } else if (warp >= 4) {
    const int q = warp & 3, part = (warp - 4) >> 2;
    const uint32_t A = t + ((uint32_t)(32 * q) << 16) + (uint32_t)(64 * part);
    uint32_t acc = 0;
    uint32_t v[64];
    if (mode != 0) {
      const long long c0 = clock64();
      for (int it = 0; it < NL; ++it) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31]),"=r"(v[32]),"=r"(v[33]),"=r"(v[34]),"=r"(v[35]),"=r"(v[36]),"=r"(v[37]),"=r"(v[38]),"=r"(v[39]),"=r"(v[40]),"=r"(v[41]),"=r"(v[42]),"=r"(v[43]),"=r"(v[44]),"=r"(v[45]),"=r"(v[46]),"=r"(v[47]),"=r"(v[48]),"=r"(v[49]),"=r"(v[50]),"=r"(v[51]),"=r"(v[52]),"=r"(v[53]),"=r"(v[54]),"=r"(v[55]),"=r"(v[56]),"=r"(v[57]),"=r"(v[58]),"=r"(v[59]),"=r"(v[60]),"=r"(v[61]),"=r"(v[62]),"=r"(v[63]) : "r"(A));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 64; ++i) acc ^= v[i];
      }
      c_ld = clock64() - c0;
      if (lane == 0 && warp == 4) out[blockIdx.x * 2 + 1] = c_ld;
    }
    sink[blockIdx.x * 640 + threadIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512) : "memory");
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 48 * 1024 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* out; uint32_t* sink;
  cudaMalloc(&out, sizeof(unsigned long long) * sms * 2);
  cudaMalloc(&sink, sizeof(uint32_t) * sms * 640);
  const int NM = 7 * 4000, NL = 4000;   // 4000 tiles of 7 MMAs; 4000 tile loads
  const char* names[3] = {"MMA only", "loads only", "MMA + loads concurrently"};
  for (int rep = 0; rep < 2; ++rep)
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(out, 0, sizeof(unsigned long long) * sms * 2);
    probe<<<sms, 640, smem>>>(mode, NM, NL, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-26s err=%s  MMA side %.1f cycles per 7 MMAs (%.1f per MMA) | load side %.1f cycles per 128 KB tile\n",
           names[mode], cudaGetErrorString(e), h[0] / 4000.0, h[0] / (double)NM, h[1] / 4000.0);
  }
  return 0;
}
