// Microbenchmark: tcgen05.ld throughput per SM for several shapes / warp counts.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SHAPE>
__global__ void kern(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t base = slot + (((warp & 3) * 32) << 16) + ((warp >> 2) * 128);
  float acc = 0.f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[128];
    if (SHAPE == 0) {  // x32, wait each
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(base + c * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 32; ++e) acc += __uint_as_float(r[e]);
      }
    } else if (SHAPE == 1) {  // x32 x4, single wait
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[c*32+0]),"=r"(r[c*32+1]),"=r"(r[c*32+2]),"=r"(r[c*32+3]),"=r"(r[c*32+4]),"=r"(r[c*32+5]),"=r"(r[c*32+6]),"=r"(r[c*32+7]),"=r"(r[c*32+8]),"=r"(r[c*32+9]),"=r"(r[c*32+10]),"=r"(r[c*32+11]),"=r"(r[c*32+12]),"=r"(r[c*32+13]),"=r"(r[c*32+14]),"=r"(r[c*32+15]),"=r"(r[c*32+16]),"=r"(r[c*32+17]),"=r"(r[c*32+18]),"=r"(r[c*32+19]),"=r"(r[c*32+20]),"=r"(r[c*32+21]),"=r"(r[c*32+22]),"=r"(r[c*32+23]),"=r"(r[c*32+24]),"=r"(r[c*32+25]),"=r"(r[c*32+26]),"=r"(r[c*32+27]),"=r"(r[c*32+28]),"=r"(r[c*32+29]),"=r"(r[c*32+30]),"=r"(r[c*32+31]) : "r"(base + c * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int e = 0; e < 128; ++e) acc += __uint_as_float(r[e]);
    } else {  // 16x256b.x8: 32 regs, lanes 16 x 256 bit
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(base + c * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 32; ++e) acc += __uint_as_float(r[e]);
      }
    }
  }
  unsigned long long t1 = clock64();
  if (acc == 1.2345f) sink[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot));
}

int main() {
  unsigned long long* d; float* s;
  cudaMalloc(&d, 8 * 148); cudaMalloc(&s, 4);
  const int iters = 2000;
  const char* names[3] = {"32x32b.x32 wait-each", "32x32b.x32 x4 one wait", "16x256b.x8 wait-each"};
  for (int shape = 0; shape < 3; ++shape)
    for (int warps = 4; warps <= 16; warps *= 2) {
      if (shape == 0) kern<0><<<148, warps * 32>>>(iters, d, s);
      if (shape == 1) kern<1><<<148, warps * 32>>>(iters, d, s);
      if (shape == 2) kern<2><<<148, warps * 32>>>(iters, d, s);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      // bytes per SM: warps * iters * 4 loads * (32 lanes * 32 regs * 4 B)
      double bytes = (double)warps * iters * 4 * 32 * 32 * 4;
      printf("%-26s warps=%2d: %8.1f B/clk/SM  (%s)\n", names[shape], warps, bytes / h, cudaGetErrorString(e));
    }
  return 0;
}
