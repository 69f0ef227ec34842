// TMEM load throughput by shape (sm_100a): 16 warps per CTA (4 per lane quadrant), one CTA
// per SM, each warp repeatedly reads its 32 lanes x 64 columns (8 KB) of a 256-column buffer
// and waits (tcgen05.wait::ld), as the candidate epilogue does per tile.  Prints cycles per
// iteration and bytes/clk/SM for each shape.  tools/probes/README: see DESIGN.md BK2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/tmem_ldbw_probe tools/probes/tmem_ldbw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tbase;
  const int q = warp & 3, part = warp >> 2;
  const uint32_t a0 = t + ((uint32_t)(32 * q) << 16) + (uint32_t)(64 * part);
  const uint32_t a16 = a0 + (16u << 16);
  uint32_t acc = 0;
  uint32_t v[64];
  __syncthreads();
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t off = (uint32_t)((it & 1) * 256);  // alternate the two buffers
    const uint32_t A = a0 + off, A16 = a16 + off;
    if (MODE == 0) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31]),"=r"(v[32]),"=r"(v[33]),"=r"(v[34]),"=r"(v[35]),"=r"(v[36]),"=r"(v[37]),"=r"(v[38]),"=r"(v[39]),"=r"(v[40]),"=r"(v[41]),"=r"(v[42]),"=r"(v[43]),"=r"(v[44]),"=r"(v[45]),"=r"(v[46]),"=r"(v[47]),"=r"(v[48]),"=r"(v[49]),"=r"(v[50]),"=r"(v[51]),"=r"(v[52]),"=r"(v[53]),"=r"(v[54]),"=r"(v[55]),"=r"(v[56]),"=r"(v[57]),"=r"(v[58]),"=r"(v[59]),"=r"(v[60]),"=r"(v[61]),"=r"(v[62]),"=r"(v[63]) : "r"(A));
    } else if (MODE == 1) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31]) : "r"(A));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : "=r"((v+32)[0]),"=r"((v+32)[1]),"=r"((v+32)[2]),"=r"((v+32)[3]),"=r"((v+32)[4]),"=r"((v+32)[5]),"=r"((v+32)[6]),"=r"((v+32)[7]),"=r"((v+32)[8]),"=r"((v+32)[9]),"=r"((v+32)[10]),"=r"((v+32)[11]),"=r"((v+32)[12]),"=r"((v+32)[13]),"=r"((v+32)[14]),"=r"((v+32)[15]),"=r"((v+32)[16]),"=r"((v+32)[17]),"=r"((v+32)[18]),"=r"((v+32)[19]),"=r"((v+32)[20]),"=r"((v+32)[21]),"=r"((v+32)[22]),"=r"((v+32)[23]),"=r"((v+32)[24]),"=r"((v+32)[25]),"=r"((v+32)[26]),"=r"((v+32)[27]),"=r"((v+32)[28]),"=r"((v+32)[29]),"=r"((v+32)[30]),"=r"((v+32)[31]) : "r"(A + 32));
    } else if (MODE == 2) {
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31]) : "r"(A));
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : "=r"((v+32)[0]),"=r"((v+32)[1]),"=r"((v+32)[2]),"=r"((v+32)[3]),"=r"((v+32)[4]),"=r"((v+32)[5]),"=r"((v+32)[6]),"=r"((v+32)[7]),"=r"((v+32)[8]),"=r"((v+32)[9]),"=r"((v+32)[10]),"=r"((v+32)[11]),"=r"((v+32)[12]),"=r"((v+32)[13]),"=r"((v+32)[14]),"=r"((v+32)[15]),"=r"((v+32)[16]),"=r"((v+32)[17]),"=r"((v+32)[18]),"=r"((v+32)[19]),"=r"((v+32)[20]),"=r"((v+32)[21]),"=r"((v+32)[22]),"=r"((v+32)[23]),"=r"((v+32)[24]),"=r"((v+32)[25]),"=r"((v+32)[26]),"=r"((v+32)[27]),"=r"((v+32)[28]),"=r"((v+32)[29]),"=r"((v+32)[30]),"=r"((v+32)[31]) : "r"(A16));
    } else if (MODE == 3) {
      asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31]) : "r"(A));
      asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : "=r"((v+32)[0]),"=r"((v+32)[1]),"=r"((v+32)[2]),"=r"((v+32)[3]),"=r"((v+32)[4]),"=r"((v+32)[5]),"=r"((v+32)[6]),"=r"((v+32)[7]),"=r"((v+32)[8]),"=r"((v+32)[9]),"=r"((v+32)[10]),"=r"((v+32)[11]),"=r"((v+32)[12]),"=r"((v+32)[13]),"=r"((v+32)[14]),"=r"((v+32)[15]),"=r"((v+32)[16]),"=r"((v+32)[17]),"=r"((v+32)[18]),"=r"((v+32)[19]),"=r"((v+32)[20]),"=r"((v+32)[21]),"=r"((v+32)[22]),"=r"((v+32)[23]),"=r"((v+32)[24]),"=r"((v+32)[25]),"=r"((v+32)[26]),"=r"((v+32)[27]),"=r"((v+32)[28]),"=r"((v+32)[29]),"=r"((v+32)[30]),"=r"((v+32)[31]) : "r"(A16));
    } else {
      asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31]) : "r"(A));
      asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : "=r"((v+32)[0]),"=r"((v+32)[1]),"=r"((v+32)[2]),"=r"((v+32)[3]),"=r"((v+32)[4]),"=r"((v+32)[5]),"=r"((v+32)[6]),"=r"((v+32)[7]),"=r"((v+32)[8]),"=r"((v+32)[9]),"=r"((v+32)[10]),"=r"((v+32)[11]),"=r"((v+32)[12]),"=r"((v+32)[13]),"=r"((v+32)[14]),"=r"((v+32)[15]),"=r"((v+32)[16]),"=r"((v+32)[17]),"=r"((v+32)[18]),"=r"((v+32)[19]),"=r"((v+32)[20]),"=r"((v+32)[21]),"=r"((v+32)[22]),"=r"((v+32)[23]),"=r"((v+32)[24]),"=r"((v+32)[25]),"=r"((v+32)[26]),"=r"((v+32)[27]),"=r"((v+32)[28]),"=r"((v+32)[29]),"=r"((v+32)[30]),"=r"((v+32)[31]) : "r"(A16));
    }
    wait_ld();
#pragma unroll
    for (int i = 0; i < 64; ++i) acc ^= v[i];
  }
  const long long c1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 16 + warp] = (unsigned long long)(c1 - c0);
  sink[blockIdx.x * 512 + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512) : "memory");
}
template <int MODE>
void run(const char* name, int sms) {
  const int iters = 20000;
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms * 16);
  cudaMalloc(&sink, sizeof(uint32_t) * sms * 512);
  probe<MODE><<<sms, 512>>>(100, cyc, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE><<<sms, 512>>>(iters, cyc, sink);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[16];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 16; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cpi = (double)mx / iters;
  printf("%-28s err=%s  cycles/iter %.1f  bytes/clk/SM %.1f  (16 warps x 8 KB per iter)  %.3f ms\n",
         name, cudaGetErrorString(err), cpi, 16.0 * 8192 / cpi, ms);
  cudaFree(cyc); cudaFree(sink);
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("32x32b.x64 (1 instr)", sms);
  run<1>("32x32b.x32 x2", sms);
  run<2>("16x256b.x8 x2 (lanes 0/16)", sms);
  run<3>("16x128b.x16 x2", sms);
  run<4>("16x64b.x32 x2", sms);
  run<0>("32x32b.x64 (1 CTA)", 1);
  run<2>("16x256b.x8 x2 (1 CTA)", 1);
  return 0;
}
