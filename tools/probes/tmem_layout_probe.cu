// TMEM load-shape layout probe (sm_100a): every TMEM cell (lane L, column c) is written with
// L*1000 + c by 32x32b stores, then read back with the 16x256b / 16x64b / 16x128b shapes;
// each thread prints which (lane, column) cells its registers received.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probes/tmem_layout_probe tools/probes/tmem_layout_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(int* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(64) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tbase;
  for (int half = 0; half < 2; ++half) {
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) r[j] = (uint32_t)((32 * warp + lane) * 1000 + 32 * half + j);
    const uint32_t a = t + ((uint32_t)(32 * warp) << 16) + 32 * half;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) {  // quadrant 1: lanes 32..63
    const uint32_t a0 = t + ((uint32_t)32 << 16);
    uint32_t v[16];
    // 16x256b.x1: 4 registers
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(a0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; ++j) out[(0 * 32 + lane) * 16 + j] = (int)v[j];
    // 16x256b.x4: 16 registers
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(a0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) out[(1 * 32 + lane) * 16 + j] = (int)v[j];
    // 16x256b.x1 at lane offset +16 (upper half of the quadrant)
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(a0 + ((uint32_t)16 << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; ++j) out[(2 * 32 + lane) * 16 + j] = (int)v[j];
    // 16x64b.x4: 4 registers
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(a0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; ++j) out[(3 * 32 + lane) * 16 + j] = (int)v[j];
    // 16x128b.x2: 4 registers
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(a0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; ++j) out[(4 * 32 + lane) * 16 + j] = (int)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(64) : "memory");
}

int main() {
  int* d;
  cudaMalloc(&d, 5 * 32 * 16 * sizeof(int));
  cudaMemset(d, 0xff, 5 * 32 * 16 * sizeof(int));
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\n", cudaGetErrorString(e));
  int h[5 * 32 * 16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[5] = {"16x256b.x1", "16x256b.x4", "16x256b.x1@+16", "16x64b.x4", "16x128b.x2"};
  const int nr[5] = {4, 16, 4, 4, 4};
  for (int s = 0; s < 5; ++s) {
    printf("== %s (lane,col)\n", names[s]);
    for (int l = 0; l < 32; ++l) {
      printf("t%2d:", l);
      for (int j = 0; j < nr[s]; ++j) {
        const int x = h[(s * 32 + l) * 16 + j];
        printf(" (%d,%d)", x / 1000, x % 1000);
      }
      printf("\n");
    }
  }
  return 0;
}
