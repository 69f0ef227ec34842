// ggm_internal.h — host-side helpers shared by the libggm translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/ggm.h"

namespace ggm {

void set_error(const char* fmt, ...);
ggm_status fail(ggm_status st, const char* fmt, ...);
int num_sms();
bool timing_enabled();
void record_timing(int slot, float ms);
void reset_launches();
void count_launches(int n);

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// gram_tc.cu: G (dim x dim fp64, row-major upper = column-major lower) += Cᵀ C on the
// tensor cores (fp32-accurate 3 x fp16 split); C = rows samples x dim, element (c, g) at
// C[c·rs + g·cs].
size_t gram_tc_workspace(int64_t max_rows, int64_t dim);
ggm_status gram_tc_accumulate(const double* C, int64_t rows, int64_t dim, int64_t rs, int64_t cs,
                              double* G, void* ws, cudaStream_t s);
ggm_status gram_tc_csr_scale(const int64_t* rp, const double* sval, int64_t nrows, void* ws,
                             cudaStream_t s);
ggm_status gram_tc_accumulate_csr(const int64_t* rp, const int32_t* col, const double* sval,
                                  int64_t d, bool rows_side, int64_t r0, int64_t r1, int64_t dim,
                                  double* G, void* ws, cudaStream_t s);
ggm_status gram_tc_csr_rank1(const int64_t* rp, const int32_t* col, const double* sval,
                             const double* z, int64_t d, bool rows_side, int64_t dim,
                             int64_t ncols, double* G, double* scratch, cudaStream_t s);

// Bump allocator over a caller-provided workspace (256-byte aligned slices).
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
  size_t used() const { return align_up(off, 256); }
};

}  // namespace ggm

// Device-side invariant checks, compiled in only for the checked build
// (tools/build_variant.sh checked -DGGM_CHECKED; compute-sanitizer is not available on the GPU
// pool): a failed check prints and traps, so the call returns GGM_ERR_CUDA.
#ifdef GGM_CHECKED
#define GGM_DCHECK(cond)                                                                \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("GGM_DCHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);            \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define GGM_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

#define GGM_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return ::ggm::fail(GGM_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,                  \
                         cudaGetErrorString(_e), __FILE__, __LINE__);                   \
  } while (0)
