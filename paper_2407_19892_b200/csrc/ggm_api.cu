// ggm_api.cu — status/error plumbing, version, device query and timing for libggm.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "ggm_internal.h"

namespace ggm {

static thread_local char g_last_error[1024] = "";
static thread_local bool g_timing = false;
static thread_local float g_timing_ms[3] = {0.f, 0.f, 0.f};
static thread_local int g_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

ggm_status fail(ggm_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return st;
}

int num_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 148;
  return sms > 0 ? sms : 148;
}

bool timing_enabled() { return g_timing; }
void reset_launches() { g_launches = 0; }
void count_launches(int n) { g_launches += n; }
void record_timing(int slot, float ms) {
  if (slot >= 0 && slot < 3) g_timing_ms[slot] = ms;
}

}  // namespace ggm

extern "C" {

const char* ggm_last_error(void) { return ggm::g_last_error; }

int ggm_version(void) { return 10000; /* 1.0.0 */ }

int ggm_device_supported(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (major == 10 && minor == 0) ? 1 : 0;
}

void ggm_set_timing(int enabled) { ggm::g_timing = enabled != 0; }

int ggm_last_launches(void) { return ggm::g_launches; }

void ggm_last_timing(float ms[3]) {
  for (int i = 0; i < 3; ++i) ms[i] = ggm::g_timing_ms[i];
}

}  // extern "C"
