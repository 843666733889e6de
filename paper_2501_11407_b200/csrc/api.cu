// C-ABI bookkeeping: error reporting and library identification.
#include "common.cuh"
#include <cstdarg>

namespace spb {
static thread_local char g_err[512] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace spb

extern "C" {
const char* spb_last_error(void) { return spb::g_err; }
int spb_version(void) { return 1; }
int spb_device_sm(void) {
  int dev = 0, maj = 0, min = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev);
  return maj * 10 + min;
}
}
