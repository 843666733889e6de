// C-ABI bookkeeping: error reporting and library identification.
#include "common.cuh"
#include <cstdarg>
#include <cstdlib>

namespace spb {
static thread_local char g_err[512] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SPB_PDL");
    return e == nullptr || atoi(e) != 0;
  }();
  return on;
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

extern "C" {
// Strided host->device copy of one time chunk of a [B][T][k] uint8 spike tensor held in
// pinned host memory into a [B][Tc][k] device chunk buffer (cudaMemcpy2DAsync): the
// streaming input path that keeps device memory independent of T.
int spb_copy_chunk_h2d(void* dst, long long dst_pitch, const void* src, long long src_pitch,
                       long long row_bytes, int rows, cudaStream_t stream) {
  SPB_CHECK_ARG(dst && src && rows >= 0 && row_bytes >= 0 && dst_pitch >= row_bytes &&
                    src_pitch >= row_bytes,
                "spb_copy_chunk_h2d: bad args");
  if (rows == 0 || row_bytes == 0) return 0;
  cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dst_pitch, src, (size_t)src_pitch,
                                    (size_t)row_bytes, (size_t)rows, cudaMemcpyHostToDevice,
                                    stream);
  if (e != cudaSuccess) {
    spb::set_error("spb_copy_chunk_h2d: %s", cudaGetErrorString(e));
    return 3;
  }
  return 0;
}
}
