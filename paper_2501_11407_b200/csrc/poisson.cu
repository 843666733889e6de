// On-device synthetic spike generation for throughput runs.
//
// The reference draws Bernoulli spike grids with numpy (`sample_events`,
// datasets.py:65-67: x[t, j] = U[0,1) < rate[label, j]) on the host; at B200 rates that
// host generation and its host->device copy would dominate a training step.  This kernel
// draws the same distribution on the device with a counter-based generator
// (Philox4x32-10, Salmon et al., SC'11), so any (sample, step, channel) is reproducible
// from (seed, counter) alone, in any order and chunking -- but the bits are NOT numpy's
// (parity runs keep the host generator, datasets.poisson_batch).  Output is the engine's
// bit-packed input format (numpy.packbits(..., bitorder="little") rows).
#include "common.cuh"

namespace spb {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = c.x * 0xD2511F53u, hi0 = __umulhi(c.x, 0xD2511F53u);
    const uint32_t lo1 = c.z * 0xCD9E8D57u, hi1 = __umulhi(c.z, 0xCD9E8D57u);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Thread = one output byte (8 channels) of one (sample, step): two Philox blocks, one
// 32-bit uniform per channel; spike iff u < rate * 2^32.
__global__ void poisson_bits_kernel(const float* __restrict__ rates, const long long* __restrict__ labels,
                                    int B, int T, int k, int t0, uint2 key, uint8_t* __restrict__ out,
                                    long long stride_b) {
  const int kb = (k + 7) >> 3;
  const long long total = (long long)B * T * kb;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int jb = (int)(idx % kb);
    const long long bt = idx / kb;
    const int t = (int)(bt % T), b = (int)(bt / T);
    const float* rrow = rates + labels[b] * (long long)k;
    const uint32_t tg = (uint32_t)(t0 + t);
    uint32_t bits = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint4 r = philox4x32_10(make_uint4((uint32_t)(jb * 2 + h), tg, (uint32_t)b, 0u), key);
      const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = jb * 8 + h * 4 + q;
        if (j < k) {
          const double thr = (double)rrow[j] * 4294967296.0;
          bits |= ((double)u[q] < thr ? 1u : 0u) << (h * 4 + q);
        }
      }
    }
    out[(long long)b * stride_b + (long long)t * kb + jb] = (uint8_t)bits;
  }
}

}  // namespace spb

using namespace spb;

extern "C" {

int spb_poisson_bits(const float* rates, const long long* labels, int B, int T, int k, int t0,
                     unsigned long long seed, uint8_t* out, long long stride_b,
                     cudaStream_t stream) {
  SPB_CHECK_ARG(rates && labels && out && B > 0 && T > 0 && k > 0 && t0 >= 0 &&
                    stride_b >= (long long)T * ((k + 7) / 8),
                "spb_poisson_bits: bad args");
  const long long total = (long long)B * T * ((k + 7) / 8);
  const int grid = (int)(total / 256 + 1 < 148LL * 32 ? total / 256 + 1 : 148LL * 32);
  poisson_bits_kernel<<<grid, 256, 0, stream>>>(
      rates, labels, B, T, k, t0, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)), out,
      stride_b);
  SPB_CHECK_LAUNCH("poisson_bits");
  return 0;
}

}  // extern "C"
