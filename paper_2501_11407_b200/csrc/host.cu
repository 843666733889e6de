// Host-side staging helpers of the drop-in (no device code).
//
// spb_host_pack_bits: uint8 spike counts [rows][k] -> bit-packed rows [rows][ceil(k/8)]
// (np.packbits(x, axis=-1, bitorder="little") layout), written straight into the pinned
// staging buffer the host-to-device copy reads.  The reference's inputs are 0/1 spikes
// (datasets.py:65-67, bench.py:63-67); the drop-in then moves k/8 instead of k bytes per
// sample-step over PCIe and K2 takes its binary recombination path.  Pooled counts > 1
// are reported (return 1) and the caller stages the bytes instead.
//
// One pass over the input, memory-bound: with AVX2 (checked at run time) 32 counts are
// checked against 0xFE.. and turned into 4 output bytes by one shift + movemask (byte i's
// bit 0 moved to its sign bit; movemask bit i = byte i, i.e. little bit order); the scalar
// path folds 8 counts into one byte with a multiply (byte i of the word lands on bit
// 56 + i of the product, the other partial products on distinct bits below 56, so nothing
// carries into the top byte).  Called from several host threads on disjoint row ranges
// (ctypes releases the GIL).
#include "common.cuh"
#include <cstring>
#include <immintrin.h>

namespace {

// bytes [0, nb) of a row: 8 counts -> 1 output byte; returns the OR of the inputs
inline uint64_t pack_scalar(const uint8_t* xr, uint8_t* orow, int b0, int full) {
  uint64_t bad = 0;
  for (int b = b0; b < full; ++b) {
    uint64_t v;
    memcpy(&v, xr + 8 * b, 8);
    bad |= v;
    orow[b] = (uint8_t)((v * 0x0102040810204080ull) >> 56);
  }
  return bad;
}

inline uint64_t pack_tail(const uint8_t* xr, uint8_t* orow, int full, int rem) {
  uint64_t bad = 0;
  if (rem) {
    uint8_t o = 0;
    for (int j = 0; j < rem; ++j) {
      const uint8_t c = xr[8 * full + j];
      bad |= c;
      o |= (uint8_t)((c & 1u) << j);
    }
    orow[full] = o;
  }
  return bad;
}

int pack_rows_scalar(const uint8_t* x, long long rows, int k, uint8_t* out) {
  const int kb = (k + 7) / 8, full = k / 8, rem = k % 8;
  for (long long r = 0; r < rows; ++r) {
    const uint8_t* xr = x + r * (long long)k;
    uint8_t* orow = out + r * (long long)kb;
    const uint64_t bad = pack_scalar(xr, orow, 0, full) | pack_tail(xr, orow, full, rem);
    if (bad & 0xFEFEFEFEFEFEFEFEull) return 1;  // a count > 1: not a binary spike tensor
  }
  return 0;
}

__attribute__((target("avx2"))) int pack_rows_avx2(const uint8_t* x, long long rows, int k,
                                                   uint8_t* out) {
  const int kb = (k + 7) / 8, full = k / 8, rem = k % 8;
  const int nv = k / 32;  // 32-count vectors per row
  const __m256i hi7 = _mm256_set1_epi8((char)0xFE);
  for (long long r = 0; r < rows; ++r) {
    const uint8_t* xr = x + r * (long long)k;
    uint8_t* orow = out + r * (long long)kb;
    __m256i acc = _mm256_setzero_si256();
    for (int v = 0; v < nv; ++v) {
      const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(xr + 32 * v));
      acc = _mm256_or_si256(acc, c);
      const uint32_t m = (uint32_t)_mm256_movemask_epi8(_mm256_slli_epi16(c, 7));
      memcpy(orow + 4 * v, &m, 4);
    }
    uint64_t bad = pack_scalar(xr, orow, 4 * nv, full) | pack_tail(xr, orow, full, rem);
    if (!_mm256_testz_si256(acc, hi7) || (bad & 0xFEFEFEFEFEFEFEFEull)) return 1;
  }
  return 0;
}

}  // namespace

extern "C" int spb_host_pack_bits(const uint8_t* x, long long rows, int k, uint8_t* out) {
  SPB_CHECK_ARG(x && out && rows >= 0 && k > 0, "spb_host_pack_bits: bad args");
  static const bool avx2 = __builtin_cpu_supports("avx2");
  return avx2 ? pack_rows_avx2(x, rows, k, out) : pack_rows_scalar(x, rows, k, out);
}
