// Weight-digit formats of the exact INT8 tensor-core projection (K2).
//
//   W[i][j] = sum_{p<P} q_p[i][j] * 2^(RB*(P-1-p)) * 2^(s_i - F) + r,   q_p int8,
//   s_i = exponent of max_j |W[i][j]|  (|W[i][j]| < 2^s_i)
//
//   P = 6, RB = 8, F = 46: balanced radix-256 digits (f32 weights) -- every weight
//          within 2^-23 of its row maximum is exact (24-bit mantissa), smaller ones are
//          rounded to 2^(s-46) (|r| <= 2^(s-47));
//   P = 7, RB = 7, F = 48: radix-128 digits (f32, former default);
//   P = 8, RB = 7, F = 55: radix-128 digits (f64 weights).
// A digit sum S_p = sum_j x_j q_p[i][j] is exact in int32; the current is recombined from
// g0 = digits 0-2 and g1 = digits 3..P-1 (both exact in int64 and in double) with ONE
// rounding:  I = fma(g0, 2^(s-F+RB*(P-3)), g1 * 2^(s-F)).  With binary spikes all digits
// fit one int64 g = g0 * 2^(RB*(P-3)) + g1 and I = (double)g * 2^(s-F) (same bits).
//
// Row order of the sliced weights wq [P][n_pad32][Kpad]: inside every group of 16 neurons
// the rows are permuted, storage slot c holding neuron perm16(c).  K2's MMA puts slot c of
// a tile in TMEM column c, and a tcgen05.ld.16x256b gives thread q (of a lane quad) the
// columns 2q, 2q+1, 8+2q, 9+2q -- under this order the four consecutive neurons 4q..4q+3,
// so each thread stores 32 contiguous bytes of a current row without any lane shuffles.
#pragma once
#include "common.cuh"

namespace spb {

__host__ __device__ constexpr int perm16(int c) {  // storage slot -> neuron (mod 16)
  return ((c & 7) >> 1) * 4 + (c >> 3) * 2 + (c & 1);
}
__host__ __device__ constexpr int pinv16(int j) {  // neuron -> storage slot (mod 16)
  return ((j & 3) >> 1) * 8 + (j >> 2) * 2 + (j & 1);
}
__host__ __device__ constexpr int wq_slot(int i) { return (i & ~15) | pinv16(i & 15); }
static_assert(perm16(pinv16(5)) == 5 && perm16(pinv16(14)) == 14 && pinv16(perm16(9)) == 9,
              "perm16 / pinv16 are inverse");

template <int P>
struct Digits {
  static_assert(P == 6 || P == 7 || P == 8, "digit count");
  static constexpr int RB = (P == 6) ? 8 : 7;
  static constexpr int F = (P == 6) ? 46 : 6 + 7 * (P - 1);
  static constexpr int HI = RB * (P - 3);          // weight of g0 relative to g1
  // single-int64 recombination is exact for binary spikes when |g| < 2^63
  static constexpr bool kSingleOk = (P <= 7);
};

__device__ __forceinline__ double digits_pow2(int e) {  // 2^e for -1022 <= e <= 1023
  return __longlong_as_double((long long)(e + 1023) << 52);
}

template <int P>
__device__ __forceinline__ long long digits_g0(int s0, int s1, int s2) {
  constexpr int RB = Digits<P>::RB;
  return ((((long long)s0 << RB) + s1) << RB) + s2;
}

// the exactly-rounded current from the two digit groups
template <int P, bool BIN>
__device__ __forceinline__ double digits_current(long long g0, long long g1, int se) {
  using D = Digits<P>;
  if constexpr (BIN && D::kSingleOk) {
    const long long g = (g0 << D::HI) + g1;
    return (double)g * digits_pow2(se - D::F);
  } else {
    return fma((double)g0, digits_pow2(se - D::F + D::HI), (double)g1 * digits_pow2(se - D::F));
  }
}

// the same with the per-neuron scale 2^(s - F) precomputed (one per neuron tile)
template <int P, bool BIN>
__device__ __forceinline__ double digits_current_scaled(long long g0, long long g1, double scale) {
  using D = Digits<P>;
  if constexpr (BIN && D::kSingleOk) {
    const long long g = (g0 << D::HI) + g1;
    return (double)g * scale;
  } else {
    return fma((double)g0, scale * (double)(1LL << D::HI), (double)g1 * scale);
  }
}

}  // namespace spb
