// K2: exact input projection I = W x_t on 5th-generation INT8 tensor cores (tcgen05).
//
// The reference computes the input current with a float matvec (`net.neuron.w @ x_t`,
// gradients.py:125) in f64.  Spike decisions must match it bit for bit (margins go
// down to ~1e-7), so the projection has to be exact to fp64 level.
// Inputs are spike counts (uint8), so we slice the weights instead of rounding them:
//
//   W[i][j] = sum_{p<P} q_p[i][j] * 2^(RB*(P-1-p)) * 2^(s_i - F) + r,   q_p int8,
//   s_i = exponent of max_j |W[i][j]|      (formats: csrc/digits.cuh)
//
// P = 6 balanced radix-256 digits (F = 46) for fp32 weights -- exact for every weight
// within 2^-23 of the row maximum -- and P = 8 radix-128 digits (F = 55) for fp64
// weights.  x (u8) * q_p (s8) is accumulated by tcgen05.mma.kind::i8 in int32 TMEM
// (exact: |acc| <= k*255*128 < 2^31), the slices are
// recombined in int64 (exact) and converted to fp64 once: the result is the (weight-
// truncated) exact sum rounded once, independent of summation order.
//
// Kernels:
//   spb_pack_spikes      x chunk [B][len][k] bytes or bits -> xq [B*Tc][Kpad] (TMA-able,
//                        zero padded; also the row source of K4)
//   spb_slice_weights    W [n][k] fp32/fp64  -> Wq [P][n_pad32][Kpad] int8, s [n] int32
//   spb_input_proj       persistent warp-specialised tcgen05 GEMM -> I [B*Tc][n] fp64
#include "tma.cuh"
#include "digits.cuh"
#include <algorithm>
#include <cstdlib>

// K2 producer warp: SPB_K2_ELECT=1 runs the spike-stage loop on the whole (converged) warp
// with expect_tx + TMA under elect.sync; 0 keeps it on lane 0 alone.
#ifndef SPB_K2_ELECT
#define SPB_K2_ELECT 1
#endif
#if SPB_K2_ELECT
#define SPB_K2_PRODUCER_LANES true
#define SPB_K2_LANE0 (lane == 0)
#else
#define SPB_K2_PRODUCER_LANES (lane == 0)
#define SPB_K2_LANE0 true
#endif

namespace spb {
namespace proj {

constexpr int BM = 128;       // (sample, step) rows per tile
constexpr int NT = 32;        // neurons per tile (per slice)
constexpr int BK = 128;       // bytes (= int8 elements) of K per stage: one 128B swizzle row
constexpr int STAGES = 4;
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr int EPI_WARPS = 8;  // 4 TMEM lane quarters x 2 halves of the 32 neurons
constexpr int TILE_A = BM * BK;

template <int P>
struct Cfg {
  static constexpr int N = P * NT;             // MMA N (224 or 256)
  static constexpr int TILE_B = N * BK;
  static constexpr int STAGE = TILE_A + TILE_B;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  // kind::i8: D s32 (c_format 2), A u8 (a_format 0), B s8 (b_format 1), both K-major
  static constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (1u << 10) |
                                    ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
};

__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// The 4 MMAs of one 128-byte K block (K = 32 bytes each) under ONE elect.sync: the
// descriptors of steps 1..3 are the step-0 descriptors + 2 (32 bytes in 16-byte units of
// the start-address field, SW128 K-major), formed inside the block.
__device__ __forceinline__ void mma_i8_x4(uint32_t tmem_d, uint64_t a, uint64_t b,
                                          uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a2, b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a3, b3, %3, 1;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc0));
}
// K-major SWIZZLE_64B operand (the 64-byte tail K block of the spikes): 8-row groups 512 B
// apart, swizzle mode 4
__device__ __forceinline__ uint64_t desc_k_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(512u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;
  return d;
}
// The 2 MMAs of the 64-byte tail K block under one elect.sync (A: SW64, B: SW128 rows).
__device__ __forceinline__ void mma_i8_x2(uint32_t tmem_d, uint64_t a, uint64_t b,
                                          uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, b1;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 b1, %2, 2;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, 1;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc0));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                   bar)
               : "memory");
}
// commit arriving on the barrier at this offset in every CTA of the cluster in mask
__device__ __forceinline__ void commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster"
               ".multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(bar),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, int32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, int32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ double pow2(int e) {  // 2^e for -1022 <= e <= 1023
  return __longlong_as_double((long long)(e + 1023) << 52);
}

// Epilogue of one 128-row x 32-neuron tile, split over 8 warps: TMEM lane quarter q and
// neuron half h (16 neurons).  Each thread pulls its row's P slice accumulators for its
// 16 neurons in two batches (slices 0-2, then 3..P-1, one tcgen05.wait each), recombines
// them exactly in int64 and writes 16 fp64 currents (128 contiguous bytes).
constexpr int NH = NT / 2;  // neurons per epilogue thread (16 epilogue warps measured slower)

// BIN (binary spikes, k <= 16384): every digit sum |S_p| < 2^21, so all P <= 7 digits
// recombine into ONE int64 g = sum_p S_p 2^(RB*(P-1-p)) (|g| < 2^63) and I = (double)g *
// 2^(s-F): one rounding of the exact sum, bitwise the value of the two-part path below,
// with half the fp64-pipe work.
// Output row of input row r0 + d (0 <= d < 32) with (b0, s0) = (r0 / rin, r0 % rin): the
// projection may read rin rows per sample (the chunk's live steps) and write rout rows per
// sample (the current buffer's KR); rin == rout is the identity.  A 32-row quarter tile
// crosses at most one sample boundary when rin >= 32.
// r / rin (r >= 0, a quotient below 2^22: the sample index) without an integer division:
// the float quotient is within one of the true one, corrected by one step either way
__device__ __forceinline__ int proj_row_div(int r, int rin) {
  int q = __float2int_rz(__fdividef((float)r, (float)rin));
  if (q * rin > r) --q;
  else if ((q + 1) * rin <= r) ++q;
  return q;
}
__device__ __forceinline__ long long proj_out_row(int b0, int s0, int d, int rin, int rout) {
  int s = s0 + d, b = b0;
  if (rin >= 32) {
    if (s >= rin) {
      s -= rin;
      ++b;
    }
  } else {
    const int q = s / rin;
    b += q;
    s -= q * rin;
  }
  return (long long)b * rout + s;
}

// SE: per-neuron exponents (int) or precomputed scales 2^(s-F) (double)
template <int P, bool BIN, typename SE = int>
__device__ __forceinline__ void proj_epilogue_tile(uint32_t tbase, const SE (&se)[NH],
                                                   double* __restrict__ out, int M, int n,
                                                   int rin, int rout, int row, int i0,
                                                   uint32_t tempty_bar, int lane,
                                                   int probe = 0) {
  const int rq = row - lane;  // this warp's quarter-tile base row
  const int b0 = proj_row_div(rq, rin), s0 = rq - b0 * rin;
  long long g0[NH], g1[NH];
  {
    int32_t r[3][NH];
#pragma unroll
    for (int p = 0; p < 3; ++p) tmem_ld16_nowait(tbase + p * NT, r[p]);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < NH; ++c) g0[c] = digits_g0<P>(r[0][c], r[1][c], r[2][c]);
  }
  {
    int32_t r[P - 3][NH];
#pragma unroll
    for (int p = 3; p < P; ++p) tmem_ld16_nowait(tbase + p * NT, r[p - 3]);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < NH; ++c) {
      long long v = r[0][c];
#pragma unroll
      for (int p = 1; p < P - 3; ++p) v = (v << Digits<P>::RB) + r[p][c];
      g1[c] = v;
    }
  }
  // the TMEM buffer is free once every epilogue warp has pulled its lanes
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  if (lane == 0) mbar_arrive(tempty_bar);
  // values of this thread's row in NEURON order: 16 doubles = 8 double2 chunks (TMEM
  // column c holds neuron perm16(c) of the 16-neuron group, digits.cuh)
  double2 ch[NH / 2];
#pragma unroll
  for (int c = 0; c < NH; c += 2) {
    double v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sl = pinv16(c + h);
      if constexpr (sizeof(SE) == sizeof(double))
        v[h] = digits_current_scaled<P, BIN>(g0[sl], g1[sl], se[c + h]);
      else
        v[h] = digits_current<P, BIN>(g0[sl], g1[sl], se[c + h]);
    }
    ch[c / 2] = make_double2(v[0], v[1]);
  }
  if (probe & 4) {  // profiling probe: no global stores
    if (ch[0].x == 1.2345e-300 && row < M) out[(long long)row * n + i0] = ch[0].y;
    return;
  }
  if ((n & 3) == 0) {
    // 4x4 transpose of 32-byte quads (4 neurons) inside each group of 4 lanes (2 xor-
    // butterfly stages): lane p of the group then holds quad p of the group's 4 rows and
    // each 256-bit store instruction writes 8 rows x 128 contiguous bytes (full lines) --
    // two thirds of the shuffles and half the store instructions of the 8x8 scheme below.
    const int p4 = lane & 3;
#pragma unroll
    for (int sh = 2; sh >= 1; sh >>= 1) {
      const bool up = (p4 & sh) != 0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        if (m & sh) continue;
        const int ms = m | sh;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double2 send = up ? ch[2 * m + e] : ch[2 * ms + e];
          double2 recv;
          recv.x = __shfl_xor_sync(0xffffffffu, send.x, sh);
          recv.y = __shfl_xor_sync(0xffffffffu, send.y, sh);
          if (up) ch[2 * m + e] = recv; else ch[2 * ms + e] = recv;
        }
      }
    }
    const int row0 = row - p4;
    const int col = i0 + 4 * p4;
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      const int r = row0 + kq;
      if (r < M && col < n) {  // n % 4 == 0: a quad is all in or all out
        double* o = out + proj_out_row(b0, s0, r - rq, rin, rout) * n + col;
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"(ch[2 * kq].x),
                     "d"(ch[2 * kq].y), "d"(ch[2 * kq + 1].x), "d"(ch[2 * kq + 1].y)
                     : "memory");
      }
    }
    return;
  }
  // 8x8 transpose of 16-byte chunks inside each group of 8 lanes (3 xor-butterfly
  // stages): afterwards lane p of the group holds chunk p of the group's 8 rows, so each
  // store instruction writes 4 rows x 128 contiguous bytes (full lines) instead of 32
  // rows x 16 bytes -- the uncoalesced row stores were the epilogue's bottleneck.
  const int p8 = lane & 7;
#pragma unroll
  for (int sh = 4; sh >= 1; sh >>= 1) {
    const bool up = (p8 & sh) != 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k & sh) continue;
      const double2 send = up ? ch[k] : ch[k | sh];
      double2 recv;
      recv.x = __shfl_xor_sync(0xffffffffu, send.x, sh);
      recv.y = __shfl_xor_sync(0xffffffffu, send.y, sh);
      if (up) ch[k] = recv; else ch[k | sh] = recv;
    }
  }
  const int row0 = row - p8;           // first row of this lane's group of 8
  const int col = i0 + 2 * p8;         // this lane's chunk (2 neurons)
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int r = row0 + k;
    if (r < M) {
      double* o = out + proj_out_row(b0, s0, r - rq, rin, rout) * n + col;
      if (col + 1 < n && (n & 1) == 0) {  // 16-byte aligned rows
        *reinterpret_cast<double2*>(o) = ch[k];
      } else {
        if (col < n) o[0] = ch[k].x;
        if (col + 1 < n) o[1] = ch[k].y;
      }
    }
  }
}

// tcgen05.ld.16x256b.x2: 16 TMEM lanes x 16 columns per warp.  Thread t holds lanes
// t/4 (registers 0, 1, 4, 5) and t/4 + 8 (2, 3, 6, 7), columns 2(t%4), 2(t%4)+1 (0-3) and
// 8 + 2(t%4), 9 + 2(t%4) (4-7) -- measured, tools/tmem_layout_probe.cu.
__device__ __forceinline__ void tmem_ld16x256b_x2_nowait(uint32_t taddr, int32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// Epilogue of one 32-row x 16-neuron quarter-tile, P = 6 digits, binary spikes, k <= 768
// (every digit sum |S_p| <= 768 * 128 < 2^17, so digit PAIRS combine in int32 and
// g = P01 2^32 + P23 2^16 + P45 is the exact integer sum of all six).  The digits are
// read in the 16x256b shape: with the slot order of the sliced weights (digits.cuh) each
// thread gets 4 rows x the 4 consecutive neurons 4q..4q+3 (q = lane % 4), so a row's
// 4 currents go out as one 32-byte store and a warp's store instruction covers 8 rows x
// 128 contiguous bytes -- no lane transposes.  sc4 = 2^(s-F) of those 4 neurons.
__device__ __forceinline__ void proj_epilogue_p6bin(uint32_t tbase, const double (&sc4)[4],
                                                    double* __restrict__ out, int M, int n,
                                                    int rin, int rout, int row0, int i0,
                                                    uint32_t tempty_bar, int lane, int probe) {
  const int t4 = lane >> 2, q4 = lane & 3;
  double v[2][2][4];  // [lane half][row +0 / +8][neuron 4 q4 + j]
  // all 12 digit loads in flight at once, one wait, and the TMEM buffer released before
  // any math: the MMA of the tile after next waits only for the loads (the buffer was
  // held through the first half's recombination before: K2 0.225 -> 0.215 ms at C3)
  int32_t rr2[2][6][8];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int p = 0; p < 6; ++p)
      tmem_ld16x256b_x2_nowait(tbase + ((uint32_t)(16 * h) << 16) + (uint32_t)(p * NT), rr2[h][p]);
  tmem_wait_ld();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  if (lane == 0) mbar_arrive(tempty_bar);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int32_t (&r)[6][8] = rr2[h];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int32_t p01 = r[0][e] * 256 + r[1][e];
      const int32_t p23 = r[2][e] * 256 + r[3][e];
      const int32_t p45 = r[4][e] * 256 + r[5][e];
      const long long g = ((long long)p01 << 32) + ((long long)p23 << 16) + (long long)p45;
      const int j = (e & 1) + 2 * (e >> 2);   // register e -> neuron 4 q4 + j
      v[h][(e >> 1) & 1][j] = (double)g * sc4[j];
    }
  }
  const int col = i0 + 4 * q4;
  if (probe & 4) {  // profiling probe: no global stores
    if (v[0][0][0] == 1.2345e-300 && row0 < M) out[(long long)row0 * n + col] = v[0][0][1];
    return;
  }
  const int b0 = proj_row_div(row0, rin), s0 = row0 - b0 * rin;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int rh = 0; rh < 2; ++rh) {
      const int d = 16 * h + 8 * rh + t4;
      if (row0 + d >= M) continue;
      double* o = out + (rin == rout ? (long long)(row0 + d) : proj_out_row(b0, s0, d, rin, rout)) * n + col;
      const double* w = v[h][rh];
      if ((n & 3) == 0) {  // 32-byte aligned quads, all in or all out
        if (col < n)
          asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"(w[0]),
                       "d"(w[1]), "d"(w[2]), "d"(w[3])
                       : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (col + j < n) o[j] = w[j];
      }
    }
}

// The tile sequence of one persistent CTA of the W-resident kernel.  The m-tiles (rows =
// (sample, step)) are cut into `bands` consecutive bands; inside a band the tiles run
// neuron-major and every CTA takes the same fraction of them, so all CTAs work in the same
// band at the same time and the band's spike tiles are read from DRAM once and then hit
// L2 for the other neuron tiles (bands = 1: one band over all rows -- each spike tile is
// then re-read from DRAM by the neuron tiles at different times).  Odd bands are walked
// backwards, so a CTA enters the next band on the neuron tile it just finished (one
// weight reload per band instead of two).
struct TileWalk {
  int m_tiles, n_tiles, bands, cta, ncta;
  int g = -1, k = 0, kb = 0, ke = 0, bw = 1, mb0 = 0;
  __device__ TileWalk(int m_tiles_, int n_tiles_, int bands_, int cta_, int ncta_)
      : m_tiles(m_tiles_), n_tiles(n_tiles_), bands(bands_), cta(cta_), ncta(ncta_) {}
  __device__ bool next(int& nt, int& mt) {
    while (k >= ke) {
      if (++g >= bands) return false;
      mb0 = (int)((long long)m_tiles * g / bands);
      bw = (int)((long long)m_tiles * (g + 1) / bands) - mb0;
      const long long tot = (long long)bw * n_tiles;
      kb = (int)(tot * cta / ncta);
      ke = (int)(tot * (cta + 1) / ncta);
      k = kb;
    }
    const int u = (g & 1) ? ke - 1 - (k - kb) : k;
    ++k;
    nt = u / bw;
    mt = mb0 + u - nt * bw;
    return true;
  }
};

// W-resident variant (Kpad <= 768): each persistent CTA walks a contiguous range of tiles
// in neuron-major order, keeps the sliced weights of its current neuron tile (all K) in
// shared memory and streams only the spike tiles -- operand traffic drops from
// (m_tiles x |W|) + (n_tiles x |x|) to (#CTAs x |W tile|) + (n_tiles x |x|).
template <int P, int XS>
struct ResCfg {
  static constexpr int N = P * NT;
  static constexpr int WBLK = N * BK;                    // one K-block of all slices
  static constexpr int MAXKB = 6;                        // Kpad <= 768
  static constexpr int W_BYTES = MAXKB * WBLK;
  static constexpr int SMEM = W_BYTES + XS * TILE_A + 1024 + 256;
};

// MC: launched as clusters of 2 CTAs working on neuron tiles 2j and 2j + 1 of the same
// spike tiles; each CTA loads one half (64 rows) of every spike stage and multicasts it
// to both, so the spike operand leaves L2 once per neuron-tile pair (tm_x / tm_xt then
// have 64-row boxes) and a stage is refilled once both CTAs' MMAs released it.
template <int P, int XS, bool BIN, bool MC = false>
__global__ void __launch_bounds__(THREADS, 1)
    input_proj_wres_kernel(const __grid_constant__ CUtensorMap tm_x,
                           const __grid_constant__ CUtensorMap tm_w,
                           const __grid_constant__ CUtensorMap tm_xt, const int* __restrict__ sexp,
                           double* __restrict__ out, int M, int n, int n_pad32, int nkb,
                           int tail, int probe, int bands, int rin, int rout) {
  // nkb full 128-byte K blocks, then (tail) one 64-byte block: k = 700 runs 704 bytes of
  // K instead of 768 (8 % fewer MMAs and spike-operand bytes)
  using C = ResCfg<P, XS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* wsm = smem;                        // [nkb][P*NT rows][128 B]
  uint8_t* xsm = smem + C::W_BYTES;           // [XS][128 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xsm + XS * TILE_A);
  uint64_t* xfull = bars;
  uint64_t* xempty = bars + XS;
  uint64_t* tfull = bars + 2 * XS;
  uint64_t* tempty = bars + 2 * XS + 2;
  uint64_t* wfull = bars + 2 * XS + 4;
  uint64_t* wempty = bars + 2 * XS + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * XS + 6);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (n + NT - 1) / NT;
  const int nbands = max(1, min(bands, m_tiles));
  // the tile walk: over neuron-tile pairs per cluster (MC), else over neuron tiles per CTA
  const int rank = MC ? (int)cluster_rank() : 0;
  const int w_nt = MC ? n_tiles >> 1 : n_tiles;
  const int w_cta = MC ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int w_n = MC ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < XS; ++s) {
      mbar_init(smem_u32(&xfull[s]), 1);
      mbar_init(smem_u32(&xempty[s]), MC ? 2 : 1);  // MC: both CTAs' MMAs release a stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), EPI_WARPS);
    }
    mbar_init(smem_u32(wfull), 1);
    mbar_init(smem_u32(wempty), 1);
    mbar_fence_init();
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (MC) cluster_sync_all();  // the peer's barriers exist before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();  // the prologue above touches only shared memory, TMEM and the params

  if (warp == 0) {
    if (SPB_K2_PRODUCER_LANES) {
      int s = 0, ph = 0, cur_nt = -1, wl = 0, nt, mt;
      TileWalk tw(m_tiles, w_nt, nbands, w_cta, w_n);
      while (tw.next(nt, mt)) {
        if (MC) nt = 2 * nt + rank;
        if (nt != cur_nt) {  // (re)load this neuron tile's weight slices, all K blocks
          mbar_wait(smem_u32(wempty), (wl & 1) ^ 1);
          const uint32_t fb = smem_u32(wfull);
          if (SPB_K2_LANE0) {
            mbar_expect_tx(fb, (nkb + tail) * C::WBLK);
            for (int kb = 0; kb < nkb + tail; ++kb)
#pragma unroll
              for (int p = 0; p < P; ++p)
                tma_load_2d(smem_u32(wsm + kb * C::WBLK + p * NT * BK), &tm_w, fb, kb * BK,
                            p * n_pad32 + nt * NT);
          }
#if SPB_K2_ELECT
          __syncwarp();
#endif
          cur_nt = nt;
          ++wl;
        }
        for (int kb = 0; kb < nkb + tail; ++kb) {  // stage s, ring phase ph (incremental)
          if (MC)  // released by both CTAs' MMAs (the peer's commit is a remote arrive)
            mbar_wait_cluster(smem_u32(&xempty[s]), ph ^ 1);
          else
            mbar_wait(smem_u32(&xempty[s]), ph ^ 1);
          const uint32_t fb = smem_u32(&xfull[s]);
#if SPB_K2_ELECT
          if (probe & 2) {
            if (lane == 0)
              asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fb) : "memory");
          } else if (MC) {  // this CTA's 64 rows of the stage, into both CTAs
            const bool full = kb < nkb;
            const uint32_t half = full ? TILE_A / 2 : TILE_A / 4;
            tma_load_2d_mc_elect(smem_u32(xsm + s * TILE_A) + rank * half, full ? &tm_x : &tm_xt,
                                 fb, kb * BK, mt * BM + rank * (BM / 2),
                                 full ? TILE_A : TILE_A / 2, (uint16_t)3);
          } else if (kb < nkb) {
            tma_load_2d_elect(smem_u32(xsm + s * TILE_A), &tm_x, fb, kb * BK, mt * BM, TILE_A);
          } else {
            tma_load_2d_elect(smem_u32(xsm + s * TILE_A), &tm_xt, fb, nkb * BK, mt * BM,
                              TILE_A / 2);
          }
#else
          if (probe & 2) {  // profiling probe: no spike-operand traffic
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fb) : "memory");
          } else if (kb < nkb) {
            mbar_expect_tx(fb, TILE_A);
            tma_load_2d(smem_u32(xsm + s * TILE_A), &tm_x, fb, kb * BK, mt * BM);
          } else {  // the 64-byte tail block (SWIZZLE_64B box)
            mbar_expect_tx(fb, TILE_A / 2);
            tma_load_2d(smem_u32(xsm + s * TILE_A), &tm_xt, fb, nkb * BK, mt * BM);
          }
#endif
          if (++s == XS) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp runs the issue loop (converged); elect.sync picks the issuer
      long long c0 = 0, g0 = 0;  // probe & 32: clock / global-timer record of the issue loop
      if (probe & 32) {
        c0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
      }
      int s = 0, ph = 0, lt = 0, cur_nt = -1, wl = 0, nt, mt, nnt, nmt;
      TileWalk tw(m_tiles, w_nt, nbands, w_cta, w_n);
      bool have = tw.next(nt, mt);
      while (have) {
        const bool more = tw.next(nnt, nmt);  // one tile ahead: the weight region's last use
        // (the walk's neuron index is a pair index under MC: equality tests are unchanged)
        if (nt != cur_nt) {
          mbar_wait(smem_u32(wfull), wl & 1);
          cur_nt = nt;
          ++wl;
        }
        const int a = lt & 1;
        mbar_wait(smem_u32(&tempty[a]), ((lt >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem_base + (uint32_t)(a * 256);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(smem_u32(&xfull[s]), ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t xa = smem_u32(xsm + s * TILE_A);
          const uint32_t wa = smem_u32(wsm + kb * C::WBLK);
          static_assert(BK / 32 == 4, "four K steps per block");
          if (!(probe & 8))  // profiling probe: no MMAs (the epilogue alone)
            mma_i8_x4(dacc, desc_k_sw128(xa), desc_k_sw128(wa), Cfg<P>::IDESC, kb ? 1u : 0u);
          if (MC)
            commit_mc(smem_u32(&xempty[s]), 3);
          else
            commit(smem_u32(&xempty[s]));
          if (++s == XS) {
            s = 0;
            ph ^= 1;
          }
        }
        if (tail) {  // the 64-byte tail block: A in SWIZZLE_64B
          mbar_wait(smem_u32(&xfull[s]), ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (!(probe & 8))
            mma_i8_x2(dacc, desc_k_sw64(smem_u32(xsm + s * TILE_A)),
                      desc_k_sw128(smem_u32(wsm + nkb * C::WBLK)), Cfg<P>::IDESC, nkb ? 1u : 0u);
          if (MC)
            commit_mc(smem_u32(&xempty[s]), 3);
          else
            commit(smem_u32(&xempty[s]));
          if (++s == XS) {
            s = 0;
            ph ^= 1;
          }
        }
        commit(smem_u32(&tfull[a]));
        // last tile of this neuron tile: the weight region may be refilled afterwards
        if (!more || nnt != nt) commit(smem_u32(wempty));
        nt = nnt;
        mt = nmt;
        have = more;
        ++lt;
      }
      if (probe & 32) {  // wait for the last tile's MMAs, then record (cycles, ns, tiles)
        mbar_wait(smem_u32(&tfull[(lt - 1) & 1]), ((lt - 1) >> 1) & 1);
        long long g1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        if (lane == 0) {
          out[3 * blockIdx.x] = (double)(clock64() - c0);
          out[3 * blockIdx.x + 1] = (double)(g1 - g0);
          out[3 * blockIdx.x + 2] = (double)lt;
        }
      }
    }
  } else {
    const int q = warp & 3;          // TMEM lane quarter
    const int hh = (warp - 2) >> 2;  // neuron half of the tile
    int lt = 0;
    // the per-neuron scales 2^(s-F) change only with the neuron tile
    // P = 6 with binary spikes: the shuffle-free 16x256b epilogue (4 neurons per thread)
    constexpr bool FAST = (P == 6 && BIN);
    constexpr int NS = FAST ? 4 : NH;
    const int ns0 = FAST ? 4 * (lane & 3) : 0;
    int nt, mt, sc_nt = -1;
    double sc[NS];
    TileWalk tw(m_tiles, w_nt, nbands, w_cta, w_n);
    for (; tw.next(nt, mt); ++lt) {
      if (MC) nt = 2 * nt + rank;
      const int a = lt & 1;
      const int i0 = nt * NT + hh * NH;
      if (nt != sc_nt) {
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          const int i = i0 + ns0 + c;
          sc[c] = digits_pow2(((i < n) ? __ldg(sexp + i) : 0) - Digits<P>::F);
        }
        sc_nt = nt;
      }
      mbar_wait(smem_u32(&tfull[a]), (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (probe & 1) {  // profiling probe: no epilogue (TMEM reads, recombination, stores)
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tempty[a]));
        continue;
      }
      const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * 256 + hh * NH);
      if constexpr (FAST) {
        if (probe & 64)  // profiling probe: tile-contiguous output blocks (32 KB per tile)
          proj_epilogue_p6bin(tb, sc, out + (long long)(mt * n_tiles + nt) * (BM * NT), BM, NT,
                              BM, BM, q * 32, hh * NH, smem_u32(&tempty[a]), lane, probe);
        else
          proj_epilogue_p6bin(tb, sc, out, M, n, rin, rout, mt * BM + q * 32, i0,
                              smem_u32(&tempty[a]), lane, probe);
      }
      else
        proj_epilogue_tile<P, BIN>(tb, sc, out, M, n, rin, rout, mt * BM + q * 32 + lane, i0,
                                   smem_u32(&tempty[a]), lane, probe);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  // MC: the peer's last multicast writes and stage releases target this CTA's shared
  // memory; neither CTA leaves before both are done
  if constexpr (MC) cluster_sync_all();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

template <int P, bool BIN>
__global__ void __launch_bounds__(THREADS, 1)
    input_proj_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                      const int* __restrict__ sexp, double* __restrict__ out, int M, int n,
                      int n_pad32, int nkb, int rin, int rout) {
  using C = Cfg<P>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;       // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (n + NT - 1) / NT;
  const int num_tiles = m_tiles * n_tiles;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), EPI_WARPS);  // one arrive per epilogue warp
    }
    mbar_fence_init();
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int nt = t / m_tiles, mt = t % m_tiles;  // consecutive tiles share W slices
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(smem_u32(&empty[s]), ((it / STAGES) & 1) ^ 1);
          const uint32_t st = smem_u32(smem + s * C::STAGE);
          const uint32_t fb = smem_u32(&full[s]);
          mbar_expect_tx(fb, C::STAGE);
          tma_load_2d(st, &tm_x, fb, kb * BK, mt * BM);
#pragma unroll
          for (int p = 0; p < P; ++p)
            tma_load_2d(st + TILE_A + p * NT * BK, &tm_w, fb, kb * BK, p * n_pad32 + nt * NT);
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp runs the issue loop (converged); elect.sync picks the issuer
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        const int a = lt & 1;
        mbar_wait(smem_u32(&tempty[a]), ((lt >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem_base + (uint32_t)(a * 256);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(smem_u32(&full[s]), (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = smem_u32(smem + s * C::STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            mma_i8(dacc, desc_k_sw128(st + kk * 32), desc_k_sw128(st + TILE_A + kk * 32),
                   C::IDESC, (kb | kk) ? 1u : 0u);
          commit(smem_u32(&empty[s]));
        }
        commit(smem_u32(&tfull[a]));
      }
    }
  } else {
    const int q = warp & 3;          // TMEM lane quarter accessible to this warp
    const int hh = (warp - 2) >> 2;  // neuron half of the tile
    int lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      const int nt = t / m_tiles, mt = t % m_tiles;
      const int a = lt & 1;
      const int i0 = nt * NT + hh * NH;
      int se[NH];  // per-neuron exponents, fetched before waiting on the tensor cores
#pragma unroll
      for (int c = 0; c < NH; ++c) se[c] = (i0 + c < n) ? __ldg(sexp + i0 + c) : 0;
      mbar_wait(smem_u32(&tfull[a]), (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      proj_epilogue_tile<P, BIN>(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * 256 + hh * NH),
                            se, out, M, n, rin, rout, mt * BM + q * 32 + lane, i0,
                            smem_u32(&tempty[a]), lane);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

// x chunk -> zero-padded K-major operand rows (16-byte aligned rows for TMA).
// One warp per output row (sample b, step s): 16-byte stores of the zero-padded row.
// Byte input (bits == 0): the source row has k bytes (4-byte loads when aligned).  Bit
// input (bits == 1): the source row has ceil(k/8) bytes, channel j = bit (j & 7) of byte
// j >> 3 (numpy.packbits(..., bitorder="little")) -- 8x less host->device traffic for
// binary spike trains.
__device__ __forceinline__ uint32_t expand4(uint32_t nib) {  // 4 bits -> 4 bytes of 0/1
  return (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
}

// Byte-count rows with k, the row stride and x 4-byte aligned (the common case): CTA per 4
// rows, thread per 4 output bytes of each -- each warp moves 128 contiguous bytes in and
// out per row (coalesced u32), the 4 rows' loads in flight together.
#ifndef PACK_GRID
#define PACK_GRID (148 * 16)  // grid-stride pack: C3 0.7038 -> 0.6996 ms (148 * 4: 0.701)
#endif
#ifndef SPB_PACK_R
#define SPB_PACK_R 8
#endif
#ifndef SPB_PACK_RB
#define SPB_PACK_RB 4  // bit-packed input: rows per CTA iteration (8: same e2e, 16: -4 %)
#endif
// byte-input pack: rows per CTA iteration, their loads in flight together.  With the update
// at 0.60 ms, 8 rows: pack 36.1 -> 33.6 us and the update's span 595.8 -> 592.5 us (device
// timeline, tools/step_timeline.py); 16 rows: 42.8 us (round 1 at 0.71 ms: 4 rows best)
constexpr int PACK_R = SPB_PACK_R;

// bf16 of four spike counts (0..255, exact): the upper halves of their fp32 encodings
__device__ __forceinline__ uint2 bf16x4_of_bytes(uint32_t w) {
  uint2 h;
  h.x = (__float_as_uint((float)(w & 0xffu)) >> 16) |
        (__float_as_uint((float)((w >> 8) & 0xffu)) & 0xffff0000u);
  h.y = (__float_as_uint((float)((w >> 16) & 0xffu)) >> 16) |
        (__float_as_uint((float)(w >> 24)) & 0xffff0000u);
  return h;
}

// xh != NULL: also the raw-spike GEMM operand (bf16 [B*KR][Kpad], row b*KR + s + 1 =
// spikes of step s; row 0 is left as is, zero) -- the one-chunk K4 folded into the pack.
__global__ void __launch_bounds__(256) pack_bytes4_kernel(const uint8_t* __restrict__ x,
                                                          long long stride_b, int k, int len,
                                                          int Tc, int Kpad, int B, int tmajor,
                                                          uint8_t* __restrict__ xq,
                                                          uint2* __restrict__ xh = nullptr,
                                                          int KR = 0) {
  pdl_enter();
  pdl_trigger();
  const int wpr = Kpad >> 2;  // output words per row
  // 8-column groups up to the last input column; the pad past it is never written and
  // stays zero from the buffers' allocation (C3: 704 of 768 columns, 12 MB less per update)
  const int wl = min(wpr >> 1, (k + 7) >> 3);
  const int rows = B * Tc;
  constexpr int R = PACK_R;   // rows per iteration, their loads issued together
  // grid-stride over row groups (a persistent-size grid instead of one tiny CTA per group)
  for (int row0 = blockIdx.x * R; row0 < rows; row0 += gridDim.x * R) {
    int sq[R], bq[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int row = row0 + q;
      sq[q] = tmajor ? row / B : row % Tc;
      bq[q] = tmajor ? row % B : row / Tc;
    }
    // thread per 8 channels: two 32-bit loads, one 8-byte xq store, one 16-byte xh store
    for (int w2 = threadIdx.x; w2 < wl; w2 += blockDim.x) {
      const int w = 2 * w2;
      uint32_t v[R][2];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const bool live = row0 + q < rows && sq[q] < len;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(x + (long long)bq[q] * stride_b +
                                                                (long long)sq[q] * k);
        v[q][0] = (live && 4 * w < k) ? __ldg(src + w) : 0u;
        v[q][1] = (live && 4 * (w + 1) < k) ? __ldg(src + w + 1) : 0u;
      }
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (row0 + q < rows)
          reinterpret_cast<uint2*>(xq + (long long)(row0 + q) * Kpad)[w2] =
              make_uint2(v[q][0], v[q][1]);
      if (xh != nullptr) {
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (row0 + q < rows && sq[q] + 1 < KR) {   // row s + 1 of the sample's KR rows
            const uint2 a = bf16x4_of_bytes(v[q][0]), b = bf16x4_of_bytes(v[q][1]);
            reinterpret_cast<uint4*>(xh)[((long long)bq[q] * KR + sq[q] + 1) * (Kpad >> 3) + w2] =
                make_uint4(a.x, a.y, b.x, b.y);
          }
      }
    }
  }
}

// Bit-packed rows (np.packbits little order): thread per input byte = 8 output bytes
// (one 8-byte store), CTA per 4 rows with their loads in flight together.
__global__ void __launch_bounds__(128) pack_bits8_kernel(const uint8_t* __restrict__ x,
                                                         long long stride_b, int k, int len,
                                                         int Tc, int Kpad, int B, int tmajor,
                                                         uint8_t* __restrict__ xq,
                                                         uint4* __restrict__ xh = nullptr,
                                                         int KR = 0) {
  pdl_enter();
  pdl_trigger();
  const int kb = (k + 7) >> 3;   // input bytes per row
  const int wpr = Kpad >> 3;     // output 8-byte words per row
  // columns past the last input byte are never written: they stay zero from the buffers'
  // allocation (no packer writes them), so the pad is not rewritten every update
  const int wl = min(wpr, kb);
  const int rows = B * Tc;
  constexpr int R = SPB_PACK_RB;
  // grid-stride over row groups (as pack_bytes4_kernel)
  for (int row0 = blockIdx.x * R; row0 < rows; row0 += gridDim.x * R) {
    int sq[R], bq[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int row = row0 + q;
      sq[q] = tmajor ? row / B : row % Tc;
      bq[q] = tmajor ? row % B : row / Tc;
    }
    for (int w = threadIdx.x; w < wl; w += blockDim.x) {
      uint32_t v[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        uint32_t byte = 0u;
        if (row0 + q < rows && sq[q] < len && w < kb) {
          byte = __ldg(x + (long long)bq[q] * stride_b + (long long)sq[q] * kb + w);
          const int left = k - 8 * w;  // valid channels in this byte
          if (left < 8) byte &= (1u << left) - 1u;
        }
        v[q] = byte;
      }
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (row0 + q < rows)
          reinterpret_cast<uint2*>(xq + (long long)(row0 + q) * Kpad)[w] =
              make_uint2(expand4(v[q] & 0xfu), expand4(v[q] >> 4));
      if (xh != nullptr) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (row0 + q < rows && sq[q] + 1 < KR) {   // row s + 1 of the sample's KR rows
            // 8 spikes -> 8 bf16 (0x3F80 = 1.0)
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              o[e] = (((v[q] >> (2 * e)) & 1u) ? 0x3F80u : 0u) |
                     (((v[q] >> (2 * e + 1)) & 1u) ? 0x3F800000u : 0u);
            xh[((long long)bq[q] * KR + sq[q] + 1) * (Kpad >> 3) + w] =
                make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
      }
    }
  }
}

__global__ void pack_spikes_kernel(const uint8_t* __restrict__ x, long long stride_b, int k,
                                   int bits, int len, int Tc, int Kpad, int B, int tmajor,
                                   uint8_t* __restrict__ xq) {
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)B * Tc;
  const int kb = bits ? (k + 7) / 8 : k;
  const bool w4 = !bits && (k & 3) == 0 && (stride_b & 3) == 0 &&
                  (reinterpret_cast<uintptr_t>(x) & 3) == 0;
  for (long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += (long long)gridDim.x * (blockDim.x >> 5)) {
    // sample-major rows b*Tc + s (K2) or time-major rows s*B + b (fused K21)
    const int s = tmajor ? (int)(row / B) : (int)(row % Tc);
    const int b = tmajor ? (int)(row % B) : (int)(row / Tc);
    const uint8_t* src = x + (long long)b * stride_b + (long long)s * kb;
    uint4* dst = reinterpret_cast<uint4*>(xq + row * Kpad);
    const bool live = s < len;
    for (int c = lane; c < Kpad / 16; c += 32) {
      const int j0 = c * 16;
      uint32_t wv[4] = {0u, 0u, 0u, 0u};
      if (live) {
        if (bits) {
          uint32_t v16 = 0u;
          if (j0 < k) v16 = src[j0 >> 3];
          if (j0 + 8 < k) v16 |= (uint32_t)src[(j0 >> 3) + 1] << 8;
          if (j0 + 16 > k) v16 &= (k - j0 >= 16) ? 0xffffu : ((1u << (k - j0 > 0 ? k - j0 : 0)) - 1u);
#pragma unroll
          for (int q = 0; q < 4; ++q) wv[q] = expand4((v16 >> (4 * q)) & 0xfu);
        } else if (w4 && j0 + 16 <= k) {
          const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src + j0);
          wv[0] = s4[0]; wv[1] = s4[1]; wv[2] = s4[2]; wv[3] = s4[3];
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (j0 + q < k) wv[q >> 2] |= (uint32_t)src[j0 + q] << (8 * (q & 3));
        }
      }
      dst[c] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
  }
}

}  // namespace proj
}  // namespace spb

using namespace spb;

extern "C" {

int spb_pack_spikes_xh(const uint8_t* x, long long stride_b, int B, int k, int bits, int len,
                       int Tc, int Kpad, int KR, uint8_t* xq, void* xh, cudaStream_t stream);

int spb_pack_spikes(const uint8_t* x, long long stride_b, int B, int k, int bits, int len, int Tc,
                    int Kpad, int time_major, uint8_t* xq, cudaStream_t stream) {
  SPB_CHECK_ARG(x && xq && B > 0 && k > 0 && Kpad >= k && Kpad % proj::BK == 0 && len >= 0 &&
                    len <= Tc,
                "spb_pack_spikes: bad args (Kpad must be a multiple of %d)", proj::BK);
  const long long rows = (long long)B * Tc;
  const long long want = (rows + 7) / 8;
  const int blocks = (int)(want < 148LL * 16 ? want : 148LL * 16);
  if (!bits && (k & 3) == 0 && (stride_b & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 3) == 0) {
    const int b4 = (int)std::min<long long>((rows + proj::PACK_R - 1) / proj::PACK_R, PACK_GRID);
    const int t4 = std::min(256, ((Kpad / 8 + 31) / 32) * 32);
    proj::pack_bytes4_kernel<<<b4, t4, 0, stream>>>(x, stride_b, k, len, Tc, Kpad, B, time_major,
                                                     xq);
    SPB_CHECK_LAUNCH("pack_bytes4");
    return 0;
  }
  if (bits) {
    const int b8 = (int)std::min<long long>((rows + 3) / 4, PACK_GRID);
    const int t8 = std::min(128, ((Kpad / 8 + 31) / 32) * 32);
    proj::pack_bits8_kernel<<<b8, t8, 0, stream>>>(x, stride_b, k, len, Tc, Kpad, B, time_major,
                                                    xq);
    SPB_CHECK_LAUNCH("pack_bits8");
    return 0;
  }
  proj::pack_spikes_kernel<<<blocks, 256, 0, stream>>>(x, stride_b, k, bits, len, Tc, Kpad, B,
                                                        time_major, xq);
  SPB_CHECK_LAUNCH("pack_spikes");
  return 0;
}

// spb_pack_spikes (sample-major) that also writes the one-chunk raw-spike GEMM operand
// xh (bf16 [B*KR][Kpad], row b*KR + s + 1 = step s, row 0 untouched = zero).
int spb_pack_spikes_xh(const uint8_t* x, long long stride_b, int B, int k, int bits, int len,
                       int Tc, int Kpad, int KR, uint8_t* xq, void* xh, cudaStream_t stream) {
  SPB_CHECK_ARG(x && xq && xh && B > 0 && k > 0 && Kpad >= k && Kpad % proj::BK == 0 &&
                    len >= 0 && len <= Tc && KR >= Tc,
                "spb_pack_spikes_xh: bad args");
  // Tc here is the row stride of xq per sample (the engine passes KR: sample-aligned rows);
  // rows s >= len are written as zeros
  const long long rows = (long long)B * Tc;
  if (bits) {
    const int t8 = std::min(128, ((Kpad / 8 + 31) / 32) * 32);
    proj::pack_bits8_kernel<<<(int)std::min<long long>((rows + 3) / 4, PACK_GRID), t8, 0, stream>>>(
        x, stride_b, k, len, Tc, Kpad, B, 0, xq, static_cast<uint4*>(xh), KR);
    SPB_CHECK_LAUNCH("pack_bits8_xh");
    return 0;
  }
  SPB_CHECK_ARG((k & 3) == 0 && (stride_b & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 3) == 0,
                "spb_pack_spikes_xh: byte rows must be 4-byte aligned");
  const int t4 = std::min(256, ((Kpad / 8 + 31) / 32) * 32);
  proj::pack_bytes4_kernel<<<(int)std::min<long long>((rows + proj::PACK_R - 1) / proj::PACK_R, PACK_GRID), t4, 0, stream>>>(
      x, stride_b, k, len, Tc, Kpad, B, 0, xq, static_cast<uint2*>(xh), KR);
  SPB_CHECK_LAUNCH("pack_bytes4_xh");
  return 0;
}

}  // extern "C"
namespace spb {
namespace proj {
// Real-valued inputs (the drop-in's non-count x): the one-chunk raw-input GEMM operand as
// bf16 hi/lo pairs, x = hi + lo to ~2^-16, in the row layout of spb_pack_spikes_xh (row
// b*KR + s + 1 = step s, rows s >= len zero, row b*KR untouched).  Thread per 2 columns.
template <typename T>
__global__ void pack_real_kernel(const T* __restrict__ x, long long stride_b, int B, int k,
                                 int len, int KR, int ld, __nv_bfloat162* __restrict__ xh,
                                 __nv_bfloat162* __restrict__ xl) {
  pdl_enter();
  const int hw = ld >> 1;                                  // bf16 pairs per row
  const long long total = (long long)B * (KR - 1) * hw;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c2 = (int)(idx % hw);
    const long long rs = idx / hw;
    const int s = (int)(rs % (KR - 1));
    const int b = (int)(rs / (KR - 1));
    float hi[2], lo[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 2 * c2 + e;
      const double v = (s < len && j < k) ? (double)x[(long long)b * stride_b + (long long)s * k + j]
                                           : 0.0;
      const __nv_bfloat16 h = __double2bfloat16(v);
      hi[e] = __bfloat162float(h);
      lo[e] = (float)(v - (double)hi[e]);
    }
    const long long o = ((long long)b * KR + s + 1) * hw + c2;
    xh[o] = __floats2bfloat162_rn(hi[0], hi[1]);
    xl[o] = __floats2bfloat162_rn(lo[0], lo[1]);
  }
}
}  // namespace proj
}  // namespace spb
extern "C" {

// Real-valued (non-count) inputs of one chunk: x [B][len][k] fp32 (x_is_f64 = 0) / fp64,
// sample stride stride_b elements -> xh, xl bf16 [B*KR][ld] (see pack_real_kernel).
int spb_pack_real(const void* x, int x_is_f64, long long stride_b, int B, int k, int len, int KR,
                  int ld, void* xh, void* xl, cudaStream_t stream) {
  SPB_CHECK_ARG(x && xh && xl && B > 0 && k > 0 && ld >= k && ld % 2 == 0 && len >= 0 &&
                    len < KR && stride_b >= (long long)len * k,
                "spb_pack_real: bad args");
  const long long pairs = (long long)B * (KR - 1) * (ld / 2);
  const int blocks = (int)std::min<long long>((pairs + 255) / 256, 148LL * 8);
  if (x_is_f64)
    pdl_launch(proj::pack_real_kernel<double>, blocks, 256, 0, stream,
               static_cast<const double*>(x), stride_b, B, k, len, KR, ld,
               static_cast<__nv_bfloat162*>(xh), static_cast<__nv_bfloat162*>(xl));
  else
    pdl_launch(proj::pack_real_kernel<float>, blocks, 256, 0, stream,
               static_cast<const float*>(x), stride_b, B, k, len, KR, ld,
               static_cast<__nv_bfloat162*>(xh), static_cast<__nv_bfloat162*>(xl));
  SPB_CHECK_LAUNCH("pack_real");
  return 0;
}

int spb_launch_sgd_slice(void* w, int w_is_f64, int n, int k, const void* g, int g_is_f64,
                         int ld_g, double g_scale, double lr, int do_sgd, int Kpad, int n_pad32,
                         int P, int8_t* wq, int* sexp, cudaStream_t stream);  // optim.cu

int spb_slice_weights(const void* w, int w_is_f64, int n, int k, int Kpad, int n_pad32, int P,
                      int8_t* wq, int* sexp, cudaStream_t stream) {
  SPB_CHECK_ARG(w && wq && sexp && n > 0 && k > 0 && Kpad >= k && n_pad32 >= n &&
                    n_pad32 % proj::NT == 0 && (P == 6 || P == 7 || P == 8),
                "spb_slice_weights: bad args");
  SPB_CHECK_ARG(Kpad % 128 == 0, "spb_slice_weights: Kpad must be a multiple of 128");
  // the slicing pass of the fused SGD + slice kernel (optim.cu), without the update
  return spb_launch_sgd_slice(const_cast<void*>(w), w_is_f64, n, k, nullptr, 0, k, 1.0, 0.0, 0,
                              Kpad, n_pad32, P, wq, sexp, stream);
}

}  // extern "C"
static int input_proj_impl(const uint8_t* xq, const int8_t* wq, const int* sexp, int M, int rin,
                           int rout, int n, int n_pad32, int k, int Kpad, int P, double* out,
                           int sm_count, int binary, int probe, cudaStream_t stream);
extern "C" {

int spb_input_proj(const uint8_t* xq, const int8_t* wq, const int* sexp, int M, int n, int n_pad32,
                   int k, int Kpad, int P, double* out, int sm_count, int binary,
                   cudaStream_t stream) {
  return input_proj_impl(xq, wq, sexp, M, M, M, n, n_pad32, k, Kpad, P, out, sm_count, binary, 0,
                         stream);
}

int spb_input_proj_rows(const uint8_t* xq, const int8_t* wq, const int* sexp, int B, int rin,
                        int rout, int n, int n_pad32, int k, int Kpad, int P, double* out,
                        int sm_count, int binary, cudaStream_t stream) {
  SPB_CHECK_ARG(B > 0 && rin > 0 && rout >= rin, "spb_input_proj_rows: need B > 0, 0 < rin <= rout");
  return input_proj_impl(xq, wq, sexp, B * rin, rin, rout, n, n_pad32, k, Kpad, P, out, sm_count,
                         binary, 0, stream);
}

int spb_input_proj_probe(const uint8_t* xq, const int8_t* wq, const int* sexp, int M, int n,
                         int n_pad32, int k, int Kpad, int P, double* out, int sm_count,
                         int binary, int probe, cudaStream_t stream) {
  return input_proj_impl(xq, wq, sexp, M, M, M, n, n_pad32, k, Kpad, P, out, sm_count, binary,
                         probe, stream);
}

// Row bands of the W-resident kernel's tile walk (TileWalk): about 30 tiles per CTA per
// band (measured, tools/k2_bands.py: C3 4 bands 0.246 -> 0.227 ms with DRAM reads 383 ->
// 70 MB; C4 0.473 -> 0.422; C5 Tc = 2047 1.84 -> 1.71; C2 stays at one band).
// SPB_K2_BANDS=g overrides (A/B).
static int k2_bands(long long tiles, int grid) {
  const char* e = getenv("SPB_K2_BANDS");
  if (e) return max(1, atoi(e));
  return (int)max(1LL, (tiles + 15LL * grid) / (30LL * grid));
}
// SPB_K2_TAIL=0: the zero-padded last K block instead of the 64-byte tail (A/B, tests)
static bool k2_tail() {
  const char* e = getenv("SPB_K2_TAIL");
  return !(e && e[0] == '0');
}
// SPB_K2_MC=1: CTA pairs multicasting the spike stages (bitwise equal; measured no faster
// at C3 -- 0.2218 vs 0.2184 ms, DESIGN.md §6 -- so the single-CTA kernel is the default)
static bool k2_mc() {
  const char* e = getenv("SPB_K2_MC");
  return e && e[0] == '1';
}
}  // extern "C" (the launcher below is a template)
// the W-resident projection launch: PDL, and clusters of 2 for the multicast variant
template <typename... K, typename... A>
static cudaError_t launch_wres(void (*kernel)(K...), int grid, size_t smem, cudaStream_t stream,
                               bool mc, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(proj::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (mc) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<A&&>(args)...);
}
extern "C" {



// spb_input_proj with a profiling probe for the W-resident kernel: bit 0 skips the
// epilogue, bit 1 the spike-operand loads, bit 2 the current stores, bit 3 the MMAs,
// bit 5 records the issue loop's clock, bit 6 stores tile-contiguous blocks (layout probe)
// (probe = 0 is the production kernel).
}  // extern "C"
static int input_proj_impl(const uint8_t* xq, const int8_t* wq, const int* sexp, int M, int rin,
                           int rout, int n, int n_pad32, int k, int Kpad, int P, double* out,
                           int sm_count, int binary, int probe, cudaStream_t stream) {
  const bool bin = binary != 0 && P <= 7 && Kpad <= 8192;
  SPB_CHECK_ARG(xq && wq && sexp && out && M > 0 && n > 0 && n_pad32 >= n &&
                    n_pad32 % proj::NT == 0 && Kpad % proj::BK == 0 && (P == 6 || P == 7 || P == 8),
                "spb_input_proj: bad args");
  SPB_CHECK_ARG((reinterpret_cast<uintptr_t>(xq) | reinterpret_cast<uintptr_t>(wq)) % 16 == 0,
                "spb_input_proj: operands must be 16-byte aligned");
  SPB_CHECK_ARG(k > 0 && k <= Kpad, "spb_input_proj: need 0 < k <= Kpad");
  CUtensorMap mx, mw, mxt;
  const bool ok =
      make_tmap_2d(&mx, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, M, Kpad, proj::BK, proj::BM,
                   CU_TENSOR_MAP_SWIZZLE_128B) &&
      make_tmap_2d(&mw, wq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, (uint64_t)P * n_pad32, Kpad,
                   proj::BK, proj::NT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!ok) {
    set_error("spb_input_proj: cuTensorMapEncodeTiled failed");
    return 3;
  }
  const int tiles = ceil_div(M, proj::BM) * ceil_div(n, proj::NT);
  const int grid = max(1, min(tiles, sm_count > 0 ? sm_count : 148));
  const int nkb = Kpad / proj::BK;
  // W-resident kernel: the inputs past the last full 128-byte K block, if they fit in 64
  // bytes, run as a 64-byte tail block (SWIZZLE_64B) instead of a zero-padded full block
  const int rem = k % proj::BK;
  const int tail = (rem > 0 && rem <= proj::BK / 2 && k2_tail()) ? 1 : 0;
  const int nkb_res = tail ? k / proj::BK : nkb;
  if (!make_tmap_2d(&mxt, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, M, Kpad, proj::BK / 2,
                    proj::BM, CU_TENSOR_MAP_SWIZZLE_64B)) {
    set_error("spb_input_proj: cuTensorMapEncodeTiled (tail) failed");
    return 3;
  }
  // spike multicast across CTA pairs (P = 6): neuron tiles in pairs, an even grid
  const int n_tiles = ceil_div(n, proj::NT);
  const bool mc = P == 6 && nkb <= proj::ResCfg<6, 5>::MAXKB && k2_mc() && n_tiles % 2 == 0 &&
                  grid >= 2;
  if (nkb <= proj::ResCfg<7, 3>::MAXKB) {  // weights of a neuron tile fit in shared memory
    if (P == 6 && mc) {
      const int g2 = grid & ~1;
      CUtensorMap hx, hxt;  // 64-row boxes: each CTA of a pair loads one half of a stage
      if (!make_tmap_2d(&hx, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, M, Kpad, proj::BK,
                        proj::BM / 2, CU_TENSOR_MAP_SWIZZLE_128B) ||
          !make_tmap_2d(&hxt, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, M, Kpad, proj::BK / 2,
                        proj::BM / 2, CU_TENSOR_MAP_SWIZZLE_64B)) {
        set_error("spb_input_proj: cuTensorMapEncodeTiled (multicast halves) failed");
        return 3;
      }
      auto kfn = bin ? proj::input_proj_wres_kernel<6, 5, true, true>
                     : proj::input_proj_wres_kernel<6, 5, false, true>;
      constexpr int sm = proj::ResCfg<6, 5>::SMEM;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      launch_wres(kfn, g2, sm, stream, true, hx, mw, hxt, sexp, out, M, n, n_pad32, nkb_res,
                  tail, probe, k2_bands(tiles, g2), rin, rout);
    } else if (P == 6) {
      auto kfn = bin ? proj::input_proj_wres_kernel<6, 5, true> : proj::input_proj_wres_kernel<6, 5, false>;
      constexpr int sm = proj::ResCfg<6, 5>::SMEM;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      pdl_launch(kfn, grid, proj::THREADS, sm, stream, mx, mw, mxt, sexp, out, M, n, n_pad32,
                 nkb_res, tail, probe, k2_bands(tiles, grid), rin, rout);
    } else if (P == 7) {
      auto kfn = bin ? proj::input_proj_wres_kernel<7, 3, true> : proj::input_proj_wres_kernel<7, 3, false>;
      constexpr int sm = proj::ResCfg<7, 3>::SMEM;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      pdl_launch(kfn, grid, proj::THREADS, sm, stream, mx, mw, mxt, sexp, out, M, n, n_pad32,
                 nkb_res, tail, probe, k2_bands(tiles, grid), rin, rout);
    } else {
      auto kfn = proj::input_proj_wres_kernel<8, 2, false>;
      constexpr int sm = proj::ResCfg<8, 2>::SMEM;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      pdl_launch(kfn, grid, proj::THREADS, sm, stream, mx, mw, mxt, sexp, out, M, n, n_pad32,
                 nkb_res, tail, probe, k2_bands(tiles, grid), rin, rout);
    }
  } else if (P == 6) {
    auto kfn = bin ? proj::input_proj_kernel<6, true> : proj::input_proj_kernel<6, false>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, proj::Cfg<6>::SMEM);
    kfn<<<grid, proj::THREADS, proj::Cfg<6>::SMEM, stream>>>(mx, mw, sexp, out, M, n, n_pad32, nkb, rin, rout);
  } else if (P == 7) {
    auto kfn = bin ? proj::input_proj_kernel<7, true> : proj::input_proj_kernel<7, false>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, proj::Cfg<7>::SMEM);
    kfn<<<grid, proj::THREADS, proj::Cfg<7>::SMEM, stream>>>(mx, mw, sexp, out, M, n, n_pad32, nkb, rin, rout);
  } else {
    auto kfn = proj::input_proj_kernel<8, false>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, proj::Cfg<8>::SMEM);
    kfn<<<grid, proj::THREADS, proj::Cfg<8>::SMEM, stream>>>(mx, mw, sexp, out, M, n, n_pad32, nkb, rin, rout);
  }
  SPB_CHECK_LAUNCH("input_proj");
  return 0;
}
