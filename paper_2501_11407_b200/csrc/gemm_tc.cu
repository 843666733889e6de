// K5: factorised e-prop gradient GEMM on 5th-generation tensor cores (tcgen05 + TMA).
//
//   grad[i][j] += sum_K A[K][i] * B[K][j],   A = chunk coefficients C (M = n neurons)
//                                            B = xbar_t or raw spikes (N = k inputs)
//   both MN-major (neurons / channels contiguous, as K1s / K4 / the pack write them),
//   K = (sample, step) pairs of one time chunk (K = B*KR), so the LIF trace psi (x) xbar
//   (gradients.py:165-172, G_u = 1 (x) xbar) is never materialised per sample.
//
// fp32 accuracy from bf16 tensor cores: every operand is split x = hi + lo (bf16 each)
// and D += Ah*Bh + Ah*Bl + Al*Bh (the lo*lo term is below fp32 rounding of the sum); the
// raw-spike B is exact in bf16 (Bl = 0, 2 MMAs).
//
// Structure (CTA pairs, one 256 x 256 output tile per pair, split-K over blockIdx.z):
//   warp 0   TMA producer (both CTAs): own Ah, Al rows (128 x BK), half of the B columns
//            (128 x BK; Bh, and Bl unless exact), MN-major SWIZZLE_128B boxes, per stage,
//            transaction bytes on the leader's barrier
//   warp 1   TMEM allocation (cta_group::2) + on the leader the converged-warp
//            tcgen05.mma.cta_group::2 issue (M=256, N=256, K=16), commits multicast
//   warps 2-5 epilogue: tcgen05.ld 32x32b.x32 -> fp32 partial tile (fixed-order reduce later)
#include "tma.cuh"
#include <cudaTypedefs.h>
#include <mutex>

namespace spb {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 32;   // per CTA: 128 neurons x 256 inputs, 32-row K blocks
constexpr int TILE_A = BM * BK * 2;          // bytes
constexpr int THREADS = 192;

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;   // SBO
  d |= (uint64_t)1u << 46;             // descriptor version (sm100)
  d |= (uint64_t)2u << 61;             // SWIZZLE_128B
  return d;
}
// MN-major, SWIZZLE_128B: 64-element MN runs (128 B rows, one per K), 8-row K groups
// 1024 B apart (SBO), the second 64-element MN half 8 KB further (LBO).
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((64u * BK * 2u) >> 4) << 16;   // LBO: next 64-wide MN block (one box)
  d |= (uint64_t)(1024u >> 4) << 32;   // SBO: next 8-row K group
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// ------------------------------------------------------------------------------------
// Why pairs (round 2): a single-CTA 128 x 256 tile streams, per 32-row K block, 32 KB of
// operands (A hi/lo for 128 neurons, B for 256 inputs) into the SM; at the MMA peak that
// is ~8.6 KB/clk chip-wide, above the L2 (LTS) throughput (~6.3 KB/clk), and its tensor
// pipe idled ~25 % (ncu: 74 % active, C3 0.140 ms).  A pair stages, per CTA, its own 128
// A rows and HALF of the 256 B columns (24 KB per K block for the same 128 x 256 outputs
// per CTA): 25 % fewer operand bytes per output, tensor pipe 94 % active, C3 0.117 ms.
constexpr int P_BNH = BN / 2;                 // B columns staged per CTA
constexpr int P_TILE_B = P_BNH * BK * 2;      // 8 KB
constexpr int P_STAGES = 6, P_STAGES_NL = 8;
constexpr int P_STAGE = 2 * TILE_A + 2 * P_TILE_B, P_STAGE_NL = 2 * TILE_A + P_TILE_B;
constexpr int P_SMEM = P_STAGES * P_STAGE + 1024 + 256;
constexpr int P_SMEM_NL = P_STAGES_NL * P_STAGE_NL + 1024 + 256;
constexpr uint32_t P_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ void umma2_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(P_IDESC), "r"(acc));
}

template <bool BLO>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    grad_gemm_pair_kernel(const __grid_constant__ CUtensorMap tm_ah,
                          const __grid_constant__ CUtensorMap tm_al,
                          const __grid_constant__ CUtensorMap tm_bh,
                          const __grid_constant__ CUtensorMap tm_bl, int M, int K,
                          int kb_per_split, float* __restrict__ partial, int ldp,
                          long long slice_stride) {
  constexpr int NST = BLO ? P_STAGES : P_STAGES_NL;
  constexpr int SB = BLO ? P_STAGE : P_STAGE_NL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * SB);
  uint64_t* full = bars;                   // [NST] (the leader's is used)
  uint64_t* empty = bars + NST;            // [NST]
  uint64_t* tmem_full = bars + 2 * NST;    // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NST + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int m0 = blockIdx.y * (2 * BM) + (int)rank * BM;   // this CTA's neurons
  const int n0 = (blockIdx.x >> 1) * BN;                   // the pair's input columns
  const int nx = n0 + (int)rank * P_BNH;                   // B columns staged here
  const int nkb = (K + BK - 1) / BK;
  const int kb0 = blockIdx.z * kb_per_split;
  const int kb1 = min(nkb, kb0 + kb_per_split);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(tmem_full), 1);
    mbar_fence_init();
    tma_prefetch_desc(&tm_ah);
    tma_prefetch_desc(&tm_al);
    tma_prefetch_desc(&tm_bh);
    if (BLO) tma_prefetch_desc(&tm_bl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote complete_tx / commit
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
        const int s = it % NST;
        mbar_wait(smem_u32(&empty[s]), ((it / NST) & 1) ^ 1);
        if (leader) mbar_expect_tx(smem_u32(&full[s]), 2 * SB);
        const uint32_t fb = mapa(smem_u32(&full[s]), 0);
        const uint32_t st = smem_u32(smem + s * SB);
        tma_load_2sm(st, &tm_ah, fb, m0, kb * BK);
        tma_load_2sm(st + TILE_A / 2, &tm_ah, fb, m0 + 64, kb * BK);
        tma_load_2sm(st + TILE_A, &tm_al, fb, m0, kb * BK);
        tma_load_2sm(st + TILE_A + TILE_A / 2, &tm_al, fb, m0 + 64, kb * BK);
        tma_load_2sm(st + 2 * TILE_A, &tm_bh, fb, nx, kb * BK);
        tma_load_2sm(st + 2 * TILE_A + P_TILE_B / 2, &tm_bh, fb, nx + 64, kb * BK);
        if (BLO) {
          tma_load_2sm(st + 2 * TILE_A + P_TILE_B, &tm_bl, fb, nx, kb * BK);
          tma_load_2sm(st + 2 * TILE_A + P_TILE_B + P_TILE_B / 2, &tm_bl, fb, nx + 64, kb * BK);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // whole warp, converged; elect.sync picks the issuer
      for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
        const int s = it % NST;
        mbar_wait_cluster(smem_u32(&full[s]), (it / NST) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t st = smem_u32(smem + s * SB);
        const uint32_t sah = st, sal = st + TILE_A, sbh = st + 2 * TILE_A,
                       sbl = st + 2 * TILE_A + P_TILE_B;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint32_t off = kk * 2048;  // 16 K rows of the MN-major tiles
          const uint64_t dah = umma_desc_mn_sw128(sah + off), dal = umma_desc_mn_sw128(sal + off);
          const uint64_t dbh = umma_desc_mn_sw128(sbh + off), dbl = umma_desc_mn_sw128(sbl + off);
          umma2_bf16(tmem_base, dah, dbh, (kb > kb0 || kk > 0) ? 1u : 0u);
          if (BLO) umma2_bf16(tmem_base, dah, dbl, 1u);
          umma2_bf16(tmem_base, dal, dbh, 1u);
        }
        commit2(smem_u32(&empty[s]));
      }
      if (kb1 > kb0) commit2(smem_u32(tmem_full));
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quarter (warp % 4); this CTA's 128 rows x 256 cols
    const int q = warp & 3;
    const bool have_work = kb1 > kb0;
    const long long slice_rows = slice_stride / ldp;
    const bool own = m0 < slice_rows;    // rows past the slice belong to the next slice
    if (have_work) {
      mbar_wait(smem_u32(tmem_full), 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
            "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
            "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (!have_work) {
#pragma unroll
        for (int v = 0; v < 32; ++v) r[v] = 0u;
      }
      // 4x4 transpose of 32-byte chunks inside each group of 4 lanes, then 256-bit
      // stores: 8 rows x 128 contiguous bytes per instruction (rows past M are padding
      // rows of the partial slice, written as computed: zero A rows give zeros)
      const int p4 = lane & 3;
#pragma unroll
      for (int sh = 2; sh >= 1; sh >>= 1) {
        const bool up = (p4 & sh) != 0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          if (m & sh) continue;
          const int ms = m | sh;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t send = up ? r[8 * m + e] : r[8 * ms + e];
            const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, sh);
            if (up) r[8 * m + e] = recv; else r[8 * ms + e] = recv;
          }
        }
      }
      const int col = n0 + c0 + 8 * p4;
      float* base = partial + (long long)blockIdx.z * slice_stride +
                    (long long)(m0 + q * 32 + (lane & ~3)) * ldp + col;
      if (own && col < ldp) {
#pragma unroll
        for (int kq = 0; kq < 4; ++kq)
          asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(
                           base + (long long)kq * ldp),
                       "r"(r[8 * kq + 0]), "r"(r[8 * kq + 1]), "r"(r[8 * kq + 2]),
                       "r"(r[8 * kq + 3]), "r"(r[8 * kq + 4]), "r"(r[8 * kq + 5]),
                       "r"(r[8 * kq + 6]), "r"(r[8 * kq + 7])
                       : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the peer is done with the pair's TMEM and barriers
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(BN));
}

// 2-D bf16 MN-major operand [K][ld] (M contiguous) with 64 x 64 boxes, 128-byte swizzle.
static bool make_map_mn(CUtensorMap* map, const void* ptr, int M, int ld, int K) {
  return make_tmap_2d(map, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)M, (uint64_t)K,
                      (uint64_t)ld * 2, 64, BK, CU_TENSOR_MAP_SWIZZLE_128B);
}

}  // namespace tc

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_tmap_2d(CUtensorMap* map, const void* ptr, CUtensorMapDataType dtype, int elem_bytes,
                  uint64_t inner, uint64_t outer, uint64_t row_stride_bytes, uint32_t box_inner,
                  uint32_t box_outer, CUtensorMapSwizzle swizzle) {
  auto enc = get_encode();
  if (!enc) return false;
  (void)elem_bytes;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dtype, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace spb

using namespace spb;

extern "C" {

// Split-K tensor-core GEMM (grad_gemm_pair_kernel) writing fp32 partial tiles:
//   partial[z][i][j] = sum_{K in split z} (Ah+Al)[K][i] (Bh+Bl)[K][j]   (lo*lo dropped)
// bl = NULL: B is exact in bf16 (raw spikes), Bl = 0 -- 2 MMAs per step instead of 3.
// Every one of the `splits` slices is written for rows < round_up(M, 128), columns < ldp
// (empty K ranges give 0); each split runs on 2 * ceil(ldp / 256) * ceil(M / 256) CTAs.
// The slice must hold whole 128-row tiles and 32-byte rows (slice_stride >=
// round_up(M, 128) * ldp, ldp % 8 == 0).  Reduced in fixed order by spb_reduce_partials.
int spb_grad_gemm_partials(const void* ah, const void* al, int lda, const void* bh,
                                const void* bl, int ldb, int M, int N_rows, int K, int splits,
                                float* partial, int ldp, long long slice_stride,
                                cudaStream_t stream) {
  SPB_CHECK_ARG(ah && al && bh && partial, "spb_grad_gemm_partials: null pointer");
  const bool blo = bl != nullptr;
  SPB_CHECK_ARG(M > 0 && N_rows > 0 && K > 0 && splits > 0 && ldp >= 8 && ldp % 8 == 0 &&
                    lda >= M && lda % 8 == 0 && ldb >= N_rows && ldb % 8 == 0 &&
                    slice_stride >= (long long)ceil_div(M, tc::BM) * tc::BM * ldp,
                "spb_grad_gemm_partials: bad sizes M=%d lda=%d N=%d K=%d ldp=%d", M, lda,
                N_rows, K, ldp);
  SPB_CHECK_ARG((reinterpret_cast<uintptr_t>(ah) | reinterpret_cast<uintptr_t>(al) |
                 reinterpret_cast<uintptr_t>(bh) | reinterpret_cast<uintptr_t>(bl)) % 16 == 0,
                "spb_grad_gemm_partials: operands must be 16-byte aligned");
  CUtensorMap mah, mal, mbh, mbl;
  if (!tc::make_map_mn(&mah, ah, M, lda, K) || !tc::make_map_mn(&mal, al, M, lda, K) ||
      !tc::make_map_mn(&mbh, bh, N_rows, ldb, K) ||
      !tc::make_map_mn(&mbl, blo ? bl : bh, N_rows, ldb, K)) {
    set_error("spb_grad_gemm_partials: cuTensorMapEncodeTiled failed");
    return 3;
  }
  const int nkb = ceil_div(K, tc::BK);
  const int kbps = ceil_div(nkb, splits);
  dim3 grid(2 * ceil_div(ldp, tc::BN), ceil_div(M, 2 * tc::BM), splits);
  if (blo) {
    cudaFuncSetAttribute(tc::grad_gemm_pair_kernel<true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, tc::P_SMEM);
    pdl_launch(tc::grad_gemm_pair_kernel<true>, grid, tc::THREADS, tc::P_SMEM, stream,
        mah, mal, mbh, mbl, M, K, kbps, partial, ldp, slice_stride);
  } else {
    cudaFuncSetAttribute(tc::grad_gemm_pair_kernel<false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, tc::P_SMEM_NL);
    pdl_launch(tc::grad_gemm_pair_kernel<false>, grid, tc::THREADS, tc::P_SMEM_NL, stream,
        mah, mal, mbh, mbl, M, K, kbps, partial, ldp, slice_stride);
  }
  SPB_CHECK_LAUNCH("grad_gemm_pair");
  return 0;
}

}  // extern "C"
