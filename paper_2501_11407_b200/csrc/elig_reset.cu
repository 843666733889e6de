// K6r: the per-synapse trace PAIR of ALIF with reset=True carried across time chunks on
// tcgen05 tensor cores (sm_100a).
//
// Reference: eprop_trace_update (gradients.py:89-94) with the ALIF block of the reset
// model (neurons.py:266-271 / test_neurons.py:144-155):
//   G_u' = (alpha - theta psi^-) G_u + theta beta psi^- G_a + x_t
//   G_a' = psi^- G_u + (rho - beta psi^-) G_a
// and the eligibility x_step = psi (G_u - beta G_a) (gradients.py:165-169).  With the
// chunk coefficients of the reset scan (forward.cu, K1r) a chunk of L steps is
//   E_end[b,i,:] = Dt[b,i] E0[b,i,:] + sum_rho W_rho[b,i] x_rho[b,:]   (2x2 Dt, W = (W_u, W_a))
//   grad[i,:]   += sum_b (M_u E0_u + M_a E0_a)[b,i,:]
// (the intra-chunk terms go through the chunk-gradient GEMM K5 on the raw input).  Both
// traces are read once and written once per chunk; the per-sample GEMMs D_u = W_u^T x and
// D_a = W_a^T x run on the tensor cores.  x is an integer count, exact in bf16, so the
// split needs only hi*x + lo*x (2 MMAs per trace).
//
// One CTA = 128 neurons x 64 inputs x a contiguous sample range.  Warp 0: TMA producer
// (per sample: both E0 tiles, double-buffered; per K block: W_u hi/lo, W_a hi/lo, x, 2-stage
// ring).  Warp 1: TMEM owner + MMA issuer (accumulators [buffer][trace] x 64 columns).
// Warps 2-17: epilogue (TMEM lane quarter x 16-column group), gradient in registers.
#include "tma.cuh"

namespace spb {
namespace rcarry {

constexpr int BM = 128, BN = 64, BK = 32, STAGES = 2;
constexpr int TW = BM * BK * 2;                 // 8 KB: one W operand tile (two 64-wide boxes)
constexpr int TX = BN * BK * 2;                 // 4 KB: x tile (one 64-wide box)
constexpr int STAGE = 4 * TW + TX;              // W_u hi/lo, W_a hi/lo, x
constexpr int ETR = BM * BN * 4;                // 32 KB: one trace's E0 tile (2 boxes of 32 cols)
constexpr int ESET = 2 * ETR;                   // both traces
constexpr int EPI_WARPS = 16;
constexpr int THREADS = 64 + EPI_WARPS * 32;
constexpr int SMEM = 2 * ESET + STAGES * STAGE + 1024 + 256;
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&r)[16]) {
  uint32_t* v = reinterpret_cast<uint32_t*>(r);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    reset_carry_kernel(const __grid_constant__ CUtensorMap tm_uh, const __grid_constant__ CUtensorMap tm_ul,
                       const __grid_constant__ CUtensorMap tm_ah, const __grid_constant__ CUtensorMap tm_al,
                       const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_eu,
                       const __grid_constant__ CUtensorMap tm_ea, const float4* __restrict__ coef,
                       float* __restrict__ eps_u, float* __restrict__ eps_a,
                       float* __restrict__ partial, int B, int n, int n_pad, int ke, int kp, int KR,
                       int b_per_split, int do_mma, int load_eps, int store_eps) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* esm = smem;                             // [2 buffers][2 traces][2 boxes][128][128 B]
  uint8_t* osm = smem + 2 * ESET;                  // [STAGES][W_u h, W_u l, W_a h, W_a l, x]
  uint64_t* bars = reinterpret_cast<uint64_t*>(osm + STAGES * STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint64_t* efull = bars + 2 * STAGES + 4;
  uint64_t* eempty = bars + 2 * STAGES + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
  const int b0 = blockIdx.z * b_per_split;
  const int nb = max(0, min(B, b0 + b_per_split) - b0);
  const int nkb = KR / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), EPI_WARPS);
      mbar_init(smem_u32(&efull[a]), 1);
      mbar_init(smem_u32(&eempty[a]), EPI_WARPS);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int lb = 0; lb < nb; ++lb) {
        const int b = b0 + lb;
        if (load_eps) {
          const int eb = lb & 1;
          mbar_wait(smem_u32(&eempty[eb]), ((lb >> 1) & 1) ^ 1);
          const uint32_t fb = smem_u32(&efull[eb]);
          mbar_expect_tx(fb, ESET);
          const uint32_t e0 = smem_u32(esm + eb * ESET);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            tma_load_2d(e0 + q * (ETR / 2), &tm_eu, fb, j0 + 32 * q, b * n_pad + i0);
            tma_load_2d(e0 + ETR + q * (ETR / 2), &tm_ea, fb, j0 + 32 * q, b * n_pad + i0);
          }
        }
        if (do_mma) {
          const int kbase = b * KR;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(smem_u32(&empty[s]), ((it / STAGES) & 1) ^ 1);
            const uint32_t st = smem_u32(osm + s * STAGE);
            const uint32_t fb = smem_u32(&full[s]);
            mbar_expect_tx(fb, STAGE);
            const int kr = kbase + kb * BK;
            const CUtensorMap* wm[4] = {&tm_uh, &tm_ul, &tm_ah, &tm_al};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              tma_load_2d(st + q * TW, wm[q], fb, i0, kr);
              tma_load_2d(st + q * TW + TW / 2, wm[q], fb, i0 + 64, kr);
            }
            tma_load_2d(st + 4 * TW, &tm_x, fb, j0, kr);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (do_mma) {  // whole warp, converged; elect.sync picks the issuer
      int it = 0;
      for (int lb = 0; lb < nb; ++lb) {
        const int a = lb & 1;
        mbar_wait(smem_u32(&tempty[a]), ((lb >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t du = tmem_base + (uint32_t)((a * 2 + 0) * BN);
        const uint32_t da = tmem_base + (uint32_t)((a * 2 + 1) * BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(smem_u32(&full[s]), (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = smem_u32(osm + s * STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint32_t off = kk * 2048;
            const uint64_t dx = desc_mn_sw128(st + 4 * TW + off, TX);
            const uint32_t first = (kb | kk) ? 1u : 0u;
            mma_bf16(du, desc_mn_sw128(st + 0 * TW + off, TW / 2), dx, first);
            mma_bf16(du, desc_mn_sw128(st + 1 * TW + off, TW / 2), dx, 1u);
            mma_bf16(da, desc_mn_sw128(st + 2 * TW + off, TW / 2), dx, first);
            mma_bf16(da, desc_mn_sw128(st + 3 * TW + off, TW / 2), dx, 1u);
          }
          commit(smem_u32(&empty[s]));
        }
        commit(smem_u32(&tfull[a]));
      }
    }
  } else {
    const int q = warp & 3;             // TMEM lane quarter
    const int cg = (warp - 2) >> 2;     // 16-column group
    const int r = q * 32 + lane;        // tile-local neuron
    const int i = i0 + r;
    const bool vi = i < n;
    const int c0 = j0 + cg * 16;
    const int box = cg >> 1, ch0 = (cg & 1) * 4;  // E0 box and first 16-byte chunk
    float g[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) g[c] = 0.f;
    for (int lb = 0; lb < nb; ++lb) {
      const int b = b0 + lb;
      const int a = lb & 1;
      const int eb = lb & 1;
      float4 k0 = make_float4(0.f, 0.f, 0.f, 0.f), k1 = k0;
      if (vi) {
        k0 = coef[((long long)b * n + i) * 2];      // M_u, M_a, Dt_uu, Dt_ua
        k1 = coef[((long long)b * n + i) * 2 + 1];  // Dt_au, Dt_aa
      }
      const uint32_t eu_row = smem_u32(esm + eb * ESET + box * (ETR / 2) + r * 128);
      const uint32_t ea_row = eu_row + ETR;
      if (load_eps) mbar_wait(smem_u32(&efull[eb]), (lb >> 1) & 1);
      float Du[16], Da[16];
      if (do_mma) {
        mbar_wait(smem_u32(&tfull[a]), (lb >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16);
        tmem_ld16(tl + (uint32_t)((a * 2 + 0) * BN + cg * 16), Du);
        tmem_ld16(tl + (uint32_t)((a * 2 + 1) * BN + cg * 16), Da);
        tmem_wait_ld();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive(smem_u32(&tempty[a]));
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) Du[c] = Da[c] = 0.f;
      }
      float* gu = eps_u + ((long long)b * n_pad + i) * ke + c0;
      float* ga = eps_a + ((long long)b * n_pad + i) * ke + c0;
#pragma unroll
      for (int v4 = 0; v4 < 4; ++v4) {
        float4 eu = make_float4(0.f, 0.f, 0.f, 0.f), ea = eu;
        if (load_eps) {  // SWIZZLE_128B: chunk c of row r at c ^ (r & 7)
          const int chk = (ch0 + v4) ^ (r & 7);
          eu = lds_f4(eu_row + (chk << 4));
          ea = lds_f4(ea_row + (chk << 4));
        }
        const float e_u[4] = {eu.x, eu.y, eu.z, eu.w}, e_a[4] = {ea.x, ea.y, ea.z, ea.w};
        float nu[4], na[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          g[v4 * 4 + c] = fmaf(k0.y, e_a[c], fmaf(k0.x, e_u[c], g[v4 * 4 + c]));
          nu[c] = fmaf(k0.w, e_a[c], fmaf(k0.z, e_u[c], Du[v4 * 4 + c]));
          na[c] = fmaf(k1.y, e_a[c], fmaf(k1.x, e_u[c], Da[v4 * 4 + c]));
        }
        if (store_eps && vi && c0 + v4 * 4 < ke) {
          *reinterpret_cast<float4*>(gu + v4 * 4) = make_float4(nu[0], nu[1], nu[2], nu[3]);
          *reinterpret_cast<float4*>(ga + v4 * 4) = make_float4(na[0], na[1], na[2], na[3]);
        }
      }
      __syncwarp();
      if (load_eps && lane == 0) arrive(smem_u32(&eempty[eb]));
    }
    if (vi) {
      float* prow = partial + ((long long)blockIdx.z * n_pad + i) * kp + c0;
#pragma unroll
      for (int v4 = 0; v4 < 4; ++v4)
        if (c0 + v4 * 4 < kp)
          *reinterpret_cast<float4*>(prow + v4 * 4) =
              make_float4(g[v4 * 4], g[v4 * 4 + 1], g[v4 * 4 + 2], g[v4 * 4 + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256));
}

}  // namespace rcarry
}  // namespace spb

using namespace spb;

extern "C" {

int spb_reset_carry_chunk(const void* wu_hi, const void* wu_lo, const void* wa_hi,
                          const void* wa_lo, int ldw, const void* xh, const float* coef,
                          float* eps_u, float* eps_a, float* partial, int B, int n, int n_pad,
                          int k, int ke, int kp, int KR, int splits, int do_mma, int load_eps,
                          int store_eps, cudaStream_t stream) {
  SPB_CHECK_ARG(coef && eps_u && eps_a && partial, "spb_reset_carry_chunk: null pointer");
  SPB_CHECK_ARG(!do_mma || (wu_hi && wu_lo && wa_hi && wa_lo && xh),
                "spb_reset_carry_chunk: missing GEMM operands");
  SPB_CHECK_ARG(n_pad % rcarry::BM == 0 && n <= n_pad && kp % 128 == 0 && kp >= k && ke >= k &&
                    ke % 4 == 0 && KR % rcarry::BK == 0,
                "spb_reset_carry_chunk: bad padding (n_pad %% 128, kp %% 128, ke %% 4, KR %% 32)");
  SPB_CHECK_ARG(B > 0 && splits > 0 && splits <= B, "spb_reset_carry_chunk: bad split");
  SPB_CHECK_ARG(!do_mma || (ldw >= n && ldw % 8 == 0), "spb_reset_carry_chunk: bad ldw");
  SPB_CHECK_ARG(!(store_eps && !do_mma), "spb_reset_carry_chunk: storing the trace needs the GEMM");
  CUtensorMap muh{}, mul{}, mah{}, mal{}, mx{}, meu{}, mea{};
  if (load_eps) {
    const bool ok =
        make_tmap_2d(&meu, eps_u, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ke, (uint64_t)B * n_pad,
                     (uint64_t)ke * 4, 32, rcarry::BM, CU_TENSOR_MAP_SWIZZLE_128B) &&
        make_tmap_2d(&mea, eps_a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ke, (uint64_t)B * n_pad,
                     (uint64_t)ke * 4, 32, rcarry::BM, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!ok) {
      set_error("spb_reset_carry_chunk: cuTensorMapEncodeTiled (eps) failed");
      return 3;
    }
  }
  if (do_mma) {
    const uint64_t K = (uint64_t)B * KR;
    const void* wp[4] = {wu_hi, wu_lo, wa_hi, wa_lo};
    CUtensorMap* wmap[4] = {&muh, &mul, &mah, &mal};
    bool ok = true;
    for (int q = 0; q < 4; ++q)
      ok = ok && make_tmap_2d(wmap[q], wp[q], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n, K,
                              (uint64_t)ldw * 2, 64, rcarry::BK, CU_TENSOR_MAP_SWIZZLE_128B);
    ok = ok && make_tmap_2d(&mx, xh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kp, K, (uint64_t)kp * 2,
                            64, rcarry::BK, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!ok) {
      set_error("spb_reset_carry_chunk: cuTensorMapEncodeTiled failed");
      return 3;
    }
  }
  const int bps = ceil_div(B, splits);
  cudaFuncSetAttribute(rcarry::reset_carry_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       rcarry::SMEM);
  dim3 grid(kp / rcarry::BN, n_pad / rcarry::BM, splits);
  rcarry::reset_carry_kernel<<<grid, rcarry::THREADS, rcarry::SMEM, stream>>>(
      muh, mul, mah, mal, mx, meu, mea, reinterpret_cast<const float4*>(coef), eps_u, eps_a,
      partial, B, n, n_pad, ke, kp, KR, bps, do_mma, load_eps, store_eps);
  SPB_CHECK_LAUNCH("reset_carry");
  return 0;
}

}  // extern "C"
