// K21: fused exact input projection + neuron dynamics (sm_100a).
//
// K2 (proj.cu) computes the exact current I = W x_t on the INT8 tensor cores and K1
// (forward.cu) integrates the LIF/ALIF dynamics from it; run separately, the fp64
// current [B*Tc][n] makes a full HBM round trip (8n bytes written and read per
// sample-step -- more than the spikes, the weights and every other operand together).
// This kernel keeps it on chip: the MMA tile is (128 SAMPLES at one time step) x (P
// digit slices x NT neurons), i.e. the spike operand is time-major (row t*B + b), so the
// epilogue thread that owns a sample row integrates its neurons' state in registers from
// one time step to the next while the tensor cores already accumulate the next step into
// the other TMEM buffer.  The recurrence never crosses threads.
//
// Reference semantics (identical arithmetic to K2 + K1, so spikes are the same bits):
//   I      -- `net.neuron.w @ x_t` (gradients.py:125): P signed 7-bit weight digits,
//             exact int32 tensor-core sums, exact int64 recombination, one fp64 rounding
//   state  -- _step_state (gradients.py:118-129) in fp64 with explicit round-to-nearest
//             operations in the reference's order; spike = heaviside / surrogate_smooth
//             (graph.py:45-52); psi = surrogate_grad (graph.py:40-42) in fp32
//   pass A -- readout spike filter zbar/zsum (gradients.py:173-174), bit raster
//   psi    -- parked for the backward chunk scan (forward.cu K1s) when requested
//
// Work unit = (128-sample block, NT-neuron tile) for all steps of the chunk; persistent
// CTAs walk units.  Warp 0: TMA producer (the unit's weight digits once, resident in
// smem; one 16 KB spike tile per K block and step through an XS-deep ring).  Warp 1: TMEM
// owner + tcgen05.mma.kind::i8 issuer (double-buffered accumulators).  Warps 2..: epilogue,
// thread = (sample row, 4 neurons).
#include "tma.cuh"
#include "digits.cuh"

namespace spb {
namespace fused {

constexpr int BM = 128;     // samples per tile (TMEM lanes)
constexpr int BK = 128;     // K bytes per stage (one 128-byte swizzle row)
constexpr int NPT = 4;      // neurons per epilogue thread
constexpr int TILE_X = BM * BK;
constexpr int MAXKB = 6;    // Kpad <= 768 (weights of a neuron tile resident in smem)

template <int P, int NT, int XS>
struct Cfg {
  static constexpr int N = P * NT;                       // MMA N
  static constexpr int WBLK = N * BK;
  static constexpr int W_BYTES = MAXKB * WBLK;
  static constexpr int EPI_WARPS = 4 * (NT / NPT);
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int ABUF = N <= 128 ? 128 : 256;      // TMEM columns per accumulator
  static constexpr int TMEM_COLS = 2 * ABUF;
  static constexpr int SMEM = W_BYTES + XS * TILE_X + 1024 + 256;
  // kind::i8: D s32, A u8 (spikes), B s8 (digits), both K-major
  static constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (1u << 10) |
                                    ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  static_assert(N % 16 == 0 && N <= 256, "bad MMA N");
};

struct FusedParams {
  int B, n, n_pad32, Tc, KR, len, t0, T, nkb, pass;  // pass 0 = A, 1 = B (psi only)
  double alpha, theta, slope, beta, rho, kappa;
  int reset, smooth, sblocks;
  int probe;  // profiling probe: bit 0 = skip the dynamics, bit 1 = skip psi stores
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
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, int32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ double pow2(int e) {
  return __longlong_as_double((long long)(e + 1023) << 52);
}
// z = spike(d): Theta(d) = [d >= 0] or surrogate_smooth(d) (graph.py:45-52)
__device__ __forceinline__ double spike_value(double d, bool smooth, double slope) {
  if (!smooth) return d >= 0.0 ? 1.0 : 0.0;
  return __dadd_rn(0.5, __ddiv_rn(d, __dadd_rn(1.0, __dmul_rn(slope, fabs(d)))));
}

template <int P, int NT, int XS, bool ALIF>
__global__ void __launch_bounds__(Cfg<P, NT, XS>::THREADS, 1)
    fused_forward_kernel(const __grid_constant__ CUtensorMap tm_x,
                         const __grid_constant__ CUtensorMap tm_w, const int* __restrict__ sexp,
                         FusedParams F, double* __restrict__ u_st, double* __restrict__ a_st,
                         double* __restrict__ zbar_st, double* __restrict__ zsum_st,
                         uint8_t* __restrict__ raster, float* __restrict__ psis) {
  using C = Cfg<P, NT, XS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* wsm = smem;                   // [nkb][P*NT rows][128 B]
  uint8_t* xsm = smem + C::W_BYTES;      // [XS][128 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xsm + XS * TILE_X);
  uint64_t* xfull = bars;
  uint64_t* xempty = bars + XS;
  uint64_t* tfull = bars + 2 * XS;
  uint64_t* tempty = bars + 2 * XS + 2;
  uint64_t* wfull = bars + 2 * XS + 4;
  uint64_t* wempty = bars + 2 * XS + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * XS + 6);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (F.n + NT - 1) / NT;
  const int nunits = ntiles * F.sblocks;
  const int len = F.len, nkb = F.nkb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < XS; ++s) {
      mbar_init(smem_u32(&xfull[s]), 1);
      mbar_init(smem_u32(&xempty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), C::EPI_WARPS);
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
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0, wl = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int nt = u / F.sblocks, sb = u % F.sblocks;
        mbar_wait(smem_u32(wempty), (wl & 1) ^ 1);  // previous unit's MMAs are done
        const uint32_t fb = smem_u32(wfull);
        mbar_expect_tx(fb, nkb * C::WBLK);
        for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
          for (int p = 0; p < P; ++p)
            tma_load_2d(smem_u32(wsm + kb * C::WBLK + p * NT * BK), &tm_w, fb, kb * BK,
                        p * F.n_pad32 + nt * NT);
        ++wl;
        for (int t = 0; t < len; ++t) {
          const int row = t * F.B + sb * BM;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % XS;
            mbar_wait(smem_u32(&xempty[s]), ((it / XS) & 1) ^ 1);
            const uint32_t xb = smem_u32(&xfull[s]);
            mbar_expect_tx(xb, TILE_X);
            tma_load_2d(smem_u32(xsm + s * TILE_X), &tm_x, xb, kb * BK, row);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp runs the issue loop (converged); elect.sync picks the issuer
      int it = 0, lt = 0, wl = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        mbar_wait(smem_u32(wfull), wl & 1);
        ++wl;
        for (int t = 0; t < len; ++t, ++lt) {
          const int a = lt & 1;
          mbar_wait(smem_u32(&tempty[a]), ((lt >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t dacc = tmem_base + (uint32_t)(a * C::ABUF);
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % XS;
            mbar_wait(smem_u32(&xfull[s]), (it / XS) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t xa = smem_u32(xsm + s * TILE_X);
            const uint32_t wa = smem_u32(wsm + kb * C::WBLK);
#pragma unroll
            for (int kk = 0; kk < BK / 32; ++kk)
              mma_i8(dacc, desc_k_sw128(xa + kk * 32), desc_k_sw128(wa + kk * 32), C::IDESC,
                     (kb | kk) ? 1u : 0u);
            commit(smem_u32(&xempty[s]));
          }
          commit(smem_u32(&tfull[a]));
        }
        commit(smem_u32(wempty));
      }
    }
  } else {
    const int q = warp & 3;               // TMEM lane quarter of this warp
    const int g = (warp - 2) >> 2;        // 8-neuron group of the tile
    const int r = q * 32 + lane;          // sample row of the tile
    const bool smooth = F.smooth != 0;
    const double theta = F.theta, beta = F.beta, slope = F.slope;
    const float slope_f = (float)F.slope;
    const int nw = (F.n + 31) >> 5;  // raster words per (sample, step)
    unsigned int* raster32 = reinterpret_cast<unsigned int*>(raster);
    int lt = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int nt = u / F.sblocks, sb = u % F.sblocks;
      const int b = sb * BM + r;
      const bool vb = b < F.B;
      const int i0 = nt * NT + g * NPT;
      int se[NPT];
      // fp64 state in registers across the whole chunk; dp = drive d of the previous
      // step (the reference re-evaluates the same expression, gradients.py:159)
      double us[NPT], as[NPT], zb[NPT], zs[NPT], dp[NPT];
#pragma unroll
      for (int c = 0; c < NPT; ++c) {
        const int i = i0 + c;
        const bool v = vb && i < F.n;
        se[c] = (i < F.n) ? __ldg(sexp + i) : 0;
        const long long bi = (long long)b * F.n + i;
        us[c] = (v && F.t0 > 0) ? u_st[bi] : 0.0;
        as[c] = (ALIF && v && F.t0 > 0) ? a_st[bi] : 0.0;
        zb[c] = (v && F.t0 > 0 && F.pass == 0) ? zbar_st[bi] : 0.0;
        zs[c] = (v && F.t0 > 0 && F.pass == 0) ? zsum_st[bi] : 0.0;
        dp[c] = ALIF ? __dsub_rn(__dsub_rn(us[c], theta), __dmul_rn(beta, as[c]))
                     : __dsub_rn(us[c], theta);
      }
      float* prow = (psis != nullptr && vb) ? psis + (long long)b * (F.KR + 1) * F.n + i0 : nullptr;
      const bool vec = (F.n & 3) == 0 && i0 + NPT <= F.n;
      if (prow != nullptr) {  // psi_{t0-1}
        float p0[NPT];
#pragma unroll
        for (int c = 0; c < NPT; ++c) p0[c] = surrogate_grad_f32((float)dp[c], slope_f);
        if (vec) {
          *reinterpret_cast<float4*>(prow) = make_float4(p0[0], p0[1], p0[2], p0[3]);
        } else {
#pragma unroll
          for (int c = 0; c < NPT; ++c)
            if (i0 + c < F.n) prow[c] = p0[c];
        }
      }
      for (int t = 0; t < len; ++t, ++lt) {
        const int a = lt & 1;
        mbar_wait(smem_u32(&tfull[a]), (lt >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * C::ABUF + g * NPT);
        int32_t dg[P][NPT];
#pragma unroll
        for (int p = 0; p < P; ++p) tmem_ld4(tb + p * NT, dg[p]);
        tmem_wait_ld();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive(smem_u32(&tempty[a]));
        uint32_t bits = 0;
        float psi[NPT];
        if (F.probe & 1) {
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < NPT; ++c)
#pragma unroll
            for (int p = 0; p < P; ++p) acc += (float)dg[p][c];
          if (acc == 1.2345f) psis[0] = acc;  // keep the loads live
          continue;
        }
#pragma unroll
        for (int c = 0; c < NPT; ++c) {
          // exact recombination of the digit sums (as proj_epilogue_tile)
          const long long g0 = digits_g0<P>(dg[0][c], dg[1][c], dg[2][c]);
          long long g1 = dg[3][c];
#pragma unroll
          for (int p = 4; p < P; ++p) g1 = (g1 << Digits<P>::RB) + dg[p][c];
          const double I = digits_current<P, false>(g0, g1, se[c]);
          // gradients.py:121-129 (LIF: beta = rho = 0, so d = u - theta exactly)
          const double z_prev = spike_value(dp[c], smooth, slope);
          if (ALIF) as[c] = __dadd_rn(__dmul_rn(F.rho, as[c]), z_prev);
          us[c] = __dadd_rn(__dmul_rn(F.alpha, us[c]), I);
          if (F.reset) us[c] = __dsub_rn(us[c], __dmul_rn(theta, z_prev));
          const double d = ALIF ? __dsub_rn(__dsub_rn(us[c], theta), __dmul_rn(beta, as[c]))
                                : __dsub_rn(us[c], theta);
          if (F.pass == 0) {
            const double zv = spike_value(d, smooth, slope);
            zb[c] = __dadd_rn(__dmul_rn(F.kappa, zb[c]), zv);
            zs[c] = __dadd_rn(zs[c], zb[c]);
            bits |= (zv > 0.5 && i0 + c < F.n) ? (1u << c) : 0u;
          }
          psi[c] = surrogate_grad_f32((float)d, slope_f);
          dp[c] = d;
        }
        if (vb) {
          // raster: 4 bits of a 32-neuron word per thread (zero-initialised by the host)
          if (F.pass == 0 && raster32 != nullptr && bits)
            atomicOr(raster32 + ((long long)b * F.T + F.t0 + t) * nw + (i0 >> 5),
                     bits << (i0 & 31));
          if (prow != nullptr && !(F.probe & 2)) {
            float* pr = prow + (long long)(t + 1) * F.n;
            if (vec) {
              *reinterpret_cast<float4*>(pr) = make_float4(psi[0], psi[1], psi[2], psi[3]);
            } else {
#pragma unroll
              for (int c = 0; c < NPT; ++c)
                if (i0 + c < F.n) pr[c] = psi[c];
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NPT; ++c) {
        const int i = i0 + c;
        if (vb && i < F.n) {
          const long long bi = (long long)b * F.n + i;
          u_st[bi] = us[c];
          a_st[bi] = as[c];
          if (F.pass == 0) {
            zbar_st[bi] = zb[c];
            zsum_st[bi] = zs[c];
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
}

template <int P, int NT, int XS, bool ALIF>
static int launch(const CUtensorMap& mx, const CUtensorMap& mw, const int* sexp,
                  const FusedParams& F, double* u, double* a, double* zbar, double* zsum,
                  uint8_t* raster, float* psis, int grid, cudaStream_t stream) {
  using C = Cfg<P, NT, XS>;
  auto kfn = fused_forward_kernel<P, NT, XS, ALIF>;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  kfn<<<grid, C::THREADS, C::SMEM, stream>>>(mx, mw, sexp, F, u, a, zbar, zsum, raster, psis);
  return 0;
}

}  // namespace fused
}  // namespace spb

using namespace spb;

extern "C" {

int spb_fused_forward_probe(int pass, const uint8_t* xq, const int8_t* wq, const int* sexp, int B,
                            int n, int n_pad32, int Kpad, int P, int Tc, int KR, int len, int t0,
                            int T, double alpha, double theta, double slope, double beta,
                            double rho, double kappa, int reset, int smooth, double* u, double* a,
                            double* zbar, double* zsum, uint8_t* raster, float* psi_scratch,
                            int sm_count, int probe, cudaStream_t stream);

int spb_fused_forward(int pass, const uint8_t* xq, const int8_t* wq, const int* sexp, int B,
                      int n, int n_pad32, int Kpad, int P, int Tc, int KR, int len, int t0, int T,
                      double alpha, double theta, double slope, double beta, double rho,
                      double kappa, int reset, int smooth, double* u, double* a, double* zbar,
                      double* zsum, uint8_t* raster, float* psi_scratch, int sm_count,
                      cudaStream_t stream) {
  return spb_fused_forward_probe(pass, xq, wq, sexp, B, n, n_pad32, Kpad, P, Tc, KR, len, t0, T,
                                 alpha, theta, slope, beta, rho, kappa, reset, smooth, u, a, zbar,
                                 zsum, raster, psi_scratch, sm_count, 0, stream);
}

// spb_fused_forward with a profiling probe (see FusedParams::probe); probe = 0 is the
// production kernel.
int spb_fused_forward_probe(int pass, const uint8_t* xq, const int8_t* wq, const int* sexp, int B,
                            int n, int n_pad32, int Kpad, int P, int Tc, int KR, int len, int t0,
                            int T, double alpha, double theta, double slope, double beta,
                            double rho, double kappa, int reset, int smooth, double* u, double* a,
                            double* zbar, double* zsum, uint8_t* raster, float* psi_scratch,
                            int sm_count, int probe, cudaStream_t stream) {
  constexpr int nt_width = 16;  // neurons per unit: N = 7*16 = 112 (P = 7) / 128 (P = 8)
  SPB_CHECK_ARG(pass == 0 || pass == 1, "spb_fused_forward: pass must be 0 (A) or 1 (B)");
  SPB_CHECK_ARG(xq && wq && sexp && u && a, "spb_fused_forward: null pointer");
  SPB_CHECK_ARG(pass == 1 || (zbar && zsum), "spb_fused_forward: pass A needs zbar/zsum");
  SPB_CHECK_ARG(pass == 0 || psi_scratch, "spb_fused_forward: pass B needs psi_scratch");
  SPB_CHECK_ARG(B > 0 && n > 0 && n_pad32 >= n && n_pad32 % 32 == 0 && Kpad % fused::BK == 0 &&
                    Kpad / fused::BK <= fused::MAXKB && (P >= 6 && P <= 8) && len >= 1 &&
                    len <= Tc && KR >= Tc + 1 && t0 >= 0 && t0 + len <= T,
                "spb_fused_forward: bad sizes (Kpad <= %d, P in {7,8})", fused::MAXKB * fused::BK);
  SPB_CHECK_ARG((reinterpret_cast<uintptr_t>(xq) | reinterpret_cast<uintptr_t>(wq)) % 16 == 0,
                "spb_fused_forward: operands must be 16-byte aligned");
  CUtensorMap mx, mw;
  const bool ok =
      make_tmap_2d(&mx, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, (uint64_t)Tc * B, Kpad,
                   fused::BK, fused::BM, CU_TENSOR_MAP_SWIZZLE_128B) &&
      make_tmap_2d(&mw, wq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, (uint64_t)P * n_pad32, Kpad,
                   fused::BK, nt_width, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!ok) {
    set_error("spb_fused_forward: cuTensorMapEncodeTiled failed");
    return 3;
  }
  fused::FusedParams F{B, n, n_pad32, Tc, KR, len, t0, T, Kpad / fused::BK, pass,
                       alpha, theta, slope, beta, rho, kappa, reset, smooth,
                       (B + fused::BM - 1) / fused::BM, probe};
  const int units = F.sblocks * ((n + nt_width - 1) / nt_width);
  const int grid = max(1, min(units, sm_count > 0 ? sm_count : 148));
  const bool alif = beta != 0.0 || rho != 0.0;  // LIF runs with beta = rho = 0
  if (P == 8 && alif)
    fused::launch<8, 16, 7, true>(mx, mw, sexp, F, u, a, zbar, zsum, raster, psi_scratch, grid, stream);
  else if (P == 8)
    fused::launch<8, 16, 7, false>(mx, mw, sexp, F, u, a, zbar, zsum, raster, psi_scratch, grid, stream);
  else if (P == 7 && alif)
    fused::launch<7, 16, 8, true>(mx, mw, sexp, F, u, a, zbar, zsum, raster, psi_scratch, grid, stream);
  else if (P == 7)
    fused::launch<7, 16, 8, false>(mx, mw, sexp, F, u, a, zbar, zsum, raster, psi_scratch, grid, stream);
  else if (alif)
    fused::launch<6, 16, 8, true>(mx, mw, sexp, F, u, a, zbar, zsum, raster, psi_scratch, grid, stream);
  else
    fused::launch<6, 16, 8, false>(mx, mw, sexp, F, u, a, zbar, zsum, raster, psi_scratch, grid, stream);
  SPB_CHECK_LAUNCH("fused_forward");
  return 0;
}

}  // extern "C"
