// Forward-side kernels of the e-prop update (sm_100a):
//   K1  spb_forward_chunk   -- LIF/ALIF dynamics + surrogate over a time chunk from the
//                              exact input current of K2 (proj.cu).
//                              pass A: spike raster, readout filter zsum.
//                              pass B: learning-signal-weighted surrogate and, by a
//                              backward scan over the chunk, the chunk-level
//                              eligibility coefficients consumed by the tensor cores.
//   K4  spb_xbar_chunk      -- presynaptic filter xbar_t = alpha*xbar_{t-1} + x_t
//
// Reference semantics: _step_state (gradients.py:118-129), heaviside/surrogate_grad
// (graph.py:40-52), the LIF trace G_u (gradients.py:89-94 with H_I = alpha, F rows = x_t,
// test_gradients.py:81-91), the ALIF trace block (neurons.py:266-273), the readout filter
// (gradients.py:163-174).
//
// Chunked eligibility algebra (two-pass form).  Within a chunk of L
// steps t = t0 + r, with A_r = rho - beta psi_{r-1}, P_r = psi_{r-1}, Lpsi_r = c_t w_sig
// psi_r, Q_r = -beta Lpsi_r and the row index rho of the staged presynaptic filter
// (rho = 0: xbar_{t0-1}, rho = r+1: xbar_{t0+r}):
//   eps_r = D(r,-1) E0 + sum_{q<=r} D(r,q) P_q xbar_{q-1},   D(r,q) = prod_{q<p<=r} A_p
//   sum_r Q_r eps_r = M E0 + sum_r R_r xbar_{r-1},   Lambda_r = Q_r + A_{r+1} Lambda_{r+1},
//                     R_r = P_r Lambda_r,  M = A_0 Lambda_0
//   E_end = Dt E0 + sum_r W_r xbar_{r-1},  W_r = P_r D(L-1,r),  Dt = prod_r A_r
// so the gradient of a chunk is ONE GEMM over (sample, rho) with coefficient
//   C_rho = R_rho [rho < L] + Lpsi_{rho-1} [rho >= 1]          (LIF: R = 0)
// plus the elementwise M E0 term, and the carried trace is a per-sample GEMM with W.
#include "common.cuh"

namespace spb {

struct FwdParams {
  int B, n, Tc, KR, len, t0, T;
  double alpha, theta, slope, beta, rho, kappa;
  int reset, alif, pass;  // pass 0 = A, 1 = B
};

constexpr int K1_THREADS = 128;  // 4 warps = 4 samples x 32 neurons

// ------------------------------------------------------------------------------------
// K1.  Warp = 32 consecutive neurons of one sample.  State u, a and the current are fp64
// so spike decisions match the f64 reference; every multiply/add of the
// state update mirrors the reference's operation order with explicit round-to-nearest
// intrinsics (no FMA contraction).  Pass B parks psi of the chunk in a global scratch
// ([b][rho][i], coalesced; L2-resident for the scan that immediately reads it back) so the
// kernel runs at full occupancy; the backward scan runs in fp32 (every quantity it
// produces feeds the fp32 / bf16-split gradient path).
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(K1_THREADS) forward_chunk_kernel(
    FwdParams P, const double* __restrict__ cur, double* __restrict__ u_st,
    double* __restrict__ a_st, double* __restrict__ zbar_st, double* __restrict__ zsum_st,
    uint32_t* __restrict__ raster, const float* __restrict__ wsig, const float* __restrict__ ctab,
    __nv_bfloat16* __restrict__ c_hi, __nv_bfloat16* __restrict__ c_lo,
    __nv_bfloat16* __restrict__ w_hi, __nv_bfloat16* __restrict__ w_lo,
    float2* __restrict__ mdt, float* __restrict__ psis) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = blockIdx.x * 32 + lane;
  const bool valid_i = i < P.n;
  const int b = blockIdx.y * (K1_THREADS / 32) + warp;
  if (b >= P.B) return;  // warp-uniform; no block-level barriers below
  const long long bi = (long long)b * P.n + i;
  double u = 0.0, a = 0.0, zbar = 0.0, zsum = 0.0;
  float w_sig = 0.0f;
  if (valid_i) {
    u = u_st[bi];
    a = a_st[bi];
    if (P.pass == 0) {
      zbar = zbar_st[bi];
      zsum = zsum_st[bi];
    } else {
      w_sig = wsig[bi];
    }
  }
  const double theta = P.theta, beta = P.beta;
  const int nw = (P.n + 31) >> 5;
  const double* crow = cur + (long long)b * P.Tc * P.n + i;
  // d_prev of step t is the drive d of step t-1 (the reference recomputes the same
  // expression from the same state, gradients.py:159): carry it.
  double d_prev = __dsub_rn(__dsub_rn(u, theta), __dmul_rn(beta, a));
  const float slope = (float)P.slope;
  float* prow = psis + (long long)b * (P.KR + 1) * P.n + i;  // pass B: psi of row rho at prow[rho*n]
  if (P.pass == 1 && valid_i) prow[0] = surrogate_grad_f32((float)d_prev, slope);  // psi_{t0-1}
  for (int s8 = 0; s8 < P.len; s8 += 8) {
    double Ib[8];
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8)
      Ib[u8] = (valid_i && s8 + u8 < P.len) ? crow[(long long)(s8 + u8) * P.n] : 0.0;
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) {
      const int s = s8 + u8;
      if (s < P.len) {
        // gradients.py:121-129 (u - theta - beta*a evaluates as (u - theta) - (beta*a))
        const double z_prev = d_prev >= 0.0 ? 1.0 : 0.0;
        a = __dadd_rn(__dmul_rn(P.rho, a), z_prev);
        u = __dadd_rn(__dmul_rn(P.alpha, u), Ib[u8]);
        if (P.reset) u = __dsub_rn(u, __dmul_rn(theta, z_prev));
        const double d = __dsub_rn(__dsub_rn(u, theta), __dmul_rn(beta, a));
        const bool z = d >= 0.0;
        if (P.pass == 0) {
          zbar = __dadd_rn(__dmul_rn(P.kappa, zbar), z ? 1.0 : 0.0);
          zsum = __dadd_rn(zsum, zbar);
          const unsigned bal = __ballot_sync(0xffffffffu, z && valid_i);
          if (raster != nullptr && lane == 0)
            raster[((long long)b * P.T + P.t0 + s) * nw + blockIdx.x] = bal;
        } else {
          // the surrogate only scales fp32 eligibilities: evaluate it in fp32
          if (valid_i) prow[(long long)(s + 1) * P.n] = surrogate_grad_f32((float)d, slope);
        }
        d_prev = d;
      }
    }
  }
  if (valid_i) {
    u_st[bi] = u;
    a_st[bi] = a;
    if (P.pass == 0) {
      zbar_st[bi] = zbar;
      zsum_st[bi] = zsum;
    }
  }
  if (P.pass == 0) return;

  // ---- backward scan over the chunk, emitting GEMM operands rho = KR-1 .. 0 ----
  if (!valid_i) return;
  const int L = P.len;
  const long long K = (long long)P.B * P.KR;
  const long long obase = (long long)i * K + (long long)b * P.KR;
  const float beta_f = (float)beta, rho_f = (float)P.rho;
  float lam = 0.f, dcum = 1.f, a_next = 0.f;
  uint32_t ch[4], cl[4], wh[4], wl[4];  // bf16x2 pairs
  // software-pipelined psi reads: rows r8 .. r8+8 of the group, next group prefetched
  float pc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) pc[q] = prow[(long long)(P.KR - 8 + q) * P.n];
  for (int r8 = P.KR - 8; r8 >= 0; r8 -= 8) {
    float pn[8];
    if (r8 >= 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) pn[q] = prow[(long long)(r8 - 8 + q) * P.n];
    }
    float cv[8], wv[8];
#pragma unroll
    for (int u8 = 7; u8 >= 0; --u8) {
      const int r = r8 + u8;
      float cval = 0.0f, wval = 0.0f;
      if (r <= L) {
        const float psi_prev = pc[u8];  // psi_{r-1}
        if (r >= 1) cval = ctab[P.t0 + r - 1] * w_sig * psi_prev;  // Lpsi_{r-1}
        if (P.alif && r < L) {
          const float psi_r = pc[u8 + 1];
          const float A = fmaf(-beta_f, psi_prev, rho_f);
          const float Q = -beta_f * (ctab[P.t0 + r] * w_sig * psi_r);
          lam = fmaf(a_next, lam, Q);             // Lambda_r (Lambda_L = 0)
          cval = fmaf(psi_prev, lam, cval);       // + R_r
          wval = psi_prev * dcum;                 // W_r = P_r D(L-1, r)
          dcum *= A;
          a_next = A;
        }
      }
      cv[u8] = cval;
      wv[u8] = wval;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      split_bf16x2(cv[2 * q], cv[2 * q + 1], ch[q], cl[q]);
      if (P.alif) split_bf16x2(wv[2 * q], wv[2 * q + 1], wh[q], wl[q]);
    }
    *reinterpret_cast<uint4*>(c_hi + obase + r8) = *reinterpret_cast<uint4*>(ch);
    *reinterpret_cast<uint4*>(c_lo + obase + r8) = *reinterpret_cast<uint4*>(cl);
    if (P.alif) {
      *reinterpret_cast<uint4*>(w_hi + obase + r8) = *reinterpret_cast<uint4*>(wh);
      *reinterpret_cast<uint4*>(w_lo + obase + r8) = *reinterpret_cast<uint4*>(wl);
    }
    pc[8] = pc[0];
#pragma unroll
    for (int q = 0; q < 8; ++q) pc[q] = pn[q];
  }
  if (P.alif) mdt[bi] = make_float2(a_next * lam, dcum);  // M = A_0 Lambda_0, Dt = prod A
}

// ------------------------------------------------------------------------------------
// K4: xbar chunk.  Thread per (sample, channel); fp64 recurrence.  Writes the bf16 hi/lo
// split, K-major over (sample, rho): xh/xl [k_rows][B*KR], rho = 0 -> xbar_{t0-1} (carry),
// rho = s+1 -> xbar_{t0+s}, zero beyond the chunk.
// ------------------------------------------------------------------------------------
__global__ void xbar_chunk_kernel(const uint8_t* __restrict__ x, long long stride_b, int B,
                                  int k, int k_rows, int KR, int len, double alpha,
                                  double* __restrict__ xbar_st, __nv_bfloat16* __restrict__ xh,
                                  __nv_bfloat16* __restrict__ xl) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (j >= k_rows) return;
  const bool valid = j < k;
  double xb = valid ? xbar_st[(long long)b * k + j] : 0.0;
  const long long K = (long long)B * KR;
  const uint8_t* xin = x + (long long)b * stride_b + j;
  __nv_bfloat16 hv[8], lv[8];
  for (int r8 = 0; r8 < KR; r8 += 8) {
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) {
      const int rho = r8 + u8;
      float v = 0.0f;
      if (rho == 0) {
        v = (float)xb;
      } else if (rho <= len) {
        if (valid) xb = __dadd_rn(__dmul_rn(alpha, xb), (double)xin[(long long)(rho - 1) * k]);
        v = (float)xb;
      }
      split_bf16(v, hv[u8], lv[u8]);
    }
    const long long off = (long long)j * K + (long long)b * KR + r8;
    *reinterpret_cast<uint4*>(xh + off) = *reinterpret_cast<uint4*>(hv);
    *reinterpret_cast<uint4*>(xl + off) = *reinterpret_cast<uint4*>(lv);
  }
  if (valid) xbar_st[(long long)b * k + j] = xb;
}

}  // namespace spb

using namespace spb;

extern "C" {

int spb_forward_chunk(int pass, const double* cur, int B, int n, int Tc, int KR, int len, int t0,
                      int T, double alpha, double theta, double slope, double beta, double rho,
                      double kappa, int reset, int alif, double* u, double* a, double* zbar,
                      double* zsum, uint32_t* raster, const float* wsig, const float* ctab,
                      void* c_hi, void* c_lo, void* w_hi, void* w_lo, float* mdt,
                      float* psi_scratch, cudaStream_t stream) {
  SPB_CHECK_ARG(pass == 0 || pass == 1, "spb_forward_chunk: pass must be 0 (A) or 1 (B)");
  SPB_CHECK_ARG(cur && u && a, "spb_forward_chunk: null pointer");
  SPB_CHECK_ARG(B > 0 && n > 0 && Tc > 0 && len >= 0 && len <= Tc && KR >= Tc + 1 && KR % 8 == 0,
                "spb_forward_chunk: bad sizes B=%d n=%d Tc=%d KR=%d len=%d", B, n, Tc, KR, len);
  SPB_CHECK_ARG(pass == 0 ? (zbar && zsum) : (wsig && ctab && c_hi && c_lo && psi_scratch),
                "spb_forward_chunk: missing pass-%c buffers", pass ? 'B' : 'A');
  SPB_CHECK_ARG(!(pass == 1 && alif && (!w_hi || !w_lo || !mdt)),
                "spb_forward_chunk: ALIF pass B needs w_hi, w_lo and mdt");
  SPB_CHECK_ARG(!(pass == 1 && reset), "spb_forward_chunk: reset=True has no two-pass form");
  FwdParams P{B, n, Tc, KR, len, t0, T, alpha, theta, slope, beta, rho, kappa, reset, alif, pass};
  dim3 grid(ceil_div(n, 32), ceil_div(B, K1_THREADS / 32));
  forward_chunk_kernel<<<grid, K1_THREADS, 0, stream>>>(
      P, cur, u, a, zbar, zsum, raster, wsig, ctab, reinterpret_cast<__nv_bfloat16*>(c_hi),
      reinterpret_cast<__nv_bfloat16*>(c_lo), reinterpret_cast<__nv_bfloat16*>(w_hi),
      reinterpret_cast<__nv_bfloat16*>(w_lo), reinterpret_cast<float2*>(mdt), psi_scratch);
  SPB_CHECK_LAUNCH("forward_chunk");
  return 0;
}

int spb_xbar_chunk(const uint8_t* x, long long stride_b, int B, int k, int k_rows, int KR,
                   int len, double alpha, double* xbar_state, void* xh, void* xl,
                   cudaStream_t stream) {
  SPB_CHECK_ARG(x && xbar_state && xh && xl, "spb_xbar_chunk: null pointer");
  SPB_CHECK_ARG(B > 0 && k > 0 && k_rows >= k && KR > 0 && KR % 8 == 0 && len >= 0 && len < KR,
                "spb_xbar_chunk: bad sizes");
  dim3 grid(ceil_div(k_rows, 128), B);
  xbar_chunk_kernel<<<grid, 128, 0, stream>>>(x, stride_b, B, k, k_rows, KR, len, alpha,
                                              xbar_state, reinterpret_cast<__nv_bfloat16*>(xh),
                                              reinterpret_cast<__nv_bfloat16*>(xl));
  SPB_CHECK_LAUNCH("xbar_chunk");
  return 0;
}

}  // extern "C"
