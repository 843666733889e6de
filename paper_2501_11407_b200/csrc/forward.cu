// Forward-side kernels of the e-prop update (sm_100a):
//   K1  spb_forward_chunk   -- LIF/ALIF dynamics + surrogate over a time chunk from the
//                              exact input current of K2 (proj.cu); pass A (spike raster,
//                              zsum) or pass B (learning-signal-weighted surrogate,
//                              eligibility coefficients)
//   K4  spb_xbar_chunk      -- presynaptic filter xbar_t = alpha*xbar_{t-1} + x_t
//
// Reference semantics: _step_state (gradients.py:118-129), heaviside/surrogate_grad
// (graph.py:40-52), the LIF trace G_u (gradients.py:89-94 with H_I = alpha, F rows = x_t,
// test_gradients.py:81-91), readout filter (gradients.py:163-174).
#include "common.cuh"
#include <algorithm>

namespace spb {

// ------------------------------------------------------------------------------------
// K1: neuron dynamics over one time chunk, reading the exact input current I (fp64,
// produced by the INT8 tensor-core projection K2, proj.cu).  Warp = 32 consecutive
// neurons of one sample.  State u, a and I are fp64 so spike decisions match the f64
// reference; every multiply/add mirrors the reference's operation order
// with explicit round-to-nearest intrinsics (no FMA contraction).
// ------------------------------------------------------------------------------------
struct FwdParams {
  int B, n, Tc, len, t0, T, coef_ld;
  double alpha, theta, slope, beta, rho, kappa;
  int reset, alif, pass;  // pass 0 = A, 1 = B
};

__global__ void __launch_bounds__(256) forward_chunk_kernel(
    FwdParams P, const double* __restrict__ cur, double* __restrict__ u_st,
    double* __restrict__ a_st, double* __restrict__ zbar_st, double* __restrict__ zsum_st,
    uint32_t* __restrict__ raster, const float* __restrict__ wsig, const double* __restrict__ ctab,
    float* __restrict__ psi2_st, float2* __restrict__ coef, __nv_bfloat16* __restrict__ lp_hi,
    __nv_bfloat16* __restrict__ lp_lo) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const bool valid_i = i < P.n;
  const int b = blockIdx.y * (blockDim.x >> 5) + warp;
  if (b >= P.B) return;
  const long long bi = (long long)b * P.n + i;
  double u = 0.0, a = 0.0, zbar = 0.0, zsum = 0.0;
  float psi2 = 1.0f, w_sig = 0.0f;
  if (valid_i) {
    u = u_st[bi];
    a = a_st[bi];
    if (P.pass == 0) {
      zbar = zbar_st[bi];
      zsum = zsum_st[bi];
    } else {
      psi2 = psi2_st[bi];
      w_sig = wsig[bi];
    }
  }
  const double theta = P.theta, beta = P.beta;
  const int K = P.B * P.Tc;
  const int nw = (P.n + 31) >> 5;
  const double* crow = cur + (long long)b * P.Tc * P.n + i;
  __nv_bfloat16 hv[8], lv[8];
  for (int s8 = 0; s8 < P.Tc; s8 += 8) {
    double Ib[8];
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8)
      Ib[u8] = (valid_i && s8 + u8 < P.len) ? crow[(long long)(s8 + u8) * P.n] : 0.0;
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) {
      const int s = s8 + u8;
      if (s < P.len) {
        const int row = b * P.Tc + s;
        const double I = Ib[u8];
        // gradients.py:121-129 (u - theta - beta*a evaluates as (u - theta) - (beta*a))
        const double d_prev = __dsub_rn(__dsub_rn(u, theta), __dmul_rn(beta, a));
        const double z_prev = d_prev >= 0.0 ? 1.0 : 0.0;
        a = __dadd_rn(__dmul_rn(P.rho, a), z_prev);
        u = __dadd_rn(__dmul_rn(P.alpha, u), I);
        if (P.reset) u = __dsub_rn(u, __dmul_rn(theta, z_prev));
        const double d = __dsub_rn(__dsub_rn(u, theta), __dmul_rn(beta, a));
        const bool z = d >= 0.0;
        const int t = P.t0 + s;
        if (P.pass == 0) {
          // readout filter of the spikes (gradients.py:173-174)
          zbar = __dadd_rn(__dmul_rn(P.kappa, zbar), z ? 1.0 : 0.0);
          zsum = __dadd_rn(zsum, zbar);
          const unsigned bal = __ballot_sync(0xffffffffu, z && valid_i);
          if (raster != nullptr && lane == 0)
            raster[((long long)b * P.T + t) * nw + blockIdx.x] = bal;
        } else {
          const double psi_d = surrogate_grad_f64(d, P.slope);
          const float psi1 = (float)surrogate_grad_f64(d_prev, P.slope);  // psi_{t-1}
          const float lpsi = (float)(ctab[t] * (double)w_sig * psi_d);    // L_t * psi_t
          if (P.alif && coef != nullptr) {
            // eps~_t = A'_t eps~_{t-1} + xbar_{t-1}; grad += Q'_t eps~_t (eps = psi_{t-1} eps~)
            const float A = (float)(P.rho - P.beta * (double)psi1);
            const float Ap = (t == 0) ? 0.0f : A * (psi2 / fmaxf(psi1, 1e-30f));
            const float Qp = -(float)P.beta * lpsi * psi1;
            if (valid_i) coef[(long long)row * P.coef_ld + i] = make_float2(Ap, Qp);
          }
          psi2 = psi1;
          split_bf16(lpsi, hv[u8], lv[u8]);
        }
      } else if (P.pass == 1) {
        hv[u8] = __float2bfloat16_rn(0.0f);
        lv[u8] = __float2bfloat16_rn(0.0f);
      }
    }
    if (P.pass == 1 && valid_i) {
      const long long off = (long long)i * K + (long long)b * P.Tc + s8;
      *reinterpret_cast<uint4*>(lp_hi + off) = *reinterpret_cast<uint4*>(hv);
      *reinterpret_cast<uint4*>(lp_lo + off) = *reinterpret_cast<uint4*>(lv);
    }
  }
  if (valid_i) {
    u_st[bi] = u;
    a_st[bi] = a;
    if (P.pass == 0) {
      zbar_st[bi] = zbar;
      zsum_st[bi] = zsum;
    } else {
      psi2_st[bi] = psi2;
    }
  }
}

// ------------------------------------------------------------------------------------
// K4: xbar chunk.  Thread per (sample, channel); fp64 recurrence.  Writes
//   xf  [B][Tc+1][k_pad] fp32 rows (row 0 = carry xbar_{t0-1}, row s+1 = xbar_{t0+s})
//   xh/xl [k_pad][B*Tc]  bf16 hi/lo split, K-major (K index = b*Tc + s) for the GEMM.
// ------------------------------------------------------------------------------------
__global__ void xbar_chunk_kernel(const uint8_t* __restrict__ x, long long stride_b, int B,
                                  int k, int k_pad, int Tc, int len, double alpha,
                                  double* __restrict__ xbar_st, float* __restrict__ xf,
                                  __nv_bfloat16* __restrict__ xh, __nv_bfloat16* __restrict__ xl) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (j >= k_pad) return;
  const bool valid = j < k;
  double xb = valid ? xbar_st[(long long)b * k + j] : 0.0;
  const long long K = (long long)B * Tc;
  float* xrow = xf + (long long)b * (Tc + 1) * k_pad + j;
  xrow[0] = (float)xb;
  const uint8_t* xin = x + (long long)b * stride_b + j;
  __nv_bfloat16 hv[8], lv[8];
  for (int s8 = 0; s8 < Tc; s8 += 8) {
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) {
      const int s = s8 + u8;
      float v = 0.0f;
      if (s < len) {
        if (valid) xb = __dadd_rn(__dmul_rn(alpha, xb), (double)xin[(long long)s * k]);
        v = (float)xb;
        xrow[(long long)(s + 1) * k_pad] = v;
      }
      split_bf16(v, hv[u8], lv[u8]);
    }
    const long long off = (long long)j * K + (long long)b * Tc + s8;
    *reinterpret_cast<uint4*>(xh + off) = *reinterpret_cast<uint4*>(hv);
    *reinterpret_cast<uint4*>(xl + off) = *reinterpret_cast<uint4*>(lv);
  }
  if (valid) xbar_st[(long long)b * k + j] = xb;
}

}  // namespace spb

using namespace spb;

extern "C" {

int spb_forward_chunk(int pass, const double* cur, int B, int n, int Tc, int len, int t0, int T,
                      double alpha, double theta, double slope, double beta, double rho,
                      double kappa, int reset, int alif, double* u, double* a, double* zbar,
                      double* zsum, uint32_t* raster, const float* wsig, const double* ctab,
                      float* psi2, float* coef, int coef_ld, void* lp_hi, void* lp_lo,
                      cudaStream_t stream) {
  SPB_CHECK_ARG(pass == 0 || pass == 1, "spb_forward_chunk: pass must be 0 (A) or 1 (B)");
  SPB_CHECK_ARG(cur && u && a, "spb_forward_chunk: null pointer");
  SPB_CHECK_ARG(B > 0 && n > 0 && Tc > 0 && Tc % 8 == 0 && len >= 0 && len <= Tc,
                "spb_forward_chunk: bad sizes B=%d n=%d Tc=%d len=%d", B, n, Tc, len);
  SPB_CHECK_ARG(pass == 0 ? (zbar && zsum) : (wsig && ctab && psi2 && lp_hi && lp_lo),
                "spb_forward_chunk: missing pass-%c buffers", pass ? 'B' : 'A');
  SPB_CHECK_ARG(!(pass == 1 && alif && (!coef || coef_ld < n)),
                "spb_forward_chunk: ALIF pass B needs coef with coef_ld >= n");
  FwdParams P{B, n, Tc, len, t0, T, coef_ld, alpha, theta, slope, beta, rho, kappa,
              reset, alif, pass};
  dim3 grid(ceil_div(n, 32), ceil_div(B, 8));
  forward_chunk_kernel<<<grid, 256, 0, stream>>>(
      P, cur, u, a, zbar, zsum, raster, wsig, ctab, psi2, reinterpret_cast<float2*>(coef),
      reinterpret_cast<__nv_bfloat16*>(lp_hi), reinterpret_cast<__nv_bfloat16*>(lp_lo));
  SPB_CHECK_LAUNCH("forward_chunk");
  return 0;
}

int spb_xbar_chunk(const uint8_t* x, long long stride_b, int B, int k, int k_pad, int Tc,
                   int len, double alpha, double* xbar_state, float* xf, void* xh, void* xl,
                   cudaStream_t stream) {
  SPB_CHECK_ARG(x && xbar_state && xf && xh && xl, "spb_xbar_chunk: null pointer");
  SPB_CHECK_ARG(B > 0 && k > 0 && k_pad >= k && Tc > 0 && Tc % 8 == 0 && len >= 0 && len <= Tc,
                "spb_xbar_chunk: bad sizes");
  dim3 grid(ceil_div(k_pad, 128), B);
  xbar_chunk_kernel<<<grid, 128, 0, stream>>>(x, stride_b, B, k, k_pad, Tc, len, alpha,
                                              xbar_state, xf,
                                              reinterpret_cast<__nv_bfloat16*>(xh),
                                              reinterpret_cast<__nv_bfloat16*>(xl));
  SPB_CHECK_LAUNCH("xbar_chunk");
  return 0;
}

}  // extern "C"
