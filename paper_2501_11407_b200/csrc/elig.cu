// Eligibility-trace gradient kernels (sm_100a):
//   K6  spb_alif_elig_chunk  -- ALIF per-synapse adaptation trace eps_a swept over a
//                               time chunk with the synapse tile held in registers
//   --  spb_reduce_partials  -- fixed-order batch-split reduction into the fp64 gradient
//   K5s spb_grad_gemm_simt   -- CUDA-core reference of the factorised GEMM (tests only)
//
// Reference: the ALIF block of eprop_trace_update (gradients.py:89-94, H_I block
// [[alpha,0],[psi^-, rho - beta psi^-]] from neurons.py:266-273 / test_neurons.py:144-155)
// and the eligibility filter x_step = psi (G_u - beta G_a) (gradients.py:165-172).
//
// Rescaled trace.  With eps_t = A_t eps_{t-1} + P_t xbar_{t-1}, A_t = rho - beta psi_{t-1},
// P_t = psi_{t-1}, the kernel carries eps~_t = eps_t / psi_{t-1}:
//     eps~_t = A'_t eps~_{t-1} + xbar_{t-1},      A'_t = A_t psi_{t-2} / psi_{t-1}
//     grad  += Q'_t eps~_t,                        Q'_t = -beta L_t psi_t psi_{t-1}
// i.e. exactly two FMAs per synapse-sample-step (one FFMA2 per synapse pair per step),
// instead of FMUL+FFMA+FFMA for the literal form.  All terms of eps~ are non-negative for
// non-negative inputs (A' > 0 when rho > beta), so the rescaling adds no cancellation.
#include "common.cuh"

namespace spb {

constexpr int K6_TI = 128;   // neurons per CTA tile
constexpr int K6_TJ = 64;    // inputs per CTA tile
constexpr int K6_SC = 16;    // time steps staged per shared-memory fill
constexpr int K6_THREADS = 256;

__global__ void __launch_bounds__(K6_THREADS, 2) alif_elig_kernel(
    const float2* __restrict__ coef,  // [B][Tc][n]  (A', Q')
    const float* __restrict__ xf,     // [B][Tc+1][k_pad]  row s = xbar_{t0-1+s}
    float* __restrict__ eps,          // [B][n_pad][k_pad] eps~ state
    float* __restrict__ partial,      // [S][n_pad][k_pad]
    int B, int n, int n_pad, int k_pad, int Tc, int len, int b_per_split, int load_eps,
    int store_eps) {
  __shared__ __align__(16) float2 coefS[K6_SC][K6_TI];
  __shared__ __align__(16) float xS[K6_SC][K6_TJ];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int li = lane >> 3, lj = lane & 7;
  const int j0 = blockIdx.x * K6_TJ, i0 = blockIdx.y * K6_TI;
  const int split = blockIdx.z;
  const int b_begin = split * b_per_split;
  const int b_end = min(B, b_begin + b_per_split);
  const int row0 = warp * 16 + li * 4;  // first of this thread's 4 neurons (tile-local)
  const int cA = lj * 4, cB = 32 + lj * 4;

  float2 g2[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int p = 0; p < 4; ++p) g2[r][p] = make_float2(0.f, 0.f);

  for (int b = b_begin; b < b_end; ++b) {
    float2 e2[4][4];
    float* ebase = eps + ((long long)b * n_pad + i0 + row0) * k_pad + j0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (load_eps) {
        const float4 va = *reinterpret_cast<const float4*>(ebase + (long long)r * k_pad + cA);
        const float4 vb = *reinterpret_cast<const float4*>(ebase + (long long)r * k_pad + cB);
        e2[r][0] = make_float2(va.x, va.y);
        e2[r][1] = make_float2(va.z, va.w);
        e2[r][2] = make_float2(vb.x, vb.y);
        e2[r][3] = make_float2(vb.z, vb.w);
      } else {
#pragma unroll
        for (int p = 0; p < 4; ++p) e2[r][p] = make_float2(0.f, 0.f);
      }
    }
    for (int s0 = 0; s0 < len; s0 += K6_SC) {
      const int steps = min(K6_SC, len - s0);
      // stage (A',Q') for TI neurons and xbar_{t-1} for TJ inputs, `steps` rows each
      for (int idx = tid; idx < K6_SC * K6_TI; idx += K6_THREADS) {
        const int ss = idx / K6_TI, c = idx % K6_TI;
        float2 v = make_float2(0.f, 0.f);
        if (ss < steps && i0 + c < n) v = coef[((long long)b * Tc + s0 + ss) * n + i0 + c];
        coefS[ss][c] = v;
      }
      for (int idx = tid; idx < K6_SC * K6_TJ; idx += K6_THREADS) {
        const int ss = idx / K6_TJ, c = idx % K6_TJ;
        float v = 0.f;
        if (ss < steps) v = xf[((long long)b * (Tc + 1) + s0 + ss) * k_pad + j0 + c];
        xS[ss][c] = v;
      }
      __syncthreads();
      for (int ss = 0; ss < steps; ++ss) {
        const float4 xa = *reinterpret_cast<const float4*>(&xS[ss][cA]);
        const float4 xb = *reinterpret_cast<const float4*>(&xS[ss][cB]);
        const float2 x2[4] = {make_float2(xa.x, xa.y), make_float2(xa.z, xa.w),
                              make_float2(xb.x, xb.y), make_float2(xb.z, xb.w)};
        const float4 c01 = *reinterpret_cast<const float4*>(&coefS[ss][row0]);
        const float4 c23 = *reinterpret_cast<const float4*>(&coefS[ss][row0 + 2]);
        const float Ar[4] = {c01.x, c01.z, c23.x, c23.z};
        const float Qr[4] = {c01.y, c01.w, c23.y, c23.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float2 A2 = make_float2(Ar[r], Ar[r]);
          const float2 Q2 = make_float2(Qr[r], Qr[r]);
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            e2[r][p] = ffma2(A2, e2[r][p], x2[p]);
            g2[r][p] = ffma2(Q2, e2[r][p], g2[r][p]);
          }
        }
      }
      __syncthreads();
    }
    if (store_eps) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        *reinterpret_cast<float4*>(ebase + (long long)r * k_pad + cA) =
            make_float4(e2[r][0].x, e2[r][0].y, e2[r][1].x, e2[r][1].y);
        *reinterpret_cast<float4*>(ebase + (long long)r * k_pad + cB) =
            make_float4(e2[r][2].x, e2[r][2].y, e2[r][3].x, e2[r][3].y);
      }
    }
  }
  float* pbase = partial + ((long long)split * n_pad + i0 + row0) * k_pad + j0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    *reinterpret_cast<float4*>(pbase + (long long)r * k_pad + cA) =
        make_float4(g2[r][0].x, g2[r][0].y, g2[r][1].x, g2[r][1].y);
    *reinterpret_cast<float4*>(pbase + (long long)r * k_pad + cB) =
        make_float4(g2[r][2].x, g2[r][2].y, g2[r][3].x, g2[r][3].y);
  }
}

__global__ void reduce_partials_kernel(const float* __restrict__ partial, int S, int n, int n_pad,
                                       int k_pad, double* __restrict__ grad) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n * k_pad) return;
  const long long stride = (long long)n_pad * k_pad;
  double acc = 0.0;
  for (int s = 0; s < S; ++s) acc += (double)partial[s * stride + idx];
  grad[idx] += acc;
}

// CUDA-core GEMM on the same bf16 hi/lo K-major operands as the tensor-core path:
// grad[i][j] += sum_K (Ah+Al)[i][K] * (Bh+Bl)[j][K]  (64x64 tiles, 4x4 per thread).
__global__ void __launch_bounds__(256) grad_gemm_simt_kernel(
    const __nv_bfloat16* __restrict__ ah, const __nv_bfloat16* __restrict__ al,
    const __nv_bfloat16* __restrict__ bh, const __nv_bfloat16* __restrict__ bl, int M, int N,
    int K, double* __restrict__ grad, int ldg) {
  __shared__ float As[32][65];
  __shared__ float Bs[32][65];
  const int tid = threadIdx.x;
  const int tm = tid >> 4, tn = tid & 15;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int idx = tid; idx < 64 * 32; idx += 256) {
      const int r = idx >> 5, kk = idx & 31;
      float va = 0.f, vb = 0.f;
      if (m0 + r < M && k0 + kk < K) {
        const long long o = (long long)(m0 + r) * K + k0 + kk;
        va = __bfloat162float(ah[o]) + __bfloat162float(al[o]);
      }
      if (n0 + r < N && k0 + kk < K) {
        const long long o = (long long)(n0 + r) * K + k0 + kk;
        vb = __bfloat162float(bh[o]) + __bfloat162float(bl[o]);
      }
      As[kk][r] = va;
      Bs[kk][r] = vb;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[kk][tm * 4 + q];
        bb[q] = Bs[kk][tn * 4 + q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fmaf(a[p], bb[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = m0 + tm * 4 + p, j = n0 + tn * 4 + q;
      if (i < M && j < N) grad[(long long)i * ldg + j] += (double)acc[p][q];
    }
}

}  // namespace spb

using namespace spb;

extern "C" {

int spb_alif_elig_chunk(const float* coef, const float* xf, float* eps, float* partial, int B,
                        int n, int n_pad, int k_pad, int Tc, int len, int splits, int load_eps,
                        int store_eps, cudaStream_t stream) {
  SPB_CHECK_ARG(coef && xf && eps && partial, "spb_alif_elig_chunk: null pointer");
  SPB_CHECK_ARG(n_pad % K6_TI == 0 && k_pad % K6_TJ == 0 && n <= n_pad,
                "spb_alif_elig_chunk: n_pad must be a multiple of %d and k_pad of %d", K6_TI,
                K6_TJ);
  SPB_CHECK_ARG(B > 0 && splits > 0 && splits <= B && len >= 0 && len <= Tc,
                "spb_alif_elig_chunk: bad sizes B=%d splits=%d len=%d Tc=%d", B, splits, len, Tc);
  const int bps = ceil_div(B, splits);
  dim3 grid(k_pad / K6_TJ, n_pad / K6_TI, splits);
  alif_elig_kernel<<<grid, K6_THREADS, 0, stream>>>(reinterpret_cast<const float2*>(coef), xf,
                                                    eps, partial, B, n, n_pad, k_pad, Tc, len,
                                                    bps, load_eps, store_eps);
  SPB_CHECK_LAUNCH("alif_elig");
  return 0;
}

int spb_reduce_partials(const float* partial, int splits, int n, int n_pad, int k_pad,
                        double* grad, cudaStream_t stream) {
  SPB_CHECK_ARG(partial && grad && splits > 0 && n > 0 && n <= n_pad,
                "spb_reduce_partials: bad args");
  const long long total = (long long)n * k_pad;
  reduce_partials_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(
      partial, splits, n, n_pad, k_pad, grad);
  SPB_CHECK_LAUNCH("reduce_partials");
  return 0;
}

int spb_grad_gemm_simt(const void* ah, const void* al, const void* bh, const void* bl, int M,
                       int N, int K, double* grad, int ldg, cudaStream_t stream) {
  SPB_CHECK_ARG(ah && al && bh && bl && grad && M > 0 && N > 0 && K > 0 && ldg >= N,
                "spb_grad_gemm_simt: bad args");
  dim3 grid(ceil_div(N, 64), ceil_div(M, 64));
  grad_gemm_simt_kernel<<<grid, 256, 0, stream>>>(
      (const __nv_bfloat16*)ah, (const __nv_bfloat16*)al, (const __nv_bfloat16*)bh,
      (const __nv_bfloat16*)bl, M, N, K, grad, ldg);
  SPB_CHECK_LAUNCH("grad_gemm_simt");
  return 0;
}

}  // extern "C"
