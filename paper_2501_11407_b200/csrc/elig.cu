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
#include "tma.cuh"

namespace spb {

constexpr int K6_TI = 128;   // neurons per CTA tile
constexpr int K6_TJ = 64;    // inputs per CTA tile
constexpr int K6_THREADS = 256;
constexpr int K6_MAX_TC = 64;

// Shared-memory stage for one sample: eps~ tile, (A',Q') rows and xbar rows of the chunk.
template <int TC>
struct K6Stage {
  static constexpr int EPS_BYTES = K6_TI * K6_TJ * 4;              // 32 KB
  static constexpr int COEF_BYTES = TC * K6_TI * 8;                // TC KB
  static constexpr int XB_BYTES = ((TC + 1) * K6_TJ * 4 + 127) / 128 * 128;
  static constexpr int BYTES = EPS_BYTES + COEF_BYTES + XB_BYTES;
};

// TMA-pipelined sweep.  Each CTA owns a 128x64 synapse tile and a contiguous range of
// samples; per sample, one elected thread TMA-loads the sample's eps~ tile, its chunk of
// (A',Q') and xbar rows into a shared-memory stage (STAGES-deep ring), the 256 threads
// sweep the chunk from registers (4 neurons x 8 inputs each, FFMA2), and write eps~ back
// with plain stores.  The gradient tile stays in registers across the sample loop.
template <int TC, int STAGES>
__global__ void __launch_bounds__(K6_THREADS, 1) alif_elig_tma_kernel(
    const __grid_constant__ CUtensorMap tm_eps, const __grid_constant__ CUtensorMap tm_coef,
    const __grid_constant__ CUtensorMap tm_xb, float* __restrict__ eps,
    float* __restrict__ partial, int B, int n_pad, int k_pad, int len, int b_per_split,
    int load_eps, int store_eps) {
  using S = K6Stage<TC>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::BYTES);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int li = lane >> 3, lj = lane & 7;
  const int j0 = blockIdx.x * K6_TJ, i0 = blockIdx.y * K6_TI;
  const int b_begin = blockIdx.z * b_per_split;
  const int nb = max(0, min(B, b_begin + b_per_split) - b_begin);
  const int row0 = warp * 16 + li * 4;
  const int cA = lj * 4, cB = 32 + lj * 4;
  const uint32_t stage_bytes =
      (load_eps ? S::EPS_BYTES : 0) + S::COEF_BYTES + (TC + 1) * K6_TJ * 4;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&full[s]), 1);
    mbar_fence_init();
    tma_prefetch_desc(&tm_eps);
    tma_prefetch_desc(&tm_coef);
    tma_prefetch_desc(&tm_xb);
  }
  __syncthreads();

  auto issue = [&](int it) {
    const int s = it % STAGES;
    const int b = b_begin + it;
    uint8_t* st = smem + s * S::BYTES;
    const uint32_t fb = smem_u32(&full[s]);
    mbar_expect_tx(fb, stage_bytes);
    if (load_eps) tma_load_2d(smem_u32(st), &tm_eps, fb, j0, b * n_pad + i0);
    tma_load_2d(smem_u32(st + S::EPS_BYTES), &tm_coef, fb, 2 * i0, b * TC);
    tma_load_2d(smem_u32(st + S::EPS_BYTES + S::COEF_BYTES), &tm_xb, fb, j0, b * (TC + 1));
  };
  if (tid == 0)
    for (int it = 0; it < min(nb, STAGES - 1); ++it) issue(it);

  float2 g2[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int p = 0; p < 4; ++p) g2[r][p] = make_float2(0.f, 0.f);

  for (int it = 0; it < nb; ++it) {
    const int s = it % STAGES;
    if (tid == 0 && it + STAGES - 1 < nb) issue(it + STAGES - 1);
    mbar_wait(smem_u32(&full[s]), (it / STAGES) & 1);
    const uint8_t* st = smem + s * S::BYTES;
    const float* es = reinterpret_cast<const float*>(st);
    const float2* cs = reinterpret_cast<const float2*>(st + S::EPS_BYTES);
    const float* xs = reinterpret_cast<const float*>(st + S::EPS_BYTES + S::COEF_BYTES);
    float2 e2[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (load_eps) {
        const float4 va = *reinterpret_cast<const float4*>(es + (row0 + r) * K6_TJ + cA);
        const float4 vb = *reinterpret_cast<const float4*>(es + (row0 + r) * K6_TJ + cB);
        e2[r][0] = make_float2(va.x, va.y);
        e2[r][1] = make_float2(va.z, va.w);
        e2[r][2] = make_float2(vb.x, vb.y);
        e2[r][3] = make_float2(vb.z, vb.w);
      } else {
#pragma unroll
        for (int p = 0; p < 4; ++p) e2[r][p] = make_float2(0.f, 0.f);
      }
    }
#pragma unroll 2
    for (int ss = 0; ss < len; ++ss) {
      const float4 xa = *reinterpret_cast<const float4*>(xs + ss * K6_TJ + cA);
      const float4 xb = *reinterpret_cast<const float4*>(xs + ss * K6_TJ + cB);
      const float2 x2[4] = {make_float2(xa.x, xa.y), make_float2(xa.z, xa.w),
                            make_float2(xb.x, xb.y), make_float2(xb.z, xb.w)};
      const float4 c01 = *reinterpret_cast<const float4*>(cs + ss * K6_TI + row0);
      const float4 c23 = *reinterpret_cast<const float4*>(cs + ss * K6_TI + row0 + 2);
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
    if (store_eps) {
      float* ebase = eps + ((long long)(b_begin + it) * n_pad + i0 + row0) * k_pad + j0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        *reinterpret_cast<float4*>(ebase + (long long)r * k_pad + cA) =
            make_float4(e2[r][0].x, e2[r][0].y, e2[r][1].x, e2[r][1].y);
        *reinterpret_cast<float4*>(ebase + (long long)r * k_pad + cB) =
            make_float4(e2[r][2].x, e2[r][2].y, e2[r][3].x, e2[r][3].y);
      }
    }
    __syncthreads();  // stage s may be refilled by the next issue
  }
  float* pbase = partial + ((long long)blockIdx.z * n_pad + i0 + row0) * k_pad + j0;
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
  SPB_CHECK_ARG(Tc == 8 || Tc == 16 || Tc == 32 || Tc == 64,
                "spb_alif_elig_chunk: chunk length must be 8, 16, 32 or 64 (got %d)", Tc);
  SPB_CHECK_ARG(B > 0 && splits > 0 && splits <= B && len >= 0 && len <= Tc,
                "spb_alif_elig_chunk: bad sizes B=%d splits=%d len=%d Tc=%d", B, splits, len, Tc);
  CUtensorMap m_eps, m_coef, m_xb;
  const bool ok =
      make_tmap_2d(&m_eps, eps, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, k_pad, (uint64_t)B * n_pad,
                   (uint64_t)k_pad * 4, K6_TJ, K6_TI, CU_TENSOR_MAP_SWIZZLE_NONE) &&
      make_tmap_2d(&m_coef, coef, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 2 * (uint64_t)n_pad,
                   (uint64_t)B * Tc, (uint64_t)n_pad * 8, 2 * K6_TI, Tc,
                   CU_TENSOR_MAP_SWIZZLE_NONE) &&
      make_tmap_2d(&m_xb, xf, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, k_pad, (uint64_t)B * (Tc + 1),
                   (uint64_t)k_pad * 4, K6_TJ, Tc + 1, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!ok) {
    set_error("spb_alif_elig_chunk: cuTensorMapEncodeTiled failed");
    return 3;
  }
  const int bps = ceil_div(B, splits);
  dim3 grid(k_pad / K6_TJ, n_pad / K6_TI, splits);
#define SPB_K6_LAUNCH(TC, ST)                                                                   \
  do {                                                                                          \
    auto kfn = alif_elig_tma_kernel<TC, ST>;                                                    \
    const int smem = ST * K6Stage<TC>::BYTES + 128 + 64;                                       \
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);               \
    kfn<<<grid, K6_THREADS, smem, stream>>>(m_eps, m_coef, m_xb, eps, partial, B, n_pad, k_pad, \
                                            len, bps, load_eps, store_eps);                     \
  } while (0)
  switch (Tc) {
    case 8: SPB_K6_LAUNCH(8, 4); break;
    case 16: SPB_K6_LAUNCH(16, 3); break;
    case 32: SPB_K6_LAUNCH(32, 3); break;
    default: SPB_K6_LAUNCH(64, 2); break;
  }
#undef SPB_K6_LAUNCH
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
