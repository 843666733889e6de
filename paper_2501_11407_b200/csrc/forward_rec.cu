// K1rec: LIF/ALIF dynamics of a RECURRENT hidden layer over one time chunk (sm_100a), and
// the operand builder that appends the previous step's spikes to the input for the
// eligibility kernels.  SURVEY.md 8(f)-4 -- parity UNPINNED: the reference has no
// recurrent weights; the semantics are those of
// oracle/eprop_ref.py:step_state_rec / eprop_forward_mode_rec:
//
//   z_{t-1} = spike(d_{t-1});  a <- rho a + z_{t-1}
//   u <- alpha u + (I_in,t + W_rec z_{t-1})   [- theta z_{t-1} with reset]
//   d = (u - theta) - beta a;  z_t = spike(d);  psi_t = surrogate(d)
//
// with I_in,t the exact projection of K2 and the recurrent current summed in fp64 over the
// active presynaptic neurons in ascending index order (deterministic).  The e-prop trace
// of W_rec is the input trace with presynaptic input z_{t-1} (H_E dropped), so pass B
// runs the unchanged scan / xbar / GEMM / carry kernels on the extended input
// x~_t = [x_t, z_{t-1}] (spb_pack_rec).
//
// One CTA per sample, 512 threads, NPT <= 4 consecutive neurons per thread (n <= 2048),
// two CTAs per SM for n <= 1024; the spikes of the previous step live in a double-buffered shared
// bitmask, compacted by one warp into an ascending active list each step (two
// __syncthreads per step) and padded with a -0.0 row to whole groups of SPB_REC_GB rows in flight
// at once.  The step is latency-bound (L2 round trips of the gather + two barriers).
// W_rec is stored transposed (wrecT[j][i] = W_rec[i][j]) so the gather of an active
// presynaptic row is coalesced across the CTA's threads.
#include "common.cuh"

namespace spb {

constexpr int REC_THREADS = 512;
constexpr int REC_MAX_N = 2048;

struct RecParams {
  int B, n, Tc, KR, len, t0, T;
  double alpha, theta, slope, beta, rho, kappa;
  int reset, alif, pass, smooth, w_f64;
};

__device__ __forceinline__ double rec_spike(double d, bool smooth, double slope) {
  if (!smooth) return d >= 0.0 ? 1.0 : 0.0;
  return __dadd_rn(0.5, __ddiv_rn(d, __dadd_rn(1.0, __dmul_rn(slope, fabs(d)))));
}

// The NPT neurons of a thread are consecutive (i = NPT*tid + c), so a gathered row of
// W_rec^T is one vector load per thread (float2 / float4 / double2 pairs) when n % NPT == 0
// (VEC), and a warp's spikes form NPT consecutive mask words, assembled with one OR-
// reduction per word.
template <int NPT, typename WT, bool VEC>
__device__ __forceinline__ void rec_load_row(const WT* __restrict__ row, int i0, int n,
                                             WT (&w)[NPT]) {
  if constexpr (VEC && NPT == 1) {
    w[0] = i0 < n ? __ldg(row + i0) : WT(0);
  } else if constexpr (VEC && sizeof(WT) == 4 && NPT == 2) {
    const float2 v = i0 < n ? __ldg(reinterpret_cast<const float2*>(row + i0)) : make_float2(0.f, 0.f);
    w[0] = v.x;
    w[1] = v.y;
  } else if constexpr (VEC && sizeof(WT) == 4 && NPT == 4) {
    const float4 v = i0 < n ? __ldg(reinterpret_cast<const float4*>(row + i0))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    w[0] = v.x;
    w[1] = v.y;
    w[2] = v.z;
    w[3] = v.w;
  } else if constexpr (VEC && sizeof(WT) == 8) {
#pragma unroll
    for (int c = 0; c < NPT; c += 2) {
      const double2 v = i0 < n ? __ldg(reinterpret_cast<const double2*>(row + i0 + c))
                               : make_double2(0.0, 0.0);
      w[c] = v.x;
      w[c + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < NPT; ++c) w[c] = (i0 + c < n) ? row[i0 + c] : WT(0);
  }
}

// Rows of -0.0 (the exact identity of IEEE addition, +0 + -0 = +0 included): the active
// list is padded with them to a whole number of gather groups, so the gather runs without
// per-row predicates or selects and the ordered sum is bitwise unchanged.
#define SPB_NZ8 -0.0, -0.0, -0.0, -0.0, -0.0, -0.0, -0.0, -0.0
#define SPB_NZ64 SPB_NZ8, SPB_NZ8, SPB_NZ8, SPB_NZ8, SPB_NZ8, SPB_NZ8, SPB_NZ8, SPB_NZ8
#define SPB_NZ512 SPB_NZ64, SPB_NZ64, SPB_NZ64, SPB_NZ64, SPB_NZ64, SPB_NZ64, SPB_NZ64, SPB_NZ64
#define SPB_NZ2048 SPB_NZ512, SPB_NZ512, SPB_NZ512, SPB_NZ512
__device__ const double kNegZeroRowF64[REC_MAX_N] = {SPB_NZ2048};
__device__ const float kNegZeroRowF32[REC_MAX_N] = {SPB_NZ2048};

template <typename WT>
__device__ __forceinline__ const WT* neg_zero_row() {
  if constexpr (sizeof(WT) == 8) return reinterpret_cast<const WT*>(kNegZeroRowF64);
  else return reinterpret_cast<const WT*>(kNegZeroRowF32);
}

// this warp's NPT mask words from each lane's NPT spike bits (bit c = neuron NPT*lane + c)
template <int NPT>
__device__ __forceinline__ uint32_t rec_mask_word(uint32_t nib, int lane, int q) {
  constexpr int LPW = 32 / NPT;  // lanes per word
  const uint32_t v = nib << (NPT * (lane % LPW));
  return __reduce_or_sync(0xffffffffu, (lane / LPW == q) ? v : 0u);
}

// WT: the stored weight type (fp32 weights are gathered as fp32 -- half the registers per
// load in flight -- and widened exactly to fp64 before the ordered sum).  Two CTAs per SM
// (<= 64 registers), so the B samples of C3 (256) run as ONE wave on 148 SMs instead of two.
template <int NPT, typename WT, bool VEC>
__global__ void __launch_bounds__(REC_THREADS, NPT <= 2 ? 2 : 1) forward_rec_kernel(
    RecParams P, const double* __restrict__ cur, const void* __restrict__ wrecT,
    double* __restrict__ u_st, double* __restrict__ a_st, double* __restrict__ zbar_st,
    double* __restrict__ zsum_st, uint32_t* __restrict__ raster, float* __restrict__ psis,
    uint32_t* __restrict__ zchunk) {
  __shared__ uint32_t mask[2][REC_MAX_N / 32];
#ifndef SPB_REC_GB
#define SPB_REC_GB 2
#endif
  constexpr int GB = sizeof(WT) == 8 ? SPB_REC_GB / 2 : SPB_REC_GB;   // spikes whose weight loads are in flight
  __shared__ const WT* act[REC_MAX_N + GB];     // active rows of W_rec^T, -0.0 row padded
  __shared__ int nact;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const int n = P.n, nw = (n + 31) >> 5;
  const bool smooth = P.smooth != 0;
  const double theta = P.theta, beta = P.beta, slope = P.slope;
  const float slope_f = (float)P.slope;
  const WT* wt = static_cast<const WT*>(wrecT);
  const int i0 = NPT * tid;            // this thread's first neuron
  const int iv = i0 < n ? i0 : 0;      // its gather offset (idle threads: the row start)
  const int wbase = NPT * warp;        // this warp's first mask word
  double u[NPT], a[NPT], zb[NPT], zs[NPT], dp[NPT];
#pragma unroll
  for (int c = 0; c < NPT; ++c) {
    const int i = i0 + c;
    const bool v = i < n;
    const long long bi = (long long)b * n + i;
    u[c] = (v && P.t0 > 0) ? u_st[bi] : 0.0;
    a[c] = (v && P.t0 > 0) ? a_st[bi] : 0.0;
    zb[c] = (v && P.t0 > 0 && P.pass == 0) ? zbar_st[bi] : 0.0;
    zs[c] = (v && P.t0 > 0 && P.pass == 0) ? zsum_st[bi] : 0.0;
    dp[c] = __dsub_rn(__dsub_rn(u[c], theta), __dmul_rn(beta, a[c]));
  }
  // z_{t0-1} from the carried state (the expression the reference re-evaluates)
  {
    uint32_t nib = 0;
#pragma unroll
    for (int c = 0; c < NPT; ++c)
      if (i0 + c < n && rec_spike(dp[c], smooth, slope) > 0.5) nib |= 1u << c;
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const uint32_t wd = rec_mask_word<NPT>(nib, lane, q);
      if (lane == q && wbase + q < nw) mask[0][wbase + q] = wd;
    }
  }
  float* prow = psis != nullptr ? psis + (long long)b * (P.KR + 1) * n : nullptr;
  if (prow != nullptr) {
#pragma unroll
    for (int c = 0; c < NPT; ++c) {
      const int i = i0 + c;
      if (i < n) prow[i] = surrogate_grad_f32((float)dp[c], slope_f);  // psi_{t0-1}
    }
  }
  __syncthreads();
  uint32_t* zrow = zchunk != nullptr ? zchunk + (long long)b * P.KR * nw : nullptr;
  if (zrow != nullptr)  // chunk row 0 = z_{t0-1}
    for (int w = tid; w < nw; w += REC_THREADS) zrow[w] = mask[0][w];
  const double* crow = cur + (long long)b * P.KR * n;   // sample-aligned rows b*KR + s
  for (int s = 0; s < P.len; ++s) {
    const uint32_t* mprev = mask[s & 1];
    uint32_t* mnext = mask[(s + 1) & 1];
    // input current of this step (exact, from K2), issued before the gather
    double I[NPT];
#pragma unroll
    for (int c = 0; c < NPT; ++c) {
      const int i = i0 + c;
      I[c] = i < n ? __ldcs(crow + (long long)s * n + i) : 0.0;
    }
    // active list of z_{t-1} (ascending), built by warp 0 from the bitmask
    if (tid < 32) {
      int base = 0;
      for (int w0 = 0; w0 < nw; w0 += 32) {
        const int w = w0 + lane;
        uint32_t bits = w < nw ? mprev[w] : 0u;
        const int cnt = __popc(bits);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        int pos = base + incl - cnt;
        while (bits) {
          act[pos++] = wt + (long long)((w << 5) + __ffs(bits) - 1) * n;
          bits &= bits - 1;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
      }
      const int padded = (base + GB - 1) / GB * GB;
      if (base + lane < padded) act[base + lane] = neg_zero_row<WT>();
      if (lane == 0) nact = padded;
    }
    __syncthreads();
    // recurrent current: sum over the active presynaptic j in ascending order, the
    // weight loads of GB spikes in flight at once
    double R[NPT];
#pragma unroll
    for (int c = 0; c < NPT; ++c) R[c] = 0.0;
    const int na = nact;   // a multiple of GB (-0.0 rows at the end)
    for (int q0 = 0; q0 < na; q0 += GB) {
      WT wv[GB][NPT];
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        if constexpr (VEC) {
          // n % NPT == 0: a valid thread's NPT weights lie inside the row; an idle thread
          // (i0 >= n) reads the row start, its sums are never used
          rec_load_row<NPT, WT, VEC>(act[q0 + q] + iv, 0, 1, wv[q]);
        } else {
          rec_load_row<NPT, WT, VEC>(act[q0 + q], i0, n, wv[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < GB; ++q)
#pragma unroll
        for (int c = 0; c < NPT; ++c) R[c] = __dadd_rn(R[c], (double)wv[q][c]);
    }
    float psi[NPT];
    uint32_t nib = 0;
#pragma unroll
    for (int c = 0; c < NPT; ++c) {
      const int i = i0 + c;
      const double z_prev = rec_spike(dp[c], smooth, slope);
      a[c] = __dadd_rn(__dmul_rn(P.rho, a[c]), z_prev);
      u[c] = __dadd_rn(__dmul_rn(P.alpha, u[c]), __dadd_rn(I[c], R[c]));
      if (P.reset) u[c] = __dsub_rn(u[c], __dmul_rn(theta, z_prev));
      const double d = __dsub_rn(__dsub_rn(u[c], theta), __dmul_rn(beta, a[c]));
      const double zv = rec_spike(d, smooth, slope);
      if (P.pass == 0) {
        zb[c] = __dadd_rn(__dmul_rn(P.kappa, zb[c]), zv);
        zs[c] = __dadd_rn(zs[c], zb[c]);
      }
      psi[c] = surrogate_grad_f32((float)d, slope_f);
      dp[c] = d;
      if (zv > 0.5 && i < n) nib |= 1u << c;
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const uint32_t wd = rec_mask_word<NPT>(nib, lane, q);
      const int wi = wbase + q;
      if (lane == q && wi < nw) {
        mnext[wi] = wd;
        if (P.pass == 0 && raster != nullptr)
          raster[((long long)b * P.T + P.t0 + s) * nw + wi] = wd;
        if (zrow != nullptr) zrow[(long long)(s + 1) * nw + wi] = wd;
      }
    }
    if (prow != nullptr) {
#pragma unroll
      for (int c = 0; c < NPT; ++c) {
        const int i = i0 + c;
        if (i < n) prow[(long long)(s + 1) * n + i] = psi[c];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < NPT; ++c) {
    const int i = i0 + c;
    if (i < n) {
      const long long bi = (long long)b * n + i;
      u_st[bi] = u[c];
      a_st[bi] = a[c];
      if (P.pass == 0) {
        zbar_st[bi] = zb[c];
        zsum_st[bi] = zs[c];
      }
    }
  }
}

// x~ operand: row (b, s) of the chunk = [xq row (k bytes) | z_{t0+s-1} bits as n bytes],
// zero padded to Kx; rows s >= len zero.  Warp per row.
__global__ void pack_rec_kernel(const uint8_t* __restrict__ xq, long long xq_sb, long long xq_st,
                                const uint32_t* __restrict__ zchunk, int B, int k, int n, int Tc,
                                int KR, int len, int Kx, uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int nw = (n + 31) >> 5;
  const long long rows = (long long)B * Tc;
  for (long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += (long long)gridDim.x * (blockDim.x >> 5)) {
    const int s = (int)(row % Tc), b = (int)(row / Tc);
    uint8_t* o = out + row * Kx;
    const bool live = s < len;
    const uint8_t* xr = xq + (long long)b * xq_sb + (long long)s * xq_st;
    const uint32_t* zr = zchunk + ((long long)b * KR + s) * nw;
    for (int c = lane; c < Kx; c += 32) {
      uint8_t v = 0;
      if (live) {
        if (c < k) v = xr[c];
        else if (c < k + n) v = (uint8_t)((zr[(c - k) >> 5] >> ((c - k) & 31)) & 1u);
      }
      o[c] = v;
    }
  }
}

}  // namespace spb

using namespace spb;

extern "C" {

int spb_forward_rec_chunk(int pass, const double* cur, const void* wrecT, int w_is_f64, int B,
                          int n, int Tc, int KR, int len, int t0, int T, double alpha,
                          double theta, double slope, double beta, double rho, double kappa,
                          int reset, int alif, int smooth, double* u, double* a, double* zbar,
                          double* zsum, uint32_t* raster, float* psi_scratch, uint32_t* zchunk,
                          cudaStream_t stream) {
  SPB_CHECK_ARG(pass == 0 || pass == 1, "spb_forward_rec_chunk: pass must be 0 (A) or 1 (B)");
  SPB_CHECK_ARG(cur && wrecT && u && a, "spb_forward_rec_chunk: null pointer");
  SPB_CHECK_ARG(pass == 1 || (zbar && zsum), "spb_forward_rec_chunk: pass A needs zbar/zsum");
  SPB_CHECK_ARG(B > 0 && n > 0 && n <= REC_MAX_N && Tc > 0 && len >= 1 && len <= Tc &&
                    KR >= Tc + 1 && t0 >= 0 && t0 + len <= T,
                "spb_forward_rec_chunk: bad sizes (n <= %d)", REC_MAX_N);
  RecParams P{B, n, Tc, KR, len, t0, T, alpha, theta, slope, beta, rho, kappa,
              reset, alif, pass, smooth, w_is_f64};
  const int npt = (n + REC_THREADS - 1) / REC_THREADS;
#define SPB_REC(NPT, WT)                                                                    \
  do {                                                                                      \
    if (n % NPT == 0)                                                                       \
      forward_rec_kernel<NPT, WT, true><<<B, REC_THREADS, 0, stream>>>(                     \
          P, cur, wrecT, u, a, zbar, zsum, raster, psi_scratch, zchunk);                    \
    else                                                                                    \
      forward_rec_kernel<NPT, WT, false><<<B, REC_THREADS, 0, stream>>>(                    \
          P, cur, wrecT, u, a, zbar, zsum, raster, psi_scratch, zchunk);                    \
  } while (0)
  if (w_is_f64) {
    if (npt <= 1) SPB_REC(1, double);
    else if (npt <= 2) SPB_REC(2, double);
    else SPB_REC(4, double);
  } else {
    if (npt <= 1) SPB_REC(1, float);
    else if (npt <= 2) SPB_REC(2, float);
    else SPB_REC(4, float);
  }
#undef SPB_REC
  SPB_CHECK_LAUNCH("forward_rec");
  return 0;
}

int spb_pack_rec(const uint8_t* xq, long long xq_sb, long long xq_st, const uint32_t* zchunk,
                 int B, int k, int n, int Tc, int KR, int len, int Kx, uint8_t* out,
                 cudaStream_t stream) {
  SPB_CHECK_ARG(xq && zchunk && out && B > 0 && k > 0 && n > 0 && Kx >= k + n && len >= 0 &&
                    len <= Tc && KR >= Tc + 1,
                "spb_pack_rec: bad args");
  const long long rows = (long long)B * Tc;
  const long long want = (rows + 7) / 8;
  const int blocks = (int)(want < 148LL * 16 ? want : 148LL * 16);
  pack_rec_kernel<<<blocks, 256, 0, stream>>>(xq, xq_sb, xq_st, zchunk, B, k, n, Tc, KR, len, Kx,
                                              out);
  SPB_CHECK_LAUNCH("pack_rec");
  return 0;
}

}  // extern "C"
