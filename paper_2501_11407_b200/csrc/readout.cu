// Readout, loss and learning signal (sm_100a):
//   K3  spb_readout_loss  -- s = W_out zsum (the time-summed leaky readout,
//                            gradients.py:163-164), softmax cross-entropy
//                            (gradients.py:66-75), g = softmax - onehot,
//                            w_sig = W_out^T g (gradients.py:178)
//   K7  spb_readout_grad  -- grad W_out = sum_b g_b (x) zsum_b (gradients.py:181), written
//   --  spb_finalize_grad -- fp64 gradient accumulator -> caller dtype, padding dropped
#include <algorithm>

#include "common.cuh"

#ifndef K3_SB
#define K3_SB 2  // samples per K3 CTA (A/B builds: -DK3_SB=1)
#endif

namespace spb {

// SB samples per CTA: every W_out element loaded serves SB samples (W_out is re-read from
// L2 by every CTA; at one sample per CTA that stream was most of K3's time inside the
// update).  Per sample the arithmetic and its order are those of one sample per CTA.
template <int SB>
__global__ void readout_loss_kernel(const double* __restrict__ wout, const double* __restrict__ zsum,
                                    const long long* __restrict__ labels, int B, int n, int m,
                                    double* __restrict__ s_out, double* __restrict__ loss,
                                    double* __restrict__ g_out, float* __restrict__ wsig,
                                    int* __restrict__ correct) {
  pdl_enter();
  extern __shared__ double sm[];  // [SB][m] logits + [SB][m] g (exps, then dL/ds)
  const int b0 = blockIdx.x * SB;
  const int nb = min(SB, B - b0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  // one warp per class (round robin): s_c = sum_i W_out[c][i] zsum[b][i], no block barriers
  for (int c = warp; c < m; c += nwarps) {
    const double* wr = wout + (long long)c * n;
    double a0[SB], a1[SB];
#pragma unroll
    for (int q = 0; q < SB; ++q) a0[q] = a1[q] = 0.0;
    const double* z[SB];
#pragma unroll
    for (int q = 0; q < SB; ++q) z[q] = zsum + (long long)(b0 + (q < nb ? q : 0)) * n;
    int i = lane;
#pragma unroll 4
    for (; i + 32 < n; i += 64) {
      const double w0 = wr[i], w1 = wr[i + 32];
#pragma unroll
      for (int q = 0; q < SB; ++q) {
        a0[q] = fma(w0, z[q][i], a0[q]);
        a1[q] = fma(w1, z[q][i + 32], a1[q]);
      }
    }
    if (i < n) {
      const double w0 = wr[i];
#pragma unroll
      for (int q = 0; q < SB; ++q) a0[q] = fma(w0, z[q][i], a0[q]);
    }
#pragma unroll
    for (int q = 0; q < SB; ++q) {
      double acc = a0[q] + a1[q];
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) sm[q * m + c] = acc;
    }
  }
  __syncthreads();
  // softmax cross-entropy (warp q: sample b0 + q): the exps run one class per lane; the
  // max, the first argmax and the sum of exps are taken in class order by one lane (the
  // reference's order)
  if (warp < nb) {
    const int b = b0 + warp;
    double* s = sm + warp * m;
    double* g = sm + (SB + warp) * m;
    // an out-of-range label (the host wrappers reject them: LabelOutOfRange) yields a NaN
    // loss and no one-hot term instead of an out-of-bounds shared-memory read
    const long long yl = labels[b];
    const bool ybad = yl < 0 || yl >= m;
    const int y = ybad ? -1 : (int)yl;
    double mx = s[0];
    int arg = 0;
    if (lane == 0) {
      for (int c = 1; c < m; ++c)
        if (s[c] > mx) { mx = s[c]; arg = c; }
    }
    mx = __shfl_sync(0xffffffffu, mx, 0);
    for (int c = lane; c < m; c += 32) g[c] = exp(s[c] - mx);
    __syncwarp();
    double logz = 0.0;
    if (lane == 0) {
      double se = 0.0;
      for (int c = 0; c < m; ++c) se += g[c];
      logz = log(se);
      loss[b] = ybad ? __longlong_as_double(0x7ff8000000000000ULL) : logz - (s[y] - mx);
      if (correct) correct[b] = (arg == y) ? 1 : 0;
    }
    logz = __shfl_sync(0xffffffffu, logz, 0);
    __syncwarp();
    for (int c = lane; c < m; c += 32) {
      const double gc = exp((s[c] - mx) - logz) - (c == y ? 1.0 : 0.0);
      g[c] = gc;
      s_out[(long long)b * m + c] = s[c];
      g_out[(long long)b * m + c] = gc;
    }
  }
  __syncthreads();
  const double* g = sm + SB * m;
  for (int i = tid; i < n; i += blockDim.x) {
    double acc[SB];
#pragma unroll
    for (int q = 0; q < SB; ++q) acc[q] = 0.0;
    for (int c = 0; c < m; ++c) {
      const double w = wout[(long long)c * n + i];
#pragma unroll
      for (int q = 0; q < SB; ++q) acc[q] = fma(w, g[q * m + c], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < SB; ++q)
      if (q < nb) wsig[(long long)(b0 + q) * n + i] = (float)acc[q];
  }
}

// gwo[c][i] = sum_b g[b][c] zsum[b][i]: block = 32 neurons x 8 batch slices (contiguous
// sample ranges), each slice summed in order, the 8 slice sums added in slice order --
// deterministic, and 8x the parallelism of one thread per (c, i).
constexpr int RG_SLICES = 8;
__global__ void __launch_bounds__(32 * RG_SLICES) readout_grad_kernel(
    const double* __restrict__ g, const double* __restrict__ zsum, int B, int n, int m,
    double* __restrict__ gwo) {
  __shared__ double part[RG_SLICES][33];
  const int lane = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const int c = blockIdx.y;
  const int per = (B + RG_SLICES - 1) / RG_SLICES;
  const int b0 = sl * per, b1 = min(B, b0 + per);
  double a0 = 0.0, a1 = 0.0;
  if (i < n) {
    int b = b0;
    for (; b + 1 < b1; b += 2) {
      a0 = fma(g[(long long)b * m + c], zsum[(long long)b * n + i], a0);
      a1 = fma(g[(long long)(b + 1) * m + c], zsum[(long long)(b + 1) * n + i], a1);
    }
    if (b < b1) a0 = fma(g[(long long)b * m + c], zsum[(long long)b * n + i], a0);
  }
  part[sl][lane] = a0 + a1;
  __syncthreads();
  if (sl == 0 && i < n) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < RG_SLICES; ++q) acc += part[q][lane];
    gwo[(long long)c * n + i] = acc;
  }
}

template <typename OT>
__global__ void finalize_kernel(const double* __restrict__ acc, int rows, int cols, int ld,
                                OT* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)rows * cols) return;
  const int r = (int)(idx / cols), c = (int)(idx % cols);
  out[idx] = (OT)acc[(long long)r * ld + c];
}

// Allreduce payload in one launch: [grad W (acc[:, :k]) | grad W_out | sum loss | #correct]
// in the payload dtype; block 0 also sums the B losses and correct flags in sample order.
template <typename OT>
__global__ void pack_grads_kernel(const double* __restrict__ acc, int n, int k, int ld,
                                  const double* __restrict__ gwo, int m,
                                  const double* __restrict__ loss, const int* __restrict__ correct,
                                  int B, OT* __restrict__ out) {
  const long long nk = (long long)n * k, total = nk + (long long)m * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    if (idx < nk) {
      const int r = (int)(idx / k), c = (int)(idx - (long long)r * k);
      out[idx] = (OT)acc[(long long)r * ld + c];
    } else {
      out[idx] = (OT)gwo[idx - nk];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double ls = 0.0;
    long long nc = 0;
    for (int b = 0; b < B; ++b) {
      ls += loss[b];
      nc += correct[b];
    }
    out[total] = (OT)ls;
    out[total + 1] = (OT)nc;
  }
}

}  // namespace spb

using namespace spb;

extern "C" {

int spb_readout_loss(const double* wout, const double* zsum, const long long* labels, int B, int n,
                     int m, double* s_out, double* loss, double* g, float* wsig, int* correct,
                     cudaStream_t stream) {
  SPB_CHECK_ARG(wout && zsum && labels && s_out && loss && g && wsig,
                "spb_readout_loss: null pointer");
  SPB_CHECK_ARG(B > 0 && n > 0 && m > 0 && m <= 4096, "spb_readout_loss: bad sizes");
  // K3_SB samples per CTA (W_out read once per CTA for all of them) when that still
  // leaves >= 64 CTAs; small batches keep one sample per CTA
  constexpr int SB = K3_SB;
  const bool multi = SB > 1 && B >= 64 * SB;
  const int sb = multi ? SB : 1;
  const size_t smem = (size_t)(2 * sb * m + 32) * sizeof(double);
  // one warp per class (up to 32 warps): the class dot products run in one round
  const int threads = 32 * (m < 8 ? 8 : (m > 32 ? 32 : m));
  auto kfn = multi ? readout_loss_kernel<SB> : readout_loss_kernel<1>;
  if (smem > 48 * 1024) {  // large m: opt in to the larger dynamic shared memory
    const cudaError_t e =
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    SPB_CHECK_ARG(e == cudaSuccess, "spb_readout_loss: smem opt-in failed: %s",
                  cudaGetErrorString(e));
  }
  pdl_launch(kfn, (B + sb - 1) / sb, threads, smem, stream, wout, zsum, labels, B, n, m, s_out,
             loss, g, wsig, correct);
  SPB_CHECK_LAUNCH("readout_loss");
  return 0;
}

int spb_readout_grad(const double* g, const double* zsum, int B, int n, int m, double* gwo,
                     cudaStream_t stream) {
  SPB_CHECK_ARG(g && zsum && gwo, "spb_readout_grad: null pointer");
  SPB_CHECK_ARG(B > 0 && n > 0 && m > 0, "spb_readout_grad: bad sizes");
  dim3 grid(ceil_div(n, 32), m);
  readout_grad_kernel<<<grid, 32 * RG_SLICES, 0, stream>>>(g, zsum, B, n, m, gwo);
  SPB_CHECK_LAUNCH("readout_grad");
  return 0;
}

int spb_pack_grads(const double* acc, int n, int k, int ld, const double* gwo, int m,
                   const double* loss, const int* correct, int B, void* out, int out_is_f64,
                   cudaStream_t stream) {
  SPB_CHECK_ARG(acc && gwo && loss && correct && out && n > 0 && k > 0 && ld >= k && m > 0 && B > 0,
                "spb_pack_grads: bad args");
  const long long total = (long long)n * k + (long long)m * n;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148 * 8);
  if (out_is_f64)
    pack_grads_kernel<double><<<blocks, 256, 0, stream>>>(acc, n, k, ld, gwo, m, loss, correct, B,
                                                          (double*)out);
  else
    pack_grads_kernel<float><<<blocks, 256, 0, stream>>>(acc, n, k, ld, gwo, m, loss, correct, B,
                                                         (float*)out);
  SPB_CHECK_LAUNCH("pack_grads");
  return 0;
}

int spb_finalize_grad(const double* acc, int rows, int cols, int ld, void* out, int out_is_f64,
                      cudaStream_t stream) {
  SPB_CHECK_ARG(acc && out && rows > 0 && cols > 0 && ld >= cols, "spb_finalize_grad: bad args");
  const long long total = (long long)rows * cols;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (out_is_f64)
    finalize_kernel<double><<<blocks, 256, 0, stream>>>(acc, rows, cols, ld, (double*)out);
  else
    finalize_kernel<float><<<blocks, 256, 0, stream>>>(acc, rows, cols, ld, (float*)out);
  SPB_CHECK_LAUNCH("finalize_grad");
  return 0;
}

}  // extern "C"
