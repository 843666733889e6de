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
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace spb {

struct FwdParams {
  int B, n, Tc, KR, len, t0, T;
  double alpha, theta, slope, beta, rho, kappa;
  int reset, alif, pass;  // pass 0 = A, 1 = B
  int smooth;             // 1: spikes are surrogate_smooth(d) (graph.py:45-47), not Theta(d)
};


constexpr int K1_THREADS = 128;  // 4 warps = 128 consecutive neurons of one sample

// ------------------------------------------------------------------------------------
// K1.  Warp = 32 consecutive neurons of one sample.  State u, a and the current are fp64
// so spike decisions match the f64 reference; every multiply/add of the
// state update mirrors the reference's operation order with explicit round-to-nearest
// intrinsics (no FMA contraction).  Pass B parks psi of the chunk in a global scratch
// ([b][rho][i], coalesced; L2-resident for the scan that immediately reads it back) so the
// kernel runs at full occupancy; the backward scan runs in fp32 (every quantity it
// produces feeds the fp32 / bf16-split gradient path).
// ------------------------------------------------------------------------------------
// Templated on the per-launch flags so the per-step loop carries no flag branches and
// walks its current / psi rows with pointer increments (the kernel is instruction-bound:
// ~70 issued instructions per neuron-step before this specialisation).
// (7 CTAs per SM, <= 73 registers: 2048 CTAs at C3 are two full waves; measured better
// than 6 once K4 no longer shares the SMs: C3 K1 0.151 -> 0.147 ms)
template <bool PASSA, bool PARK, bool RESET, bool SMOOTH>
__global__ void __launch_bounds__(K1_THREADS, 7) forward_chunk_kernel(
    FwdParams P, const double* __restrict__ cur, double* __restrict__ u_st,
    double* __restrict__ a_st, double* __restrict__ zbar_st, double* __restrict__ zsum_st,
    uint32_t* __restrict__ raster, const float* __restrict__ wsig, float* __restrict__ psis) {
  pdl_enter();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // CTA = one sample x 128 consecutive neurons: every step it streams 1 KB of current
  // and writes 512 B of psi contiguously (DRAM-friendly), warp = 32 neurons
  const int wbase = blockIdx.x * K1_THREADS + warp * 32;
  const int i = wbase + lane;
  const bool valid_i = i < P.n;
  const int b = blockIdx.y;
  if (wbase >= P.n) return;  // warp-uniform; no block-level barriers below
  const long long bi = (long long)b * P.n + i;
  double u = 0.0, a = 0.0, zbar = 0.0, zsum = 0.0;  // t0 == 0: fresh state (no read)
  if (valid_i && P.t0 > 0) {
    u = u_st[bi];
    a = a_st[bi];
    if (PASSA) {
      zbar = zbar_st[bi];
      zsum = zsum_st[bi];
    }
  }
  const double theta = P.theta, beta = P.beta, alpha = P.alpha, rho = P.rho, kappa = P.kappa;
  const int n = P.n;
  const int nw = (n + 31) >> 5;
  // invalid lanes read a valid address (their own row start) and discard the value
  // current rows are sample-aligned: row b*KR + s (K2's layout)
  const double* cp = cur + (long long)b * P.KR * n + (valid_i ? i : wbase);
  // d_prev of step t is the drive d of step t-1 (the reference recomputes the same
  // expression from the same state, gradients.py:159): carry it.
  double d_prev = __dsub_rn(__dsub_rn(u, theta), __dmul_rn(beta, a));
  const float slope = (float)P.slope;
  const double slope_d = P.slope;
  // psi of row rho at prow[rho*n] (pass B; optional in pass A, which lets a one-chunk
  // sequence skip the pass-B dynamics entirely)
  const bool park = PARK && valid_i;
  float* pp = PARK ? psis + (long long)b * (P.KR + 1) * n + (valid_i ? i : wbase) : nullptr;
  if (park) pp[0] = surrogate_grad_f32((float)d_prev, slope);  // psi_{t0-1}
  uint32_t* rp = (PASSA && raster != nullptr)
                     ? raster + ((long long)b * P.T + P.t0) * nw + (wbase >> 5) : nullptr;
  const int len = P.len;
  // software pipeline: the current of steps s8+8..s8+15 is in flight while steps
  // s8..s8+7 integrate (16 outstanding 8-byte loads per thread).  Blocks of 8 steps that
  // lie entirely inside the chunk run without per-step bounds checks (the guards were a
  // third of the loop's integer instructions; the kernel is issue-bound).
  auto step = [&](double I) {
    // gradients.py:121-129 (u - theta - beta*a evaluates as (u - theta) - (beta*a))
    const double z_prev = spike_value(d_prev, SMOOTH, slope_d);
    a = __dadd_rn(__dmul_rn(rho, a), z_prev);
    u = __dadd_rn(__dmul_rn(alpha, u), I);
    if (RESET) u = __dsub_rn(u, __dmul_rn(theta, z_prev));
    const double d = __dsub_rn(__dsub_rn(u, theta), __dmul_rn(beta, a));
    if (PASSA) {
      const double zv = spike_value(d, SMOOTH, slope_d);
      zbar = __dadd_rn(__dmul_rn(kappa, zbar), zv);
      zsum = __dadd_rn(zsum, zbar);
      // raster = z > 0.5 (gradients.py:362)
      const unsigned bal = __ballot_sync(0xffffffffu, zv > 0.5 && valid_i);
      if (rp != nullptr) {
        if (lane == 0) rp[0] = bal;
        rp += nw;
      }
    }
    // the surrogate only scales fp32 eligibilities: evaluate it in fp32
    if (PARK) {
      pp += n;
      if (park) pp[0] = surrogate_grad_f32((float)d, slope);
    }
    d_prev = d;
  };
  double In[8];
  if (len >= 8) {
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) In[u8] = __ldcs(cp + (long long)u8 * n);
  } else {
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) In[u8] = u8 < len ? __ldcs(cp + (long long)u8 * n) : 0.0;
  }
  const long long n8 = 8LL * n;
  const int full = len & ~7;   // steps in complete blocks of 8
  int s8 = 0;
  for (; s8 < full; s8 += 8) {
    double Ib[8];
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) Ib[u8] = In[u8];
    cp += n8;
    if (s8 + 16 <= len) {
#pragma unroll
      for (int u8 = 0; u8 < 8; ++u8) In[u8] = __ldcs(cp + (long long)u8 * n);
    } else {
#pragma unroll
      for (int u8 = 0; u8 < 8; ++u8)
        In[u8] = (s8 + 8 + u8 < len) ? __ldcs(cp + (long long)u8 * n) : 0.0;
    }
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) step(Ib[u8]);
  }
  // the last partial block (its current is already in In)
#pragma unroll
  for (int u8 = 0; u8 < 7; ++u8)
    if (s8 + u8 < len) step(In[u8]);
  if (valid_i) {
    u_st[bi] = u;
    a_st[bi] = a;
    if (PASSA) {
      zbar_st[bi] = zbar;
      zsum_st[bi] = zsum;
    }
  }
}

template <bool PASSA, bool PARK>
static void launch_forward(const FwdParams& P, dim3 grid, cudaStream_t stream, const double* cur,
                           double* u, double* a, double* zbar, double* zsum, uint32_t* raster,
                           const float* wsig, float* psis) {
  const bool reset = P.reset != 0, smooth = P.smooth != 0;
#define SPB_K1(R, S)                                                                          \
  pdl_launch(forward_chunk_kernel<PASSA, PARK, R, S>, grid, K1_THREADS, 0, stream, P, cur, u, a, \
             zbar, zsum, raster, wsig, psis)
  if (reset && smooth) SPB_K1(true, true);
  else if (reset) SPB_K1(true, false);
  else if (smooth) SPB_K1(false, true);
  else SPB_K1(false, false);
#undef SPB_K1
}

// ------------------------------------------------------------------------------------
// K1s: backward scan over one chunk (pass B).  Thread = (sample, 2 neighbouring neurons):
// it reads the psi rows K1 parked in the scratch (float2, coalesced, 4 rows prefetched)
// from rho = L down to 0 and emits the GEMM operands MN-major -- C[b*KR + rho][i] and,
// when the trace has to be carried to a next chunk, W -- as bf16x2 hi/lo pairs, i.e.
// 128-byte coalesced stores per warp and row.  fp32 throughout (every output feeds the
// fp32 / bf16-split gradient path).
// ------------------------------------------------------------------------------------
constexpr int K1S_THREADS = 128;  // 4 warps = 256 consecutive neurons of one sample


// FILT (pass 3, one fresh chunk, reset = 0): the presynaptic filter is folded into the
// coefficients -- sum_rho C_rho xbar_{rho-1} = sum_rho Ct_rho x_{rho-1} (+ Ct_0 xbar_{-1}
// = 0) with Ct_rho = C_rho + alpha Ct_{rho+1} -- so the gradient GEMM runs on the RAW
// spikes, exact in bf16 (2 MMAs instead of 3, half the operand bytes, no filter kernel).
// (7 CTAs per SM, <= 73 registers: the C3 grid of B x n/256 = 1024 CTAs is one wave;
// blocks of 8 rows -- 12 or 16 spill and measured slower: C3 0.7036 vs 0.715 / 0.733 ms)
#ifndef SCAN_BLK
#define SCAN_BLK 8
#endif
#ifndef SCAN_OCC
#define SCAN_OCC 7
#endif
template <bool ALIF, bool CARRY, bool FILT = false>
__global__ void __launch_bounds__(K1S_THREADS, SCAN_OCC) chunk_scan_kernel(
    FwdParams P, const float* __restrict__ wsig, const float* __restrict__ ctab,
    uint32_t* __restrict__ c_hi, uint32_t* __restrict__ c_lo, uint32_t* __restrict__ w_hi,
    uint32_t* __restrict__ w_lo, int ldc, float2* __restrict__ mdt,
    const float* __restrict__ psis) {
  pdl_enter();
  pdl_trigger();
  extern __shared__ float cs[];  // cs[r] = c_{t0+r-1}, r = 0..L
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = P.len;
  for (int r = threadIdx.x; r <= L; r += K1S_THREADS)
    cs[r] = (P.t0 + r - 1 >= 0) ? ctab[P.t0 + r - 1] : 0.f;
  __syncthreads();
  const int i = blockIdx.x * 2 * K1S_THREADS + warp * 64 + 2 * lane;  // neurons i, i+1
  // samples in reverse launch order: K1 parked the psi of the last samples most recently,
  // so the first scan CTAs find it in L2
  const int b = (int)gridDim.y - 1 - (int)blockIdx.y;
  if (b >= P.B || i >= P.n) return;
  const int n = P.n;
  const bool has2 = i + 1 < n;
  const long long bi = (long long)b * n + i;
  const float ws0 = wsig[bi], ws1 = has2 ? wsig[bi + 1] : 0.f;
  const float beta = (float)P.beta, rho = (float)P.rho;
  const float* prow = psis + (long long)b * (P.KR + 1) * n + i;
  const bool vec = has2 && (n & 1) == 0;  // float2 rows are 8-byte aligned only for even n
  auto ldpsi = [&](int r) -> float2 {
    if (r < 0) return make_float2(0.f, 0.f);
    const float* q = prow + (long long)r * n;
    if (vec) return __ldcs(reinterpret_cast<const float2*>(q));
    return make_float2(__ldcs(q), has2 ? __ldcs(q + 1) : 0.f);
  };
  const long long ld2 = ldc >> 1;  // row stride in bf16x2 words
  const long long row0 = (long long)b * P.KR * ld2 + (i >> 1);
  uint32_t* chp = c_hi + row0;
  uint32_t* clp = c_lo + row0;
  uint32_t* whp = CARRY ? w_hi + row0 : nullptr;
  uint32_t* wlp = CARRY ? w_lo + row0 : nullptr;
  for (int r = P.KR - 1; r > L; --r) {  // rows past the chunk
    chp[r * ld2] = 0u;
    clp[r * ld2] = 0u;
    if (CARRY) { whp[r * ld2] = 0u; wlp[r * ld2] = 0u; }
  }
  // walk the rows backwards with pointer decrements; PF psi rows in flight per thread
  chp += L * ld2;
  clp += L * ld2;
  if (CARRY) { whp += L * ld2; wlp += L * ld2; }
  float lam0 = 0.f, dcum0 = 1.f, an0 = 0.f, lam1 = 0.f, dcum1 = 1.f, an1 = 0.f;
  float ft0 = 0.f, ft1 = 0.f, fw0 = 0.f, fw1 = 0.f;  // FILT: running Ct, Wt
  const float falpha = (float)P.alpha;
  // one row r (psi row r = psi_{r-1}); MID: 1 <= r < L, i.e. no boundary case -- rows L
  // and 0 and the last partial block take the checked path
  float2 up = make_float2(0.f, 0.f);  // psi row r+1
  auto row = [&](const int r, const float2 cur, auto mid_tag) {
    constexpr bool MID = decltype(mid_tag)::value;
    const float c_prev = cs[r];
    const float c_r = (MID || r < L) ? cs[r + 1] : 0.f;
    // L_{r-1} psi_{r-1} (row r >= 1) [+ R_r = P_r Lambda_r, ALIF]; W_r = P_r D(L-1, r)
    float c0 = (MID || r >= 1) ? c_prev * ws0 * cur.x : 0.f;
    float c1 = (MID || r >= 1) ? c_prev * ws1 * cur.y : 0.f;
    float w0 = 0.f, w1 = 0.f;
    if (ALIF && (MID || r < L)) {
      const float A0 = fmaf(-beta, cur.x, rho), A1 = fmaf(-beta, cur.y, rho);
      lam0 = fmaf(an0, lam0, -beta * (c_r * ws0 * up.x));
      lam1 = fmaf(an1, lam1, -beta * (c_r * ws1 * up.y));
      c0 = fmaf(cur.x, lam0, c0);
      c1 = fmaf(cur.y, lam1, c1);
      w0 = cur.x * dcum0;
      w1 = cur.y * dcum1;
      dcum0 *= A0;
      dcum1 *= A1;
      an0 = A0;
      an1 = A1;
    }
    if (FILT) {
      ft0 = fmaf(falpha, ft0, c0);
      ft1 = fmaf(falpha, ft1, c1);
      c0 = ft0;
      c1 = ft1;
      if (CARRY) {  // the carry GEMM runs on the raw spikes too
        fw0 = fmaf(falpha, fw0, w0);
        fw1 = fmaf(falpha, fw1, w1);
        w0 = fw0;
        w1 = fw1;
      }
    }
    uint32_t h, l;
    split_bf16x2(c0, c1, h, l);
    *chp = h;
    *clp = l;
    chp -= ld2;
    clp -= ld2;
    if (CARRY) {
      split_bf16x2(w0, w1, h, l);
      *whp = h;
      *wlp = l;
      whp -= ld2;
      wlp -= ld2;
    }
    up = cur;
  };
  using checked = std::integral_constant<bool, false>;
  using mid = std::integral_constant<bool, true>;
  row(L, ldpsi(L), checked{});
  // rows L-1 .. 1 in blocks of SCAN_BLK: the next block's psi loads are issued before
  // this block is processed (1-2 blocks in flight per thread, no register shifting);
  // complete blocks run without per-row boundary checks (the loop is issue-bound)
  int r8 = L - 1;
  float2 nxt[SCAN_BLK];
#pragma unroll
  for (int u = 0; u < SCAN_BLK; ++u) nxt[u] = ldpsi(r8 - u);
  for (; r8 - (SCAN_BLK - 1) >= 1; r8 -= SCAN_BLK) {
    float2 blk[SCAN_BLK];
#pragma unroll
    for (int u = 0; u < SCAN_BLK; ++u) blk[u] = nxt[u];
#pragma unroll
    for (int u = 0; u < SCAN_BLK; ++u) nxt[u] = ldpsi(r8 - SCAN_BLK - u);
#pragma unroll
    for (int u = 0; u < SCAN_BLK; ++u) row(r8 - u, blk[u], mid{});
  }
  // the last rows (r8 .. 0, at most SCAN_BLK of them, already loaded)
#pragma unroll
  for (int u = 0; u < SCAN_BLK; ++u)
    if (r8 - u >= 0) row(r8 - u, nxt[u], checked{});
  if (ALIF && mdt != nullptr) {  // M also feeds the last chunk's inter-chunk term
    mdt[bi] = make_float2(an0 * lam0, dcum0);  // M = A_0 Lambda_0, Dt = prod A
    if (has2) mdt[bi + 1] = make_float2(an1 * lam1, dcum1);
  }
}

// ------------------------------------------------------------------------------------
// K1s on time segments: the same outputs as chunk_scan_kernel with S = 4 warps per 64
// neurons, warp s scanning rows [lo_s, hi_s] of the chunk -- 4x the warps in flight for
// the same bytes (the one-warp-per-64-neurons scan is latency-bound at small B*n).  The
// ALIF recursion lam_r = A_{r+1} lam_{r+1} + q_r is linear in the value entering a
// segment, so a first sweep gives each segment its local bottom value (entry 0), the
// product G of its A factors and the product D of its carry factors; the segments then
// meet in shared memory (top segment first, fixed order) and a second sweep emits the
// rows.  fp32 results equal the sequential scan's up to fp32 rounding.
// ------------------------------------------------------------------------------------
constexpr int SEG = 4;

// FILT as in chunk_scan_kernel (LIF only here: Ct is linear in the segment entry, so a
// first sweep gives each segment its local bottom value and alpha^rows).
template <bool ALIF, bool CARRY, bool FILT = false>
__global__ void __launch_bounds__(SEG * 32) chunk_scan_seg_kernel(
    FwdParams P, const float* __restrict__ wsig, const float* __restrict__ ctab,
    uint32_t* __restrict__ c_hi, uint32_t* __restrict__ c_lo, uint32_t* __restrict__ w_hi,
    uint32_t* __restrict__ w_lo, int ldc, float2* __restrict__ mdt,
    const float* __restrict__ psis) {
  extern __shared__ float cs[];  // cs[r] = c_{t0+r-1}, r = 0..L
  __shared__ float2 sh_l[SEG][32], sh_g[SEG][32], sh_d[SEG][32];
  const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
  const int L = P.len;
  for (int r = threadIdx.x; r <= L; r += SEG * 32)
    cs[r] = (P.t0 + r - 1 >= 0) ? ctab[P.t0 + r - 1] : 0.f;
  const int i = blockIdx.x * 64 + 2 * lane;  // neurons i, i+1
  const int b = blockIdx.y;
  const int n = P.n;
  const bool live = i < n;
  const bool has2 = i + 1 < n;
  const long long bi = (long long)b * n + i;
  const float ws0 = live ? wsig[bi] : 0.f, ws1 = has2 ? wsig[bi + 1] : 0.f;
  const float beta = (float)P.beta, rho = (float)P.rho;
  const float* prow = psis + (long long)b * (P.KR + 1) * n + (live ? i : 0);
  const bool vec = has2 && (n & 1) == 0;
  auto ldpsi = [&](int r) -> float2 {
    if (r < 0 || r > L || !live) return make_float2(0.f, 0.f);
    const float* q = prow + (long long)r * n;
    if (vec) return __ldcg(reinterpret_cast<const float2*>(q));
    return make_float2(__ldcg(q), has2 ? __ldcg(q + 1) : 0.f);
  };
  // rows [lo, hi] of this warp's segment (top segment ends at L)
  const int per = (L + 1 + SEG - 1) / SEG;
  const int lo = seg * per, hi = min(L, lo + per - 1);
  const long long ld2 = ldc >> 1;
  const long long row0 = (long long)b * P.KR * ld2 + (i >> 1);
  // rows past the chunk: zero (spread over the warps)
  for (int r = L + 1 + seg; r < P.KR; r += SEG)
    if (live) {
      c_hi[row0 + r * ld2] = 0u;
      c_lo[row0 + r * ld2] = 0u;
      if (CARRY) { w_hi[row0 + r * ld2] = 0u; w_lo[row0 + r * ld2] = 0u; }
    }
  // entry state of the segment: row hi+1's psi and A (none above the top row L)
  const float2 up0 = (hi < L) ? ldpsi(hi + 1) : make_float2(0.f, 0.f);
  const float an0_in = (ALIF && hi < L && hi + 1 < L) ? fmaf(-beta, up0.x, rho) : 0.f;
  const float an1_in = (ALIF && hi < L && hi + 1 < L) ? fmaf(-beta, up0.y, rho) : 0.f;
  float lam0 = 0.f, lam1 = 0.f, dcum0 = 1.f, dcum1 = 1.f;
  __syncthreads();  // cs
  if (ALIF && lo <= hi) {
    // sweep 1: local bottom value, G = prod of the A's applied to the entry, D = prod A_r
    float l0 = 0.f, l1 = 0.f, g0 = 1.f, g1 = 1.f, d0 = 1.f, d1 = 1.f;
    float an0 = an0_in, an1 = an1_in;
    float2 up = up0;
    float2 nx1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) nx1[u] = (hi - u >= lo) ? ldpsi(hi - u) : make_float2(0.f, 0.f);
    for (int r8 = hi; r8 >= lo; r8 -= 8) {
      float2 bk1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) bk1[u] = nx1[u];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        nx1[u] = (r8 - 8 - u >= lo) ? ldpsi(r8 - 8 - u) : make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
      const int r = r8 - u;
      if (r < lo) break;
      const float2 cur = bk1[u];
      if (r < L) {
        const float c_r = cs[r + 1];
        const float A0 = fmaf(-beta, cur.x, rho), A1 = fmaf(-beta, cur.y, rho);
        l0 = fmaf(an0, l0, -beta * (c_r * ws0 * up.x));
        l1 = fmaf(an1, l1, -beta * (c_r * ws1 * up.y));
        g0 *= an0;
        g1 *= an1;
        d0 *= A0;
        d1 *= A1;
        an0 = A0;
        an1 = A1;
      }
      up = cur;
      }
    }
    sh_l[seg][lane] = make_float2(l0, l1);
    sh_g[seg][lane] = make_float2(g0, g1);
    sh_d[seg][lane] = make_float2(d0, d1);
  }
  static_assert(!(FILT && ALIF), "segmented FILT scan is LIF only");
  const float falpha = (float)P.alpha;
  float ft0 = 0.f, ft1 = 0.f;
  if (FILT) {
    if (lo <= hi) {  // sweep 1: this segment's Ct at row lo from a zero entry, alpha^rows
      float f0 = 0.f, f1 = 0.f, ap = 1.f;
      float2 nx1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) nx1[u] = (hi - u >= lo) ? ldpsi(hi - u) : make_float2(0.f, 0.f);
      for (int r8 = hi; r8 >= lo; r8 -= 8) {
        float2 bk1[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) bk1[u] = nx1[u];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          nx1[u] = (r8 - 8 - u >= lo) ? ldpsi(r8 - 8 - u) : make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
        const int r = r8 - u;
        if (r < lo) break;
        const float2 cur = bk1[u];
        const float c_prev = cs[r];
        const float c0 = r >= 1 ? c_prev * ws0 * cur.x : 0.f;
        const float c1 = r >= 1 ? c_prev * ws1 * cur.y : 0.f;
        f0 = fmaf(falpha, f0, c0);
        f1 = fmaf(falpha, f1, c1);
        ap *= falpha;
        }
      }
      sh_l[seg][lane] = make_float2(f0, f1);
      sh_g[seg][lane] = make_float2(ap, ap);
    }
    __syncthreads();
    for (int q = SEG - 1; q > seg; --q) {  // the segments above, top first
      const int qlo = q * per, qhi = min(L, qlo + per - 1);
      if (qlo > qhi) continue;
      const float2 gl = sh_l[q][lane], gg = sh_g[q][lane];
      ft0 = fmaf(gg.x, ft0, gl.x);
      ft1 = fmaf(gg.y, ft1, gl.y);
    }
  }
  if (ALIF) {
    __syncthreads();
    // entry of this segment: the segments above, top first (fixed order)
    for (int q = SEG - 1; q > seg; --q) {
      const int qlo = q * per, qhi = min(L, qlo + per - 1);
      if (qlo > qhi) continue;
      const float2 gl = sh_l[q][lane], gg = sh_g[q][lane], gd = sh_d[q][lane];
      lam0 = fmaf(gg.x, lam0, gl.x);
      lam1 = fmaf(gg.y, lam1, gl.y);
      dcum0 *= gd.x;
      dcum1 *= gd.y;
    }
  }
  if (lo > hi) return;
  // sweep 2: the rows, exactly the sequential scan's step from the segment's entry
  uint32_t* chp = c_hi + row0 + (long long)hi * ld2;
  uint32_t* clp = c_lo + row0 + (long long)hi * ld2;
  uint32_t* whp = CARRY ? w_hi + row0 + (long long)hi * ld2 : nullptr;
  uint32_t* wlp = CARRY ? w_lo + row0 + (long long)hi * ld2 : nullptr;
  float an0 = an0_in, an1 = an1_in;
  float2 up = up0;
  float2 nxt[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) nxt[u] = (hi - u >= lo) ? ldpsi(hi - u) : make_float2(0.f, 0.f);
  for (int r8 = hi; r8 >= lo; r8 -= 8) {
    float2 blk[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) blk[u] = nxt[u];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      nxt[u] = (r8 - 8 - u >= lo) ? ldpsi(r8 - 8 - u) : make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
    const int r = r8 - u;
    if (r < lo) break;
    const float2 cur = blk[u];
    const float c_prev = cs[r], c_r = (r < L) ? cs[r + 1] : 0.f;
    float c0 = r >= 1 ? c_prev * ws0 * cur.x : 0.f;
    float c1 = r >= 1 ? c_prev * ws1 * cur.y : 0.f;
    float w0 = 0.f, w1 = 0.f;
    if (ALIF && r < L) {
      const float A0 = fmaf(-beta, cur.x, rho), A1 = fmaf(-beta, cur.y, rho);
      lam0 = fmaf(an0, lam0, -beta * (c_r * ws0 * up.x));
      lam1 = fmaf(an1, lam1, -beta * (c_r * ws1 * up.y));
      c0 = fmaf(cur.x, lam0, c0);
      c1 = fmaf(cur.y, lam1, c1);
      w0 = cur.x * dcum0;
      w1 = cur.y * dcum1;
      dcum0 *= A0;
      dcum1 *= A1;
      an0 = A0;
      an1 = A1;
    }
    if (FILT) {
      ft0 = fmaf(falpha, ft0, c0);
      ft1 = fmaf(falpha, ft1, c1);
      c0 = ft0;
      c1 = ft1;
    }
    if (live) {
      uint32_t h, l;
      split_bf16x2(c0, c1, h, l);
      *chp = h;
      *clp = l;
      if (CARRY) {
        split_bf16x2(w0, w1, h, l);
        *whp = h;
        *wlp = l;
      }
    }
    chp -= ld2;
    clp -= ld2;
    if (CARRY) { whp -= ld2; wlp -= ld2; }
    up = cur;
    }
  }
  if (ALIF && mdt != nullptr && seg == 0 && live) {  // M = A_0 Lambda_0, Dt = prod A
    mdt[bi] = make_float2(an0 * lam0, dcum0);
    if (has2) mdt[bi + 1] = make_float2(an1 * lam1, dcum1);
  }
}

// ------------------------------------------------------------------------------------
// K1r: backward scan of one chunk with reset=True (neurons.py:266-271: the soft reset makes
// G_u per-synapse, h_uu = alpha - theta psi^-, and couples it to G_a, h_ua = theta beta
// psi^-).  The trace g = (G_u, G_a) of one synapse obeys g_r = A_r g_{r-1} + e_u x_r with
//   A_r = [[alpha - theta P_r, theta beta P_r], [P_r, rho - beta P_r]],  P_r = psi_{r-1}
// (LIF: beta = rho = 0, only G_u lives), and step r adds q_r . g_r to the gradient with
// q_r = Lpsi_r (1, -beta).  Backwards over the chunk:
//   lambda_r = q_r + A_{r+1}^T lambda_{r+1}           -> C_{r+1} = lambda_r,u  (GEMM row of x_r)
//   Phi_r    = A_{L-1} ... A_{r+1}                     -> W_{r+1} = Phi_r e_u   (carry rows)
//   M = A_0^T lambda_0,  Dt = Phi_{-1}                  (boundary term M.E0, E_end = Dt E0 + D)
// Row 0 (no x) is zero; the GEMM operand is the raw input (K4 with alpha = 0).  Outputs:
// c (bf16 hi/lo), w_u = (w_hi, w_lo), ALIF also w_a = (wa_hi, wa_lo); coefficients: LIF
// float2 (M_u, Dt_uu) in mdt, ALIF float[8] (M_u, M_a, Dt_uu, Dt_ua, Dt_au, Dt_aa, 0, 0).
// ------------------------------------------------------------------------------------
struct ResetLane {
  float lu = 0.f, la = 0.f;                          // lambda_{r+1}
  float nuu = 0.f, nua = 0.f, nau = 0.f, naa = 0.f;  // A_{r+1}
  float puu = 1.f, pua = 0.f, pau = 0.f, paa = 1.f;  // Phi_r
  __device__ __forceinline__ void step(float P, float lpsi, float alpha, float theta, float beta,
                                       float rho, bool alif, float& cval, float& wu, float& wa) {
    const float auu = fmaf(-theta, P, alpha);
    const float aua = alif ? theta * beta * P : 0.f;
    const float aau = alif ? P : 0.f;
    const float aaa = alif ? fmaf(-beta, P, rho) : 0.f;
    const float qa = alif ? -beta * lpsi : 0.f;
    const float nlu = fmaf(nau, la, fmaf(nuu, lu, lpsi));
    const float nla = fmaf(naa, la, fmaf(nua, lu, qa));
    lu = nlu;
    la = nla;
    cval = lu;
    wu = puu;
    wa = pau;
    const float quu = fmaf(pua, aau, puu * auu), qua = fmaf(pua, aaa, puu * aua);
    const float qau = fmaf(paa, aau, pau * auu), qaa = fmaf(paa, aaa, pau * aua);
    puu = quu; pua = qua; pau = qau; paa = qaa;
    nuu = auu; nua = aua; nau = aau; naa = aaa;
  }
};

__global__ void __launch_bounds__(K1S_THREADS) reset_scan_kernel(
    FwdParams P, const float* __restrict__ wsig, const float* __restrict__ ctab,
    uint32_t* __restrict__ c_hi, uint32_t* __restrict__ c_lo, uint32_t* __restrict__ w_hi,
    uint32_t* __restrict__ w_lo, uint32_t* __restrict__ wa_hi, uint32_t* __restrict__ wa_lo,
    int ldc, float* __restrict__ coef, const float* __restrict__ psis) {
  extern __shared__ float cs[];  // cs[r] = c_{t0+r}, r = 0..L-1
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = P.len;
  for (int r = threadIdx.x; r < L; r += K1S_THREADS) cs[r] = ctab[P.t0 + r];
  __syncthreads();
  const int i = blockIdx.x * 2 * K1S_THREADS + warp * 64 + 2 * lane;
  const int b = blockIdx.y;
  if (b >= P.B || i >= P.n) return;
  const bool has2 = i + 1 < P.n;
  const bool alif = P.alif != 0;
  const long long bi = (long long)b * P.n + i;
  const float ws0 = wsig[bi], ws1 = has2 ? wsig[bi + 1] : 0.f;
  const float alpha = (float)P.alpha, theta = (float)P.theta, beta = (float)P.beta,
              rho = (float)P.rho;
  const bool carry = w_hi != nullptr;
  const float* prow = psis + (long long)b * (P.KR + 1) * P.n + i;
  const bool even_n = (P.n & 1) == 0;  // float2 rows are 8-byte aligned only for even n
  auto ldpsi = [&](int r) -> float2 {
    if (r < 0) return make_float2(0.f, 0.f);
    const float* q = prow + (long long)r * P.n;
    if (has2 && even_n) return *reinterpret_cast<const float2*>(q);
    return make_float2(q[0], has2 ? q[1] : 0.f);
  };
  const long long ld2 = ldc >> 1;
  const long long base = (long long)b * P.KR * ld2 + (i >> 1);
  uint32_t* chp = c_hi + base;
  uint32_t* clp = c_lo + base;
  for (int r = P.KR - 1; r > L; --r) {
    chp[r * ld2] = 0u;
    clp[r * ld2] = 0u;
    if (carry) {
      w_hi[base + r * ld2] = 0u;
      w_lo[base + r * ld2] = 0u;
      if (alif) { wa_hi[base + r * ld2] = 0u; wa_lo[base + r * ld2] = 0u; }
    }
  }
  chp[0] = 0u;  // row 0 carries no input
  clp[0] = 0u;
  if (carry) {
    w_hi[base] = 0u;
    w_lo[base] = 0u;
    if (alif) { wa_hi[base] = 0u; wa_lo[base] = 0u; }
  }
  ResetLane s0, s1;
  // step r uses P_r = psi row r and Lpsi_r = c_r w_sig psi row r+1
  float2 up = ldpsi(L);
  // rows in blocks of 8, the next block's loads in flight (as chunk_scan_kernel)
  float2 nxt[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) nxt[u] = ldpsi(L - 1 - u);
  for (int r8 = L - 1; r8 >= 0; r8 -= 8) {
    float2 blk[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) blk[u] = nxt[u];
#pragma unroll
    for (int u = 0; u < 8; ++u) nxt[u] = ldpsi(r8 - 8 - u);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
    const int r = r8 - u;
    if (r < 0) break;
    const float2 cur = blk[u];
    const float cr = cs[r];
    float c0, u0, a0, c1, u1, a1;
    s0.step(cur.x, cr * ws0 * up.x, alpha, theta, beta, rho, alif, c0, u0, a0);
    s1.step(cur.y, cr * ws1 * up.y, alpha, theta, beta, rho, alif, c1, u1, a1);
    const long long o = (long long)(r + 1) * ld2;
    uint32_t h, l;
    split_bf16x2(c0, c1, h, l);
    chp[o] = h;
    clp[o] = l;
    if (carry) {
      split_bf16x2(u0, u1, h, l);
      w_hi[base + o] = h;
      w_lo[base + o] = l;
      if (alif) {
        split_bf16x2(a0, a1, h, l);
        wa_hi[base + o] = h;
        wa_lo[base + o] = l;
      }
    }
    up = cur;
    }
  }
  if (coef != nullptr) {
    const ResetLane* sl[2] = {&s0, &s1};
    for (int h = 0; h < (has2 ? 2 : 1); ++h) {
      const ResetLane& s = *sl[h];
      const float mu = fmaf(s.nau, s.la, s.nuu * s.lu);
      const float ma = fmaf(s.naa, s.la, s.nua * s.lu);
      if (alif) {
        float4* cp = reinterpret_cast<float4*>(coef + (bi + h) * 8);
        cp[0] = make_float4(mu, ma, s.puu, s.pua);
        cp[1] = make_float4(s.pau, s.paa, 0.f, 0.f);
      } else {
        reinterpret_cast<float2*>(coef)[bi + h] = make_float2(mu, s.puu);
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// K4: xbar chunk.  Thread per (sample, 2 neighbouring channels); fp64 recurrences; the
// input bytes of 8 steps are loaded ahead of the dependent chain.  Writes the bf16 hi/lo
// split MN-major (channels contiguous): xh/xl [B*KR][kp], row b*KR + rho, rho = 0 ->
// xbar_{t0-1} (carry), rho = s+1 -> xbar_{t0+s}, zero beyond the chunk -- one 128-byte
// coalesced bf16x2 store per warp and row.
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) xbar_chunk_kernel(
    const uint8_t* __restrict__ x, long long stride_b, long long stride_t, int B, int k, int kp,
    int KR, int len, int fresh, double alpha, double* __restrict__ xbar_st,
    uint32_t* __restrict__ xh, uint32_t* __restrict__ xl) {
  const int jp = blockIdx.x * blockDim.x + threadIdx.x;  // channel pair
  const int j = 2 * jp;
  const int b = blockIdx.y;
  if (j >= kp) return;
  const bool v0 = j < k, v1 = j + 1 < k;
  double xb0 = (v0 && !fresh) ? xbar_st[(long long)b * k + j] : 0.0;
  double xb1 = (v1 && !fresh) ? xbar_st[(long long)b * k + j + 1] : 0.0;
  const uint8_t* xin = x + (long long)b * stride_b + j;
  const long long ld2 = kp >> 1;
  uint32_t* oh = xh + (long long)b * KR * ld2 + jp;
  uint32_t* ol = xl != nullptr ? xl + (long long)b * KR * ld2 + jp : nullptr;
  for (int r8 = 0; r8 < KR; r8 += 8) {
    uint32_t x0[8], x1[8];
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) {
      const int rho = r8 + u8;
      const bool live = rho >= 1 && rho <= len;
      x0[u8] = (v0 && live) ? xin[(long long)(rho - 1) * stride_t] : 0u;
      x1[u8] = (v1 && live) ? xin[(long long)(rho - 1) * stride_t + 1] : 0u;
    }
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) {
      const int rho = r8 + u8;
      float f0 = 0.f, f1 = 0.f;
      if (rho == 0) {
        f0 = (float)xb0;
        f1 = (float)xb1;
      } else if (rho <= len) {
        xb0 = __dadd_rn(__dmul_rn(alpha, xb0), (double)x0[u8]);
        xb1 = __dadd_rn(__dmul_rn(alpha, xb1), (double)x1[u8]);
        f0 = (float)xb0;
        f1 = (float)xb1;
      }
      uint32_t h, l;
      split_bf16x2(f0, f1, h, l);
      oh[(long long)rho * ld2] = h;
      if (xl != nullptr) ol[(long long)rho * ld2] = l;
    }
  }
  if (v0) xbar_st[(long long)b * k + j] = xb0;
  if (v1) xbar_st[(long long)b * k + j + 1] = xb1;
}

// K4 on 4 neighbouring channels per thread (row strides and x 4-byte aligned): one 32-bit
// spike load and two 8-byte bf16x4 stores per step -- half the instructions per byte of
// the 2-channel kernel above, same values.
// raw != 0 (multi-chunk raw-spike operand): rows rho >= 1 hold the raw spikes, row 0 is
// zero and the entry state xbar_{t0-1} goes to xs_hi/xs_lo [B][kp] instead (the GEMMs
// add its term separately); the fp64 filter state is still advanced with alpha.
__global__ void __launch_bounds__(128) xbar_chunk4_kernel(
    const uint8_t* __restrict__ x, long long stride_b, long long stride_t, int B, int k, int kp,
    int KR, int len, int fresh, double alpha, double* __restrict__ xbar_st,
    uint2* __restrict__ xh, uint2* __restrict__ xl, int raw = 0,
    uint2* __restrict__ xs_hi = nullptr, uint2* __restrict__ xs_lo = nullptr) {
  const int jq = blockIdx.x * blockDim.x + threadIdx.x;  // channel quad
  const int j = 4 * jq;
  const int b = blockIdx.y;
  if (j >= kp) return;
  double xb[4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
    xb[c] = (j + c < k && !fresh) ? xbar_st[(long long)b * k + j + c] : 0.0;
  // channels >= k read padding bytes of the operand row (zero) or nothing at all
  const bool any = j < k;
  const uint32_t* xin = reinterpret_cast<const uint32_t*>(x + (long long)b * stride_b + j);
  const long long st4 = stride_t >> 2;
  const long long ld4 = kp >> 2;
  uint2* oh = xh + (long long)b * KR * ld4 + jq;
  uint2* ol = xl != nullptr ? xl + (long long)b * KR * ld4 + jq : nullptr;
  const uint32_t keep = j + 4 <= k ? 0xffffffffu : (0xffffffffu >> (8 * (j + 4 - k)));
  for (int r8 = 0; r8 < KR; r8 += 8) {
    uint32_t xw[8];
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) {
      const int rho = r8 + u8;
      const bool live = any && rho >= 1 && rho <= len;
      xw[u8] = live ? (__ldg(xin + (long long)(rho - 1) * st4) & keep) : 0u;
    }
#pragma unroll
    for (int u8 = 0; u8 < 8; ++u8) {
      const int rho = r8 + u8;
      float f[4] = {0.f, 0.f, 0.f, 0.f};
      if (rho == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) f[c] = (float)xb[c];
        if (raw) {  // entry state to xs, zero row
          uint2 h, l;
          split_bf16x2(f[0], f[1], h.x, l.x);
          split_bf16x2(f[2], f[3], h.y, l.y);
          xs_hi[(long long)b * ld4 + jq] = h;
          xs_lo[(long long)b * ld4 + jq] = l;
#pragma unroll
          for (int c = 0; c < 4; ++c) f[c] = 0.f;
        }
      } else if (rho <= len) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t xv = (xw[u8] >> (8 * c)) & 0xffu;
          xb[c] = __dadd_rn(__dmul_rn(alpha, xb[c]), (double)xv);
          f[c] = raw ? (float)xv : (float)xb[c];
        }
      }
      uint2 h, l;
      split_bf16x2(f[0], f[1], h.x, l.x);
      split_bf16x2(f[2], f[3], h.y, l.y);
      oh[(long long)rho * ld4] = h;
      if (xl != nullptr) ol[(long long)rho * ld4] = l;
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (j + c < k) xbar_st[(long long)b * k + j + c] = xb[c];
}

// K4 on time segments: warp s of a CTA filters rows rho in [S s, S s + S - 1] of 128
// channels (4 per lane), S = KR / nseg rows per segment (64 up to KR = 512, then the
// KR / 8 of 8 segments) -- nseg x the threads of xbar_chunk4_kernel for the same bytes.  The filter is linear: sweep 1 runs each segment from a
// zero entry (segment 0 from the true carry) to get its end value, the segments meet in
// shared memory in time order (E <- alpha^len E + end), and sweep 2 re-reads the spike
// bytes (L1/L2-hot) and writes the rows from the true entry.  fp64 throughout; the values
// equal the sequential filter's up to fp64 rounding (they are then split to bf16 hi/lo).
constexpr int XSEG_ROWS = 64;

__global__ void __launch_bounds__(256) xbar_seg_kernel(
    const uint8_t* __restrict__ x, long long stride_b, long long stride_t, int B, int k, int kp,
    int KR, int len, int fresh, double alpha, double* __restrict__ xbar_st,
    uint2* __restrict__ xh, uint2* __restrict__ xl, int raw = 0,
    uint2* __restrict__ xs_hi = nullptr, uint2* __restrict__ xs_lo = nullptr) {
  __shared__ double sh_end[8][32][4];
  __shared__ double sh_pow[8];
  const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
  const int nseg = blockDim.x >> 5;
  const int jq = blockIdx.x * 32 + lane;  // channel quad
  const int j = 4 * jq;
  const int b = blockIdx.y;
  const bool any = j < k;
  const uint32_t keep = j + 4 <= k ? 0xffffffffu : (any ? (0xffffffffu >> (8 * (j + 4 - k))) : 0u);
  const uint32_t* xin = reinterpret_cast<const uint32_t*>(x + (long long)b * stride_b + (any ? j : 0));
  const long long st4 = stride_t >> 2;
  double xb_in[4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
    xb_in[c] = (j + c < k && !fresh) ? xbar_st[(long long)b * k + j + c] : 0.0;
  const int srows = KR / nseg;
  const int lo = seg * srows, hi = lo + srows - 1;
  auto xword = [&](int rho) -> uint32_t {  // spikes of step rho - 1 (rows 1..len)
    return (any && rho >= 1 && rho <= len) ? (__ldg(xin + (long long)(rho - 1) * st4) & keep) : 0u;
  };
  // ---- sweep 1: end value of this segment from a zero entry (segment 0: the carry) ----
  if (seg + 1 < nseg) {
    double y[4];
    double apow = 1.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) y[c] = (seg == 0) ? xb_in[c] : 0.0;
    for (int r8 = lo; r8 <= hi; r8 += 8) {
      uint32_t w8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) w8[u] = xword(r8 + u);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int rho = r8 + u;
        if (rho >= 1 && rho <= len) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            y[c] = __dadd_rn(__dmul_rn(alpha, y[c]), (double)((w8[u] >> (8 * c)) & 0xffu));
          apow = __dmul_rn(apow, alpha);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) sh_end[seg][lane][c] = y[c];
    if (lane == 0) sh_pow[seg] = apow;
  }
  __syncthreads();
  // ---- entry of this segment: the segments before it, in time order ----
  double xv[4];
  if (seg == 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) xv[c] = xb_in[c];
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) xv[c] = 0.0;
    for (int q = 0; q < seg; ++q) {
      const double ap = sh_pow[q];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        xv[c] = (q == 0) ? sh_end[0][lane][c] : __dadd_rn(__dmul_rn(ap, xv[c]), sh_end[q][lane][c]);
    }
  }
  if (jq >= (kp >> 2)) return;
  // ---- sweep 2: the rows ----
  const long long ld4 = kp >> 2;
  uint2* oh = xh + ((long long)b * KR + lo) * ld4 + jq;
  uint2* ol = xl != nullptr ? xl + ((long long)b * KR + lo) * ld4 + jq : nullptr;
  for (int r8 = lo; r8 <= hi; r8 += 8) {
    uint32_t w8[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) w8[u] = xword(r8 + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int rho = r8 + u;
      float f[4] = {0.f, 0.f, 0.f, 0.f};
      if (rho == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) f[c] = (float)xv[c];
        if (raw) {  // entry state to xs, zero row (see xbar_chunk4_kernel)
          uint2 h, l;
          split_bf16x2(f[0], f[1], h.x, l.x);
          split_bf16x2(f[2], f[3], h.y, l.y);
          xs_hi[(long long)b * ld4 + jq] = h;
          xs_lo[(long long)b * ld4 + jq] = l;
#pragma unroll
          for (int c = 0; c < 4; ++c) f[c] = 0.f;
        }
      } else if (rho <= len) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t xb8 = (w8[u] >> (8 * c)) & 0xffu;
          xv[c] = __dadd_rn(__dmul_rn(alpha, xv[c]), (double)xb8);
          f[c] = raw ? (float)xb8 : (float)xv[c];
        }
      }
      uint2 h, l;
      split_bf16x2(f[0], f[1], h.x, l.x);
      split_bf16x2(f[2], f[3], h.y, l.y);
      oh[(long long)(rho - lo) * ld4] = h;
      if (xl != nullptr) ol[(long long)(rho - lo) * ld4] = l;
    }
    // the carried state xbar_{t0+len-1} lives in row len: its segment stores it
    if (r8 <= len && len < r8 + 8) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (j + c < k) xbar_st[(long long)b * k + j + c] = xv[c];
    }
  }
}

}  // namespace spb

using namespace spb;

// segmented scan selection (SPB_SCAN_SEG=0 restores the one-sweep scan, for A/B runs)
static bool seg_scan() {
  const char* e = getenv("SPB_SCAN_SEG");
  return !(e && e[0] == '0');
}

extern "C" {

int spb_forward_chunk(int pass, const double* cur, int B, int n, int Tc, int KR, int len, int t0,
                      int T, double alpha, double theta, double slope, double beta, double rho,
                      double kappa, int reset, int alif, int smooth, double* u, double* a,
                      double* zbar, double* zsum, uint32_t* raster, const float* wsig,
                      const float* ctab, void* c_hi, void* c_lo, void* w_hi, void* w_lo,
                      void* wa_hi, void* wa_lo, int ldc, float* mdt, float* psi_scratch,
                      cudaStream_t stream) {
  SPB_CHECK_ARG(pass >= 0 && pass <= 4,
                "spb_forward_chunk: pass must be 0 (A), 1 (B), 2 (B scan only), 3 (B scan only, "
                "input filter folded into C / W) or 4 (B, input filter folded)");
  SPB_CHECK_ARG(pass < 3 || !reset, "spb_forward_chunk: passes 3 / 4 need reset = 0");
  const bool filt = pass >= 3;
  if (pass == 3) pass = 2;
  if (pass == 4) pass = 1;
  SPB_CHECK_ARG(pass == 2 || (cur && u && a), "spb_forward_chunk: null pointer");
  SPB_CHECK_ARG(B > 0 && n > 0 && Tc > 0 && len >= 0 && len <= Tc && KR >= Tc + 1 && KR % 8 == 0,
                "spb_forward_chunk: bad sizes B=%d n=%d Tc=%d KR=%d len=%d", B, n, Tc, KR, len);
  SPB_CHECK_ARG(pass == 0 ? (zbar && zsum) : (wsig && ctab && c_hi && c_lo && psi_scratch),
                "spb_forward_chunk: missing pass-%c buffers", pass ? 'B' : 'A');
  SPB_CHECK_ARG(!(pass == 0 && psi_scratch && (u == nullptr)), "spb_forward_chunk: bad pass A");
  SPB_CHECK_ARG(!(pass >= 1 && alif && !reset && (!mdt || (w_hi && !w_lo))),
                "spb_forward_chunk: ALIF pass B needs mdt (and w_lo with w_hi)");
  SPB_CHECK_ARG(pass == 0 || (ldc >= n && ldc % 8 == 0), "spb_forward_chunk: ldc must be >= n, %% 8");
  SPB_CHECK_ARG(!(pass >= 1 && reset && alif && w_hi && !(wa_hi && wa_lo)),
                "spb_forward_chunk: ALIF reset carry needs wa_hi/wa_lo");
  SPB_CHECK_ARG(!(pass >= 1 && reset && !mdt && w_hi),
                "spb_forward_chunk: reset carry needs the coefficient buffer (mdt)");
  FwdParams P{B, n, Tc, KR, len, t0, T, alpha, theta, slope, beta, rho, kappa, reset, alif, pass,
              smooth};
  dim3 grid(ceil_div(n, K1_THREADS), B);
  if (pass <= 1) {
    if (pass == 0 && psi_scratch)
      launch_forward<true, true>(P, grid, stream, cur, u, a, zbar, zsum, raster, wsig, psi_scratch);
    else if (pass == 0)
      launch_forward<true, false>(P, grid, stream, cur, u, a, zbar, zsum, raster, wsig, nullptr);
    else
      launch_forward<false, true>(P, grid, stream, cur, u, a, zbar, zsum, raster, wsig, psi_scratch);
    SPB_CHECK_LAUNCH("forward_chunk");
  }
  if (pass >= 1 && reset) {
    dim3 sgrid(ceil_div(n, 2 * K1S_THREADS), B);
    reset_scan_kernel<<<sgrid, K1S_THREADS, (len > 0 ? len : 1) * sizeof(float), stream>>>(
        P, wsig, ctab, reinterpret_cast<uint32_t*>(c_hi), reinterpret_cast<uint32_t*>(c_lo),
        reinterpret_cast<uint32_t*>(w_hi), reinterpret_cast<uint32_t*>(w_lo),
        reinterpret_cast<uint32_t*>(wa_hi), reinterpret_cast<uint32_t*>(wa_lo), ldc, mdt,
        psi_scratch);
    SPB_CHECK_LAUNCH("reset_scan");
  } else if (pass >= 1) {
    dim3 sgrid(ceil_div(n, 2 * K1S_THREADS), B);
    const bool carry = alif && w_hi != nullptr;
    auto kfn = alif ? (carry ? (filt ? chunk_scan_kernel<true, true, true>
                                     : chunk_scan_kernel<true, true>)
                             : (filt ? chunk_scan_kernel<true, false, true>
                                     : chunk_scan_kernel<true, false>))
                    : (filt ? chunk_scan_kernel<false, false, true>
                            : chunk_scan_kernel<false, false>);
    // segments pay off where the one-sweep grid is small (C2: 0.058 -> 0.031 ms); for
    // ALIF they cost a second psi sweep, a loss once the grid fills the GPU (C3)
    if (seg_scan() && (!alif || (!filt && (long long)B * ceil_div(n, 2 * K1S_THREADS) < 2LL * 148))) {
      auto sfn = alif ? (carry ? chunk_scan_seg_kernel<true, true>
                               : chunk_scan_seg_kernel<true, false>)
                      : (filt ? chunk_scan_seg_kernel<false, false, true>
                              : chunk_scan_seg_kernel<false, false>);
      dim3 g2(ceil_div(n, 64), B);
      sfn<<<g2, SEG * 32, (len + 1) * sizeof(float), stream>>>(
          P, wsig, ctab, reinterpret_cast<uint32_t*>(c_hi), reinterpret_cast<uint32_t*>(c_lo),
          reinterpret_cast<uint32_t*>(w_hi), reinterpret_cast<uint32_t*>(w_lo), ldc,
          reinterpret_cast<float2*>(mdt), psi_scratch);
      SPB_CHECK_LAUNCH("chunk_scan_seg");
      return 0;
    }
    pdl_launch(kfn, sgrid, K1S_THREADS, (len + 1) * sizeof(float), stream,
        P, wsig, ctab, reinterpret_cast<uint32_t*>(c_hi), reinterpret_cast<uint32_t*>(c_lo),
        reinterpret_cast<uint32_t*>(w_hi), reinterpret_cast<uint32_t*>(w_lo), ldc,
        reinterpret_cast<float2*>(mdt), psi_scratch);
    SPB_CHECK_LAUNCH("chunk_scan");
  }
  return 0;
}

static int xbar_launch(const uint8_t* x, long long stride_b, long long stride_t, int B, int k,
                       int kp, int KR, int len, int fresh, double alpha, double* xbar_state,
                       void* xh, void* xl, bool segmented, cudaStream_t stream,
                       void* xs_hi = nullptr, void* xs_lo = nullptr);

int spb_xbar_chunk(const uint8_t* x, long long stride_b, long long stride_t, int B, int k, int kp,
                   int KR, int len, int fresh, double alpha, double* xbar_state, void* xh,
                   void* xl, cudaStream_t stream) {
  return xbar_launch(x, stride_b, stride_t, B, k, kp, KR, len, fresh, alpha, xbar_state, xh, xl,
                     false, stream);
}

// K4 on 64-row time segments (more threads, for a K4 on the critical path; the one-chunk
// K4 overlapped with K1 keeps the sequential kernel, measured better there).
// SPB_XBAR_SEG=0 falls back to the sequential kernel (A/B runs, tests).
int spb_xbar_chunk_seg(const uint8_t* x, long long stride_b, long long stride_t, int B, int k,
                       int kp, int KR, int len, int fresh, double alpha, double* xbar_state,
                       void* xh, void* xl, cudaStream_t stream) {
  const char* es = getenv("SPB_XBAR_SEG");
  return xbar_launch(x, stride_b, stride_t, B, k, kp, KR, len, fresh, alpha, xbar_state, xh, xl,
                     !(es && es[0] == '0'), stream);
}

// Multi-chunk raw-spike operand (xh rows rho >= 1 = raw spikes, row 0 = 0, hi only) with
// the fp64 filter state advanced by alpha and the entry state xbar_{t0-1} written to
// xs_hi / xs_lo [B][kp] (bf16 hi/lo) for the GEMMs' row-0 terms.
int spb_xbar_chunk_raw(const uint8_t* x, long long stride_b, long long stride_t, int B, int k,
                       int kp, int KR, int len, int fresh, double alpha, double* xbar_state,
                       void* xh, void* xs_hi, void* xs_lo, cudaStream_t stream) {
  SPB_CHECK_ARG(xs_hi && xs_lo, "spb_xbar_chunk_raw: null entry-state buffer");
  SPB_CHECK_ARG((stride_b | stride_t) % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 4 == 0,
                "spb_xbar_chunk_raw: the spike rows must be 4-byte aligned");
  const char* es = getenv("SPB_XBAR_SEG");
  return xbar_launch(x, stride_b, stride_t, B, k, kp, KR, len, fresh, alpha, xbar_state, xh,
                     nullptr, !(es && es[0] == '0'), stream, xs_hi, xs_lo);
}

}  // extern "C"

static int xbar_launch(const uint8_t* x, long long stride_b, long long stride_t, int B, int k,
                       int kp, int KR, int len, int fresh, double alpha, double* xbar_state,
                       void* xh, void* xl, bool segmented, cudaStream_t stream, void* xs_hi,
                       void* xs_lo) {
  const int raw = xs_hi != nullptr ? 1 : 0;
  // xl = NULL: only the hi part is written (alpha = 0 raw-spike operand: lo is 0)
  SPB_CHECK_ARG(x && xbar_state && xh && (xl || alpha == 0.0 || raw),
                "spb_xbar_chunk: null pointer");
  SPB_CHECK_ARG(B > 0 && k > 0 && kp >= k && kp % 8 == 0 && KR > 0 && KR % 8 == 0 && len >= 0 &&
                    len < KR,
                "spb_xbar_chunk: bad sizes");
  const bool al4 = (stride_b | stride_t) % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(xh) % 8 == 0 &&
                   reinterpret_cast<uintptr_t>(xl) % 8 == 0;
  const int nseg = std::min(8, KR / XSEG_ROWS);
  if (segmented && al4 && KR % XSEG_ROWS == 0 && (KR / nseg) % 8 == 0) {
    dim3 gs(ceil_div(kp / 4, 32), B);
    xbar_seg_kernel<<<gs, 32 * nseg, 0, stream>>>(
        x, stride_b, stride_t, B, k, kp, KR, len, fresh, alpha, xbar_state,
        reinterpret_cast<uint2*>(xh), reinterpret_cast<uint2*>(xl), raw,
        reinterpret_cast<uint2*>(xs_hi), reinterpret_cast<uint2*>(xs_lo));
    SPB_CHECK_LAUNCH("xbar_seg");
    return 0;
  }
  if (al4) {
    dim3 grid4(ceil_div(kp / 4, 128), B);
    xbar_chunk4_kernel<<<grid4, 128, 0, stream>>>(x, stride_b, stride_t, B, k, kp, KR, len, fresh,
                                                  alpha, xbar_state, reinterpret_cast<uint2*>(xh),
                                                  reinterpret_cast<uint2*>(xl), raw,
                                                  reinterpret_cast<uint2*>(xs_hi),
                                                  reinterpret_cast<uint2*>(xs_lo));
    SPB_CHECK_LAUNCH("xbar_chunk4");
    return 0;
  }
  SPB_CHECK_ARG(!raw, "spb_xbar_chunk_raw: unaligned operand");
  dim3 grid(ceil_div(kp / 2, 128), B);
  xbar_chunk_kernel<<<grid, 128, 0, stream>>>(x, stride_b, stride_t, B, k, kp, KR, len, fresh,
                                              alpha, xbar_state,
                                              reinterpret_cast<uint32_t*>(xh),
                                              reinterpret_cast<uint32_t*>(xl));
  SPB_CHECK_LAUNCH("xbar_chunk");
  return 0;
}


