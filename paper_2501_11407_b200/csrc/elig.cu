// Eligibility-trace kernels of the ALIF adaptation trace eps_a (sm_100a):
//   K6  spb_alif_carry_chunk -- per-synapse trace carried across time chunks on tcgen05
//                               tensor cores, with the inter-chunk gradient term fused
//   --  spb_reduce_partials  -- fixed-order split reduction into the fp64 gradient
//   K5s spb_grad_gemm_simt   -- CUDA-core reference of the factorised GEMM (tests only)
//
// Reference: the ALIF block of eprop_trace_update (gradients.py:89-94, H_I block
// [[alpha,0],[psi^-, rho - beta psi^-]] from neurons.py:266-273 / test_neurons.py:144-155)
// and the eligibility filter x_step = psi (G_u - beta G_a) (gradients.py:165-172).
//
// The trace eps[b][i][j] (= G_a) is the only per-synapse state.  With the chunk
// coefficients of K1 (forward.cu: W_r, M, Dt) a whole chunk of L steps is
//     E_end[b,i,:] = Dt[b,i] E0[b,i,:] + sum_r W_r[b,i] xbar_{r-1}[b,:]     (per-sample GEMM, K = L)
//     grad[i,:]   += sum_b M[b,i] E0[b,i,:]                               (inter-chunk term)
// while every intra-chunk contribution goes through the factorised GEMM K5.  eps is read
// once and written once per chunk (8 bytes per synapse per chunk), and the per-step FMA
// work of the literal recursion moves onto the tensor cores.
//
// Kernel structure: see K6 below (CTA pairs, streamed eps boxes).  The single-CTA
// 128 x 128 version of round 1 (0.56 of HBM at C5, L2-operand bound) was replaced.
#include "tma.cuh"

#include <cstdlib>

namespace spb {

// ------------------------------------------------------------------------------------
// K6: the carry on CTA PAIRS (tcgen05.mma.cta_group::2, M = 256, N = 256).
//
// Why pairs: per (sample, 128 x 128 tile) a single-CTA kernel streams 384 KB of W hi/lo
// and spike operands from L2 for 128 KB of eps traffic, so at C5 its launch was bound by
// the L2 (LTS) throughput, not by HBM (round 1, ncu: DRAM 45 %, long-scoreboard stalls).
// A pair covers 256 neurons x 256 inputs: each CTA stages its own 128 W rows (A) and HALF
// of the 256 input columns (B), and receives its 128 rows x all 256 columns in its own
// TMEM, so the operand bytes per eps byte halve.  The eps tile of a CTA (128 x 256 fp32 =
// 128 KB per sample) is streamed through a ring of 8 TMA boxes of 128 rows x 32 columns
// with its own load warp and store warp, so the eps stream runs continuously instead of a
// tile at a time.  Roles: warp 0 operand TMA (both CTAs; bytes land on the leader's
// barrier), warp 1 TMEM allocator (cta_group::2) and, on the leader, the MMA issuer
// (commits multicast to both CTAs), warp 2 eps box loads, warp 3 eps box stores (E_end
// written in place), warps 4-19 epilogue (4 TMEM lane quarters x 4 column groups of 2
// boxes; the gradient tile grad += M E0 stays in registers across the CTA's samples).
// Measured (profiles/r2): C5 shape, Tc = 511: 441 us per launch for 2.18 GB of DRAM
// traffic = 0.75 of HBM (round-1 single-CTA kernel: 598 us, 0.56).
// ------------------------------------------------------------------------------------
namespace carry {

// MN-major SWIZZLE_128B operand: 64-element MN runs (128 B rows, one per K), 8-row K
// groups 1024 B apart (SBO), the second 64-element MN half one box (LBO) further.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

constexpr int BM = 128;                 // neurons per CTA (the pair: 256)
constexpr int BN = 256;                 // inputs per pair tile = MMA N
constexpr int BNH = BN / 2;             // B-operand columns staged by each CTA
constexpr int BK = 32;                  // K rows per operand stage
constexpr int TILE = BM * BK * 2;       // 8 KB: 128 MN x 32 K bf16 (two 64-wide SW128 boxes)
constexpr int EBOX = BM * 32 * 4;       // 16 KB eps box: 128 rows x 32 fp32 (SW128)
constexpr int BOXES = BN / 32;          // eps boxes per (sample, CTA)
constexpr int NBOX = 8;                 // eps ring slots
constexpr int EPI0 = 4;                 // warps 0-3: operand TMA, MMA, eps load, eps store
constexpr int EPI_WARPS = 16;
constexpr int THREADS = (EPI0 + EPI_WARPS) * 32;
template <bool RAW>
struct Cfg {
  static constexpr int NT = RAW ? 3 : 4;          // W hi, W lo, x hi (, x lo)
  static constexpr int SB = NT * TILE;
  static constexpr int NST = RAW ? 4 : 3;
  static constexpr int SMEM = NBOX * EBOX + NST * SB + 1024 + 512;
};
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ void mma2_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&r)[8]) {
  uint32_t* v = reinterpret_cast<uint32_t*>(r);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <bool RAW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    alif_carry_pair_kernel(const __grid_constant__ CUtensorMap tm_wh,
                           const __grid_constant__ CUtensorMap tm_wl,
                           const __grid_constant__ CUtensorMap tm_xh,
                           const __grid_constant__ CUtensorMap tm_xl,
                           const __grid_constant__ CUtensorMap tm_eps,
                           const float2* __restrict__ mdt, float* __restrict__ partial, int B,
                           int n, int n_pad, int kp, int KR, int b_per_split, int do_mma,
                           int load_eps, int store_eps, const __nv_bfloat16* __restrict__ wh_g,
                           const __nv_bfloat16* __restrict__ wl_g, int ldw,
                           const __nv_bfloat16* __restrict__ xs_hi,
                           const __nv_bfloat16* __restrict__ xs_lo) {
  using C = Cfg<RAW>;
  constexpr int NST = C::NST, SB = C::SB;
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* esm = smem;                             // [NBOX][128 rows][128 B]
  uint8_t* osm = smem + NBOX * EBOX;               // [NST][NT][TILE]
  uint64_t* bars = reinterpret_cast<uint64_t*>(osm + NST * SB);
  uint64_t* full = bars;                           // [NST] (the leader's is used)
  uint64_t* empty = full + NST;                    // [NST]
  uint64_t* tfull = empty + NST;                   // [2]
  uint64_t* tempty = tfull + 2;                    // [2] (the leader's is used)
  uint64_t* efull = tempty + 2;                    // [NBOX]
  uint64_t* eempty = efull + NBOX;                 // [NBOX]
  uint64_t* eready = eempty + NBOX;                // [NBOX]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(eready + NBOX);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int j0 = (blockIdx.x >> 1) * BN;           // the pair's first input column
  const int jx = j0 + (int)rank * BNH;             // this CTA's B-operand columns
  const int i0 = blockIdx.y * (2 * BM) + (int)rank * BM;   // this CTA's neurons
  const bool own = i0 < n_pad;                     // rows past n_pad: next sample's rows
  const int b0 = blockIdx.z * b_per_split;
  const int nb = max(0, min(B, b0 + b_per_split) - b0);
  const int nkb = KR / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 2 * EPI_WARPS);   // epilogue warps of BOTH CTAs
    }
    for (int e = 0; e < NBOX; ++e) {
      mbar_init(smem_u32(&efull[e]), 1);
      mbar_init(smem_u32(&eempty[e]), 1);
      mbar_init(smem_u32(&eready[e]), 4);              // the 4 lane-quarter warps of a group
    }
    mbar_fence_init();
    if (do_mma) {
      tma_prefetch_desc(&tm_wh);
      tma_prefetch_desc(&tm_wl);
      tma_prefetch_desc(&tm_xh);
      if (!RAW) tma_prefetch_desc(&tm_xl);
    }
    if (load_eps || store_eps) tma_prefetch_desc(&tm_eps);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive / complete_tx
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  // registers: the producer warpgroup (warps 0-3) gives its share to the epilogue, whose
  // gradient tile (64 fp32 per thread) lives in registers: 128 x 56 + 512 x 104 <= 640 x 96
  if (warp < EPI0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
    if (warp == 0) {
      if (lane == 0 && do_mma) {  // this CTA's operand K-blocks of every sample's GEMM
        int it = 0;
        for (int lb = 0; lb < nb; ++lb) {
          const int kbase = (b0 + lb) * KR;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % NST;
            mbar_wait(smem_u32(&empty[s]), ((it / NST) & 1) ^ 1);
            if (leader) mbar_expect_tx(smem_u32(&full[s]), 2 * SB);
            const uint32_t lb_full = mapa(smem_u32(&full[s]), 0);
            const uint32_t st = smem_u32(osm + s * SB);
            const int kr = kbase + kb * BK;
            tma_load_2sm(st, &tm_wh, lb_full, i0, kr);
            tma_load_2sm(st + TILE / 2, &tm_wh, lb_full, i0 + 64, kr);
            tma_load_2sm(st + TILE, &tm_wl, lb_full, i0, kr);
            tma_load_2sm(st + TILE + TILE / 2, &tm_wl, lb_full, i0 + 64, kr);
            tma_load_2sm(st + 2 * TILE, &tm_xh, lb_full, jx, kr);
            tma_load_2sm(st + 2 * TILE + TILE / 2, &tm_xh, lb_full, jx + 64, kr);
            if (!RAW) {
              tma_load_2sm(st + 3 * TILE, &tm_xl, lb_full, jx, kr);
              tma_load_2sm(st + 3 * TILE + TILE / 2, &tm_xl, lb_full, jx + 64, kr);
            }
          }
        }
      }
    } else if (warp == 1) {
      if (leader && do_mma) {  // whole warp, converged; elect.sync picks the issuer
        int it = 0;
        for (int lb = 0; lb < nb; ++lb) {
          const int a = lb & 1;
          mbar_wait_cluster(smem_u32(&tempty[a]), ((lb >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t d = tmem_base + (uint32_t)(a * BN);
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % NST;
            mbar_wait_cluster(smem_u32(&full[s]), (it / NST) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t st = smem_u32(osm + s * SB);
  #pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t off = kk * 2048;  // 16 K rows of the MN-major tiles
              const uint64_t dwh = desc_mn_sw128(st + off, TILE / 2),
                             dwl = desc_mn_sw128(st + TILE + off, TILE / 2);
              const uint64_t dxh = desc_mn_sw128(st + 2 * TILE + off, TILE / 2),
                             dxl = desc_mn_sw128(st + 3 * TILE + off, TILE / 2);
              mma2_bf16(d, dwh, dxh, (kb | kk) ? 1u : 0u);
              if (!RAW) mma2_bf16(d, dwh, dxl, 1u);
              mma2_bf16(d, dwl, dxh, 1u);
            }
            commit2(smem_u32(&empty[s]));
          }
          commit2(smem_u32(&tfull[a]));
        }
      }
    } else if (warp == 2) {
      if (lane == 0) {  // eps boxes of every sample, in (sample, box) order through the ring
        const bool ld = load_eps && own;
        for (int lb = 0; lb < nb; ++lb) {
          for (int bx = 0; bx < BOXES; ++bx) {
            const int gi = lb * BOXES + bx, slot = gi % NBOX, u = gi / NBOX;
            mbar_wait(smem_u32(&eempty[slot]), (u & 1) ^ 1);
            const uint32_t fb = smem_u32(&efull[slot]);
            if (ld) {
              mbar_expect_tx(fb, EBOX);
              tma_load_2d(smem_u32(esm + slot * EBOX), &tm_eps, fb, j0 + 32 * bx,
                          (b0 + lb) * n_pad + i0);
            } else {
              arrive(fb);
            }
          }
        }
      }
    } else if (warp == 3) {
      if (lane == 0) {  // E_end boxes back to HBM; a slot is freed once its store has read it
        const bool st_e = store_eps && own;
        int prev = -1;
        for (int lb = 0; lb < nb; ++lb) {
          for (int bx = 0; bx < BOXES; ++bx) {
            const int gi = lb * BOXES + bx, slot = gi % NBOX, u = gi / NBOX;
            mbar_wait(smem_u32(&eready[slot]), u & 1);
            if (st_e) {
              tma_store_2d(&tm_eps, smem_u32(esm + slot * EBOX), j0 + 32 * bx,
                           (b0 + lb) * n_pad + i0);
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              if (prev >= 0) arrive(smem_u32(&eempty[prev]));
              prev = slot;
            } else {
              arrive(smem_u32(&eempty[slot]));
            }
          }
        }
        if (st_e) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // E_end written
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 104;" ::: "memory");
    const int e = warp - EPI0;
    const int q = warp & 3;            // TMEM lane quarter of this warp
    const int cg = e >> 2;             // column group: boxes cg and cg + 4
    const int r = q * 32 + lane;       // tile-local neuron row
    const int i = i0 + r;
    const bool vi = i < n;
    const bool lde = load_eps && own;
    const bool entry = RAW && xs_hi != nullptr && store_eps;
    const uint32_t lead_tempty0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t lead_tempty1 = mapa(smem_u32(&tempty[1]), 0);
    float g[2 * 32];
#pragma unroll
    for (int c = 0; c < 64; ++c) g[c] = 0.f;
    for (int lb = 0; lb < nb; ++lb) {
      const int b = b0 + lb;
      const int a = lb & 1;
      const float2 md = vi ? mdt[(long long)b * n + i] : make_float2(0.f, 0.f);
      // RAW: entry-state term Wt_0[b,i] * xbar_{t0-1}[b, c] (xs absent: fresh state)
      float w0e = 0.f;
      if (entry && vi) {
        const long long o = (long long)b * KR * ldw + i;
        w0e = __bfloat162float(wh_g[o]) + __bfloat162float(wl_g[o]);
      }
      if (do_mma) {
        mbar_wait(smem_u32(&tfull[a]), (lb >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int bx = cg + 4 * h;
        const int gi = lb * BOXES + bx, slot = gi % NBOX, u = gi / NBOX;
        const int c0 = j0 + 32 * bx;
        const bool xs_ok = entry && c0 < kp;
        const uint32_t erow = smem_u32(esm + slot * EBOX + r * 128);
        mbar_wait(smem_u32(&efull[slot]), u & 1);
#pragma unroll
        for (int o8 = 0; o8 < 4; ++o8) {   // 8 columns per TMEM load
          float D[8];
          if (do_mma) {
            tmem_ld8(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * BN + bx * 32 + o8 * 8), D);
          } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) D[c] = 0.f;
          }
#pragma unroll
          for (int w2 = 0; w2 < 2; ++w2) {
            const int v4 = o8 * 2 + w2;
            float4 e0 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (lde)  // SWIZZLE_128B: 16-byte chunk v4 of row r sits at chunk v4 ^ (r & 7)
              e0 = lds_f4(erow + ((v4 ^ (r & 7)) << 4));
            float* gg = g + 32 * h + 4 * v4;
            gg[0] = fmaf(md.x, e0.x, gg[0]);
            gg[1] = fmaf(md.x, e0.y, gg[1]);
            gg[2] = fmaf(md.x, e0.z, gg[2]);
            gg[3] = fmaf(md.x, e0.w, gg[3]);
            if (store_eps) {  // E_end in place over E0 (same swizzled chunk)
              float4 en;
              en.x = fmaf(md.y, e0.x, D[4 * w2 + 0]);
              en.y = fmaf(md.y, e0.y, D[4 * w2 + 1]);
              en.z = fmaf(md.y, e0.z, D[4 * w2 + 2]);
              en.w = fmaf(md.y, e0.w, D[4 * w2 + 3]);
              if (xs_ok) {
                const long long xo = (long long)b * kp + c0 + 4 * v4;
                const uint2 hq = *reinterpret_cast<const uint2*>(xs_hi + xo);
                const uint2 lq = *reinterpret_cast<const uint2*>(xs_lo + xo);
                const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hq);
                const __nv_bfloat162* l2 = reinterpret_cast<const __nv_bfloat162*>(&lq);
                const float2 h01 = __bfloat1622float2(h2[0]), h23 = __bfloat1622float2(h2[1]);
                const float2 l01 = __bfloat1622float2(l2[0]), l23 = __bfloat1622float2(l2[1]);
                en.x = fmaf(w0e, h01.x + l01.x, en.x);
                en.y = fmaf(w0e, h01.y + l01.y, en.y);
                en.z = fmaf(w0e, h23.x + l23.x, en.z);
                en.w = fmaf(w0e, h23.y + l23.y, en.w);
              }
              sts_f4(erow + ((v4 ^ (r & 7)) << 4), en);
            }
          }
        }
        if (store_eps) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive(smem_u32(&eready[slot]));
      }
      if (do_mma) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive_remote(a ? lead_tempty1 : lead_tempty0);
      }
    }
    if (own) {
      // grad tile through a 4x4 lane transpose of 32-byte chunks and 256-bit stores: each
      // instruction writes 8 rows x 128 contiguous bytes (rows past n are zero padding)
      const int p4 = lane & 3;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c0 = j0 + 32 * (cg + 4 * h);
        float* gh = g + 32 * h;
#pragma unroll
        for (int sh = 2; sh >= 1; sh >>= 1) {
          const bool up = (p4 & sh) != 0;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            if (m & sh) continue;
            const int ms = m | sh;
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              const float send = up ? gh[8 * m + x] : gh[8 * ms + x];
              const float recv = __shfl_xor_sync(0xffffffffu, send, sh);
              if (up) gh[8 * m + x] = recv; else gh[8 * ms + x] = recv;
            }
          }
        }
        if (c0 < kp) {
          float* base = partial + ((long long)blockIdx.z * n_pad + i0 + q * 32 + (lane & ~3)) * kp +
                        c0 + 8 * p4;
#pragma unroll
          for (int kq = 0; kq < 4; ++kq)
            asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(
                             base + (long long)kq * kp),
                         "f"(gh[8 * kq + 0]), "f"(gh[8 * kq + 1]), "f"(gh[8 * kq + 2]),
                         "f"(gh[8 * kq + 3]), "f"(gh[8 * kq + 4]), "f"(gh[8 * kq + 5]),
                         "f"(gh[8 * kq + 6]), "f"(gh[8 * kq + 7])
                         : "memory");
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the peer is done with the pair's TMEM and barriers
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

}  // namespace carry

// 4 consecutive elements per thread (float4 partial loads, all S slices in flight before
// the fixed-order fp64 sums), k_pad % 4 == 0.
__global__ void reduce_partials_kernel(const float* __restrict__ partial, int S, int n, int n_pad,
                                       int k_pad, int accumulate, double* __restrict__ grad) {
  pdl_enter();
  const long long idx = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (idx >= (long long)n * k_pad) return;
  const long long stride = (long long)n_pad * k_pad;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int s = 0;
  for (; s + 4 <= S; s += 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = __ldcs(reinterpret_cast<const float4*>(partial + (s + u) * stride + idx));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 += (double)v[u].x;
      a1 += (double)v[u].y;
      a2 += (double)v[u].z;
      a3 += (double)v[u].w;
    }
  }
  for (; s < S; ++s) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(partial + s * stride + idx));
    a0 += (double)v.x;
    a1 += (double)v.y;
    a2 += (double)v.z;
    a3 += (double)v.w;
  }
  double2* g2 = reinterpret_cast<double2*>(grad + idx);
  if (accumulate) {
    const double2 o0 = g2[0], o1 = g2[1];
    a0 = o0.x + a0;
    a1 = o0.y + a1;
    a2 = o1.x + a2;
    a3 = o1.y + a3;
  }
  g2[0] = make_double2(a0, a1);
  g2[1] = make_double2(a2, a3);
}

// CUDA-core GEMM on the same bf16 hi/lo operands as the tensor-core path:
// grad[i][j] += sum_K (Ah+Al)[K][i] * (Bh+Bl)[K][j]  (64x64 tiles, 4x4 per thread).
__global__ void __launch_bounds__(256) grad_gemm_simt_kernel(
    const __nv_bfloat16* __restrict__ ah, const __nv_bfloat16* __restrict__ al, int lda,
    const __nv_bfloat16* __restrict__ bh, const __nv_bfloat16* __restrict__ bl, int ldb, int M,
    int N, int K, double* __restrict__ grad, int ldg) {
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
        const long long o = (long long)(k0 + kk) * lda + m0 + r;
        va = __bfloat162float(ah[o]) + __bfloat162float(al[o]);
      }
      if (n0 + r < N && k0 + kk < K) {
        const long long o = (long long)(k0 + kk) * ldb + n0 + r;
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

int spb_reduce_partials(const float* partial, int splits, int n, int n_pad, int k_pad,
                        int accumulate, double* grad, cudaStream_t stream) {
  SPB_CHECK_ARG(partial && grad && splits > 0 && n > 0 && n <= n_pad && k_pad % 4 == 0,
                "spb_reduce_partials: bad args (k_pad %% 4 == 0)");
  const long long total = (long long)n * k_pad;
  pdl_launch(reduce_partials_kernel, (unsigned)((total / 4 + 255) / 256), 256, 0, stream,
      partial, splits, n, n_pad, k_pad, accumulate, grad);
  SPB_CHECK_LAUNCH("reduce_partials");
  return 0;
}

int spb_grad_gemm_simt(const void* ah, const void* al, int lda, const void* bh, const void* bl,
                       int ldb, int M, int N, int K, double* grad, int ldg, cudaStream_t stream) {
  SPB_CHECK_ARG(ah && al && bh && bl && grad && M > 0 && N > 0 && K > 0 && ldg >= N && lda >= M &&
                    ldb >= N,
                "spb_grad_gemm_simt: bad args");
  dim3 grid(ceil_div(N, 64), ceil_div(M, 64));
  grad_gemm_simt_kernel<<<grid, 256, 0, stream>>>(
      (const __nv_bfloat16*)ah, (const __nv_bfloat16*)al, lda, (const __nv_bfloat16*)bh,
      (const __nv_bfloat16*)bl, ldb, M, N, K, grad, ldg);
  SPB_CHECK_LAUNCH("grad_gemm_simt");
  return 0;
}

}  // extern "C"

// K6 launcher: `splits` sample ranges, each over a grid of (2 * ceil(kp / 256),
// ceil(n_pad / 256)) CTAs (clusters of 2 along x).
extern "C" int spb_alif_carry_chunk(const void* wh, const void* wl, int ldw, const void* xh,
                                   const void* xl, const float* mdt, float* eps, float* partial,
                                   int B, int n, int n_pad, int k, int ke, int kp, int KR,
                                   int splits, int do_mma, int load_eps, int store_eps,
                                   const void* xs_hi, const void* xs_lo, cudaStream_t stream) {
  using namespace spb;
  SPB_CHECK_ARG(mdt && eps && partial, "spb_alif_carry_chunk: null pointer");
  const bool raw = xl == nullptr;
  SPB_CHECK_ARG(!(xs_hi && !raw) && !(xs_hi && !xs_lo),
                "spb_alif_carry_chunk: the entry-state term needs the raw operand (xl = NULL)");
  SPB_CHECK_ARG(!do_mma || (wh && wl && xh), "spb_alif_carry_chunk: missing GEMM operands");
  SPB_CHECK_ARG(n_pad % carry::BM == 0 && n <= n_pad && kp % 128 == 0 && kp >= k && ke >= k &&
                    ke % 4 == 0 && KR % carry::BK == 0,
                "spb_alif_carry_chunk: bad padding (n_pad %% 128, kp %% 128, ke %% 4, KR %% 32)");
  SPB_CHECK_ARG(B > 0 && splits > 0 && splits <= B, "spb_alif_carry_chunk: bad split");
  SPB_CHECK_ARG(!do_mma || (ldw >= n && ldw % 8 == 0), "spb_alif_carry_chunk: bad ldw");
  SPB_CHECK_ARG(!(store_eps && !do_mma), "spb_alif_carry_chunk: storing eps needs the GEMM");
  CUtensorMap mwh{}, mwl{}, mxh{}, mxl{}, meps{};
  if ((load_eps || store_eps) &&
      !make_tmap_2d(&meps, eps, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ke, (uint64_t)B * n_pad,
                    (uint64_t)ke * 4, 32, carry::BM, CU_TENSOR_MAP_SWIZZLE_128B)) {
    set_error("spb_alif_carry_chunk: cuTensorMapEncodeTiled (eps) failed");
    return 3;
  }
  if (do_mma) {
    const uint64_t K = (uint64_t)B * KR;
    const bool ok =
        make_tmap_2d(&mwh, wh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n, K, (uint64_t)ldw * 2, 64,
                     carry::BK, CU_TENSOR_MAP_SWIZZLE_128B) &&
        make_tmap_2d(&mwl, wl, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n, K, (uint64_t)ldw * 2, 64,
                     carry::BK, CU_TENSOR_MAP_SWIZZLE_128B) &&
        make_tmap_2d(&mxh, xh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kp, K, (uint64_t)kp * 2, 64,
                     carry::BK, CU_TENSOR_MAP_SWIZZLE_128B) &&
        make_tmap_2d(&mxl, raw ? xh : xl, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kp, K,
                     (uint64_t)kp * 2, 64, carry::BK, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!ok) {
      set_error("spb_alif_carry_chunk: cuTensorMapEncodeTiled failed");
      return 3;
    }
  }
  const int bps = ceil_div(B, splits);
  dim3 grid(2 * ceil_div(kp, carry::BN), ceil_div(n_pad, 2 * carry::BM), splits);
  const auto* whb = static_cast<const __nv_bfloat16*>(wh);
  const auto* wlb = static_cast<const __nv_bfloat16*>(wl);
  const auto* xsh = static_cast<const __nv_bfloat16*>(xs_hi);
  const auto* xsl = static_cast<const __nv_bfloat16*>(xs_lo);
  if (raw) {
    auto kfn = carry::alif_carry_pair_kernel<true>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, carry::Cfg<true>::SMEM);
    pdl_launch(kfn, grid, carry::THREADS, carry::Cfg<true>::SMEM, stream, mwh, mwl, mxh, mxl,
               meps, reinterpret_cast<const float2*>(mdt), partial, B, n, n_pad, kp, KR, bps,
               do_mma, load_eps, store_eps, whb, wlb, ldw, xsh, xsl);
  } else {
    auto kfn = carry::alif_carry_pair_kernel<false>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, carry::Cfg<false>::SMEM);
    pdl_launch(kfn, grid, carry::THREADS, carry::Cfg<false>::SMEM, stream, mwh, mwl, mxh, mxl,
               meps, reinterpret_cast<const float2*>(mdt), partial, B, n, n_pad, kp, KR, bps,
               do_mma, load_eps, store_eps, whb, wlb, ldw, (const __nv_bfloat16*)nullptr,
               (const __nv_bfloat16*)nullptr);
  }
  SPB_CHECK_LAUNCH("alif_carry");
  return 0;
}
