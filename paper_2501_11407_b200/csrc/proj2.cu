// K2 on CTA PAIRS: the exact INT8 input projection with tcgen05.mma.cta_group::2 (sm_100a).
//
// Same arithmetic and output as proj.cu (digits.cuh): I = W x_t exactly, rounded once to
// fp64.  What changes is the operand flow.  In the single-CTA kernel every MMA
// (M=128 rows x N=P*32 digit-neuron columns x K=32 bytes) reads its A tile (spike rows)
// and its B tile (weight digits) from the SM's shared memory -- ~10 KB per 96-cycle MMA at
// N = 192, together with the TMA writes of the spike stream more than the shared-memory
// port sustains, and the 147 KB weight tile leaves room for only 5 spike stages.  Here two
// CTAs of a cluster run ONE M=256 MMA: each CTA supplies its own 128 spike rows (A) and
// HALF of the weight digits (B rows [r*N/2, (r+1)*N/2) -- digits 0..P/2-1 on rank 0,
// P/2..P-1 on rank 1), and receives its 128 rows x all N columns in its own TMEM.  Per SM
// the B reads and the resident weight tile halve (72 KB at P = 6), so 8 spike stages fit.
//
// Roles (both CTAs): warp 0 TMA producer (own W half once per neuron tile, own spike rows
// per K block; transaction bytes land on the LEADER's barriers), warp 1 TMEM allocator
// (cta_group::2) and, on the leader only, the MMA issuer (commits multicast to both CTAs),
// warps 2-9 epilogue (proj.cu's, arriving on the leader's TMEM-empty barrier).
#include "tma.cuh"
#include "digits.cuh"

namespace spb {
namespace proj2 {

constexpr int BM = 128;       // spike rows per CTA (the pair covers 256)
constexpr int NT = 32;        // neurons per tile
constexpr int BK = 128;       // K bytes per stage
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 TMEM/MMA, warps 2-9 epilogue
constexpr int EPI_WARPS = 8;
constexpr int TILE_A = BM * BK;
constexpr int MAXKB = 6;      // Kpad <= 768
constexpr int NH = NT / 2;    // neurons per epilogue thread

template <int P, int XS>
struct Cfg {
  static_assert(P % 2 == 0, "the weight digits split evenly over the CTA pair");
  static constexpr int N = P * NT;                 // full MMA N (192 / 256)
  static constexpr int DH = P / 2;                 // digits held by each CTA
  static constexpr int WBLK = DH * NT * BK;        // one K block of this CTA's digits
  static constexpr int W_BYTES = MAXKB * WBLK;
  static constexpr int SMEM = W_BYTES + XS * TILE_A + 1024 + 256;
  static constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (1u << 10) |
                                    ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
// TMA into this CTA's smem, completing transaction bytes on the LEADER's barrier
__device__ __forceinline__ void tma_load_2sm(uint32_t dst, const CUtensorMap* map,
                                             uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ void mma2_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// arrive on the barrier at this offset in BOTH CTAs once the issued MMAs complete
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\t.reg .pred e;\n\tmov.b16 m, 3;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, int32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Epilogue of this CTA's 128 rows x 32 neurons (as proj.cu: exact recombination, 8x8
// warp transpose, 4 full lines per store), the TMEM release going to the leader.
template <int P, bool BIN>
__device__ __forceinline__ void epilogue_tile(uint32_t tbase, const int (&se)[NH],
                                              double* __restrict__ out, int M, int n, int row,
                                              int i0, uint32_t leader_tempty, int lane) {
  long long g0[NH], g1[NH];
  {
    int32_t r[3][NH];
#pragma unroll
    for (int p = 0; p < 3; ++p) tmem_ld16_nowait(tbase + p * NT, r[p]);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < NH; ++c) g0[c] = digits_g0<P>(r[0][c], r[1][c], r[2][c]);
  }
  {
    int32_t r[P - 3][NH];
#pragma unroll
    for (int p = 3; p < P; ++p) tmem_ld16_nowait(tbase + p * NT, r[p - 3]);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < NH; ++c) {
      long long v = r[0][c];
#pragma unroll
      for (int p = 1; p < P - 3; ++p) v = (v << Digits<P>::RB) + r[p][c];
      g1[c] = v;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  if (lane == 0) arrive_remote(leader_tempty);
  double2 ch[NH / 2];
#pragma unroll
  for (int c = 0; c < NH; c += 2)
    ch[c / 2] = make_double2(digits_current<P, BIN>(g0[c], g1[c], se[c]),
                             digits_current<P, BIN>(g0[c + 1], g1[c + 1], se[c + 1]));
  const int p8 = lane & 7;
#pragma unroll
  for (int sh = 4; sh >= 1; sh >>= 1) {
    const bool up = (p8 & sh) != 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k & sh) continue;
      const double2 send = up ? ch[k] : ch[k | sh];
      double2 recv;
      recv.x = __shfl_xor_sync(0xffffffffu, send.x, sh);
      recv.y = __shfl_xor_sync(0xffffffffu, send.y, sh);
      if (up) ch[k] = recv; else ch[k | sh] = recv;
    }
  }
  const int row0 = row - p8;
  const int col = i0 + 2 * p8;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int r = row0 + k;
    if (r < M) {
      double* o = out + (long long)r * n + col;
      if (col + 1 < n && (n & 1) == 0) {  // 16-byte aligned rows
        *reinterpret_cast<double2*>(o) = ch[k];
      } else {
        if (col < n) o[0] = ch[k].x;
        if (col + 1 < n) o[1] = ch[k].y;
      }
    }
  }
}

template <int P, int XS, bool BIN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    input_proj_pair_kernel(const __grid_constant__ CUtensorMap tm_x,
                           const __grid_constant__ CUtensorMap tm_w, const int* __restrict__ sexp,
                           double* __restrict__ out, int M, int n, int n_pad32, int nkb) {
  using C = Cfg<P, XS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* wsm = smem;                        // [nkb][DH*NT rows][128 B]
  uint8_t* xsm = smem + C::W_BYTES;           // [XS][128 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xsm + XS * TILE_A);
  uint64_t* xfull = bars;
  uint64_t* xempty = bars + XS;
  uint64_t* tfull = bars + 2 * XS;
  uint64_t* tempty = bars + 2 * XS + 2;
  uint64_t* wfull = bars + 2 * XS + 4;
  uint64_t* wempty = bars + 2 * XS + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * XS + 6);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int m2_tiles = (M + 2 * BM - 1) / (2 * BM);
  const int n_tiles = (n + NT - 1) / NT;
  const long long total = (long long)m2_tiles * n_tiles;
  const int ncl = gridDim.x / 2, cl = blockIdx.x / 2;
  const int t_begin = (int)(total * cl / ncl);
  const int t_end = (int)(total * (cl + 1) / ncl);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < XS; ++s) {
      mbar_init(smem_u32(&xfull[s]), 1);
      mbar_init(smem_u32(&xempty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 2 * EPI_WARPS);  // epilogue warps of BOTH CTAs
    }
    mbar_init(smem_u32(wfull), 1);
    mbar_init(smem_u32(wempty), 1);
    mbar_fence_init();
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w);
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

  if (warp == 0) {
    if (lane == 0) {
      int it = 0, wl = 0, cur_nt = -1;
      for (int t = t_begin; t < t_end; ++t) {
        const int nt = t / m2_tiles, mt2 = t % m2_tiles;
        if (nt != cur_nt) {  // this CTA's weight digits of the neuron tile, all K blocks
          mbar_wait(smem_u32(wempty), (wl & 1) ^ 1);
          if (leader) mbar_expect_tx(smem_u32(wfull), 2 * nkb * C::WBLK);
          const uint32_t lb = mapa(smem_u32(wfull), 0);
          for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
            for (int d = 0; d < C::DH; ++d)
              tma_load_2sm(smem_u32(wsm + kb * C::WBLK + d * NT * BK), &tm_w, lb, kb * BK,
                           ((int)rank * C::DH + d) * n_pad32 + nt * NT);
          cur_nt = nt;
          ++wl;
        }
        const int row = mt2 * 2 * BM + (int)rank * BM;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % XS;
          mbar_wait(smem_u32(&xempty[s]), ((it / XS) & 1) ^ 1);
          if (leader) mbar_expect_tx(smem_u32(&xfull[s]), 2 * TILE_A);
          tma_load_2sm(smem_u32(xsm + s * TILE_A), &tm_x, mapa(smem_u32(&xfull[s]), 0), kb * BK,
                       row);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // whole warp, converged; elect.sync picks the issuer
      int it = 0, lt = 0, wl = 0, cur_nt = -1;
      for (int t = t_begin; t < t_end; ++t, ++lt) {
        const int nt = t / m2_tiles;
        if (nt != cur_nt) {
          mbar_wait_cluster(smem_u32(wfull), wl & 1);
          cur_nt = nt;
          ++wl;
        }
        const int a = lt & 1;
        mbar_wait_cluster(smem_u32(&tempty[a]), ((lt >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem_base + (uint32_t)(a * 256);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % XS;
          mbar_wait_cluster(smem_u32(&xfull[s]), (it / XS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t xa = smem_u32(xsm + s * TILE_A);
          const uint32_t wa = smem_u32(wsm + kb * C::WBLK);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            mma2_i8(dacc, desc_k_sw128(xa + kk * 32), desc_k_sw128(wa + kk * 32), C::IDESC,
                    (kb | kk) ? 1u : 0u);
          commit2(smem_u32(&xempty[s]));
        }
        commit2(smem_u32(&tfull[a]));
        if (t + 1 == t_end || (t + 1) / m2_tiles != nt) commit2(smem_u32(wempty));
      }
    }
  } else {
    const int q = warp & 3;
    const int hh = (warp - 2) >> 2;
    const uint32_t leader_tempty[2] = {mapa(smem_u32(&tempty[0]), 0),
                                       mapa(smem_u32(&tempty[1]), 0)};
    int lt = 0;
    for (int t = t_begin; t < t_end; ++t, ++lt) {
      const int nt = t / m2_tiles, mt2 = t % m2_tiles;
      const int a = lt & 1;
      const int i0 = nt * NT + hh * NH;
      int se[NH];
#pragma unroll
      for (int c = 0; c < NH; ++c) se[c] = (i0 + c < n) ? __ldg(sexp + i0 + c) : 0;
      mbar_wait(smem_u32(&tfull[a]), (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      epilogue_tile<P, BIN>(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * 256 + hh * NH),
                            se, out, M, n, mt2 * 2 * BM + (int)rank * BM + q * 32 + lane, i0,
                            leader_tempty[a], lane);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the peer is done with the pair's TMEM and barriers
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

}  // namespace proj2
}  // namespace spb

using namespace spb;

extern "C" {

// K2 on CTA pairs (even P only: 6 = f32 radix-256 digits, 8 = f64), Kpad <= 768.
int spb_input_proj_pair(const uint8_t* xq, const int8_t* wq, const int* sexp, int M, int n,
                        int n_pad32, int Kpad, int P, double* out, int sm_count, int binary,
                        cudaStream_t stream) {
  SPB_CHECK_ARG(xq && wq && sexp && out && M > 0 && n > 0 && n_pad32 >= n && n_pad32 % 32 == 0 &&
                    Kpad % proj2::BK == 0 && Kpad / proj2::BK <= proj2::MAXKB &&
                    (P == 6 || P == 8),
                "spb_input_proj_pair: bad args (P in {6, 8}, Kpad <= 768)");
  SPB_CHECK_ARG((reinterpret_cast<uintptr_t>(xq) | reinterpret_cast<uintptr_t>(wq)) % 16 == 0,
                "spb_input_proj_pair: operands must be 16-byte aligned");
  CUtensorMap mx, mw;
  const bool ok =
      make_tmap_2d(&mx, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, M, Kpad, proj2::BK, proj2::BM,
                   CU_TENSOR_MAP_SWIZZLE_128B) &&
      make_tmap_2d(&mw, wq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kpad, (uint64_t)P * n_pad32, Kpad,
                   proj2::BK, proj2::NT, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!ok) {
    set_error("spb_input_proj_pair: cuTensorMapEncodeTiled failed");
    return 3;
  }
  const int units = ((M + 255) / 256) * ((n + 31) / 32);
  const int sms = sm_count > 0 ? sm_count : 148;
  const int pairs = max(1, min(units, sms / 2));
  const int nkb = Kpad / proj2::BK;
  const bool bin = binary != 0 && P == 6;
  if (P == 6) {
    auto kfn = bin ? proj2::input_proj_pair_kernel<6, 8, true> : proj2::input_proj_pair_kernel<6, 8, false>;
    constexpr int sm = proj2::Cfg<6, 8>::SMEM;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    kfn<<<2 * pairs, proj2::THREADS, sm, stream>>>(mx, mw, sexp, out, M, n, n_pad32, nkb);
  } else {
    auto kfn = proj2::input_proj_pair_kernel<8, 7, false>;
    constexpr int sm = proj2::Cfg<8, 7>::SMEM;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    kfn<<<2 * pairs, proj2::THREADS, sm, stream>>>(mx, mw, sexp, out, M, n, n_pad32, nkb);
  }
  SPB_CHECK_LAUNCH("input_proj_pair");
  return 0;
}

}  // extern "C"
