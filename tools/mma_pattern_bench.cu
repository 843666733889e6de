// Microbenchmark of tcgen05 kind::i8 issue patterns at the K2 shape (M=128, N=192, K=32B):
//   mode 0: back-to-back MMAs, fixed descriptors
//   mode 1: descriptors walk 5 smem stages x 4 K-steps (distinct addresses, like K2)
//   mode 2: mode 1 + tcgen05.commit to an mbarrier after every 4 MMAs (no waits)
//   mode 3: mode 2 + a producer thread that waits each stage's commit and re-arms a "full"
//           barrier the MMA thread waits on (the K2 ring without TMA), depth 5
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_pattern_bench tools/mma_pattern_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar), "r"(phase) : "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
constexpr int XS = 5;
__global__ void __launch_bounds__(320, 1) bench(int mode, int stages_total, unsigned long long* cyc, int N, int fill) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[XS], empty[XS], done, tfull[2], tempty[2];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  // fill = 1: pseudo-random operand bytes (tensor-core power depends on the data)
  for (int i = tid; i < 224 * 1024; i += blockDim.x)
    base[i] = fill ? (uint8_t)((i * 2654435761u) >> 13) : 0;
  if (tid == 0) {
    for (int s = 0; s < XS; ++s) { mbar_init(su32(&full[s]), 1); mbar_init(su32(&empty[s]), 1); }
    mbar_init(su32(&done), 1);
    for (int a = 0; a < 2; ++a) { mbar_init(su32(&tfull[a]), 1); mbar_init(su32(&tempty[a]), mode >= 7 ? 8 : 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  // mode 9: K2's shared-memory layout -- six 192-row weight blocks (144 KB) first, the
  // five 16 KB spike stages after them
  const uint32_t xa0 = mode == 9 ? su32(base + 6 * 24576) : su32(base);
  const uint32_t wa0 = mode == 9 ? su32(base) : su32(base + XS * 16384);
  if (mode == 4 && tid < 32) {
    // warp-converged issue: every lane runs the loop, one elected lane issues (no R2UR /
    // divergent-uniform loop around each tcgen05.mma)
    const unsigned long long t0 = clock64();
    for (int it = 0; it < stages_total; ++it) {
      const int s = it % XS;
      const uint32_t xa = xa0 + s * 16384;
      const uint32_t wa = wa0 + (it % 4) * (N * 128);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "elect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(desc_k_sw128(xa + kk * 32)), "l"(desc_k_sw128(wa + kk * 32)), "r"(idesc), "r"(it | kk));
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&done)) : "memory");
    mbar_wait(su32(&done), 0);
    if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
  } else if (mode == 5 && tid < 32) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < stages_total; ++it) {
      const int s = it % XS;
      mbar_wait(su32(&full[s]), (it / XS) & 1);
      const uint32_t xa = xa0 + s * 16384;
      const uint32_t wa = wa0 + (it % 4) * (N * 128);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "elect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(desc_k_sw128(xa + kk * 32)), "l"(desc_k_sw128(wa + kk * 32)), "r"(idesc), "r"(it | kk));
      }
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&empty[s])) : "memory");
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&done)) : "memory");
    mbar_wait(su32(&done), 0);
    if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
  } else if (mode >= 6 && tid < 32) {
    // K2-like: tiles of 5.5 K blocks (22 MMAs), two TMEM accumulators (cols 0 / 256),
    // tfull commit per tile, the MMA warp waits the epilogue's tempty before reusing one
    const unsigned long long t0 = clock64();
    const int tiles = stages_total / 6;
    int it = 0;
    for (int t = 0; t < tiles; ++t) {
      const int a = t & 1;
      if (t >= 2) mbar_wait(su32(&tempty[a]), ((t >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kb = 0; kb < 6; ++kb, ++it) {
        const int s = it % XS;
        mbar_wait(su32(&full[s]), (it / XS) & 1);
        const uint32_t xa = xa0 + s * 16384;
        const uint32_t wa = mode == 9 ? wa0 + kb * (N * 128) : wa0 + kb * (N * 128) % (4 * N * 128);
        const int nk = kb < 5 ? 4 : 2;
        if (mode >= 8 && nk == 4) {   // K2's pattern: the 4 MMAs of a K block under one elect
          const uint64_t a0 = desc_k_sw128(xa), b0 = desc_k_sw128(wa);
          asm volatile(
              "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
              "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a2, b2, %3, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a3, b3, %3, 1;\n\t}" ::"r"(tmem + a * 256),
              "l"(a0), "l"(b0), "r"(idesc), "r"(kb));
        } else
        for (int kk = 0; kk < nk; ++kk) {
          asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "elect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + a * 256),
                       "l"(desc_k_sw128(xa + kk * 32)), "l"(desc_k_sw128(wa + kk * 32)), "r"(idesc), "r"(kb | kk));
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&empty[s])) : "memory");
      }
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&tfull[a])) : "memory");
    }
    mbar_wait(su32(&tfull[(tiles - 1) & 1]), ((tiles - 1) >> 1) & 1);
    if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
  } else if (mode >= 6 && tid >= 64 && (mode >= 7 || tid < 96)) {
    // "epilogue": wait tfull, arrive tempty (mode 6: one warp, mode 7: 8 warps like K2)
    const int tiles = stages_total / 6;
    for (int t = 0; t < tiles; ++t) {
      const int a = t & 1;
      mbar_wait(su32(&tfull[a]), (t >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if ((tid & 31) == 0) arrive(su32(&tempty[a]));
      __syncwarp();
    }
  } else if (tid == 32 && mode >= 6) {
    for (int it = 0; it < (stages_total / 6) * 6; ++it) {
      const int s = it % XS;
      if (it >= XS) mbar_wait(su32(&empty[s]), ((it / XS) - 1) & 1);
      arrive(su32(&full[s]));
    }
  } else if (tid == 32 && mode == 5) {
    for (int it = 0; it < stages_total; ++it) {
      const int s = it % XS;
      if (it >= XS) mbar_wait(su32(&empty[s]), ((it / XS) - 1) & 1);
      arrive(su32(&full[s]));
    }
  } else if (tid == 0 && mode < 4) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < stages_total; ++it) {
      const int s = it % XS;
      if (mode == 3) mbar_wait(su32(&full[s]), (it / XS) & 1);
      const uint32_t xa = (mode == 0) ? xa0 : xa0 + s * 16384;
      const uint32_t wa = (mode == 0) ? wa0 : wa0 + (it % 4) * (N * 128);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t off = (mode == 0) ? 0 : kk * 32;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(desc_k_sw128(xa + off)), "l"(desc_k_sw128(wa + off)), "r"(idesc), "r"(it | kk));
      }
      if (mode >= 2) commit(su32(&empty[s]));
    }
    commit(su32(&done));
    mbar_wait(su32(&done), 0);
    cyc[blockIdx.x] = clock64() - t0;
  } else if (tid == 32 && mode == 3) {
    for (int it = 0; it < stages_total; ++it) {
      const int s = it % XS;
      if (it >= XS) mbar_wait(su32(&empty[s]), ((it / XS) - 1) & 1);
      arrive(su32(&full[s]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int smem = 224 * 1024 + 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = getenv("MMA_STAGES") ? atoi(getenv("MMA_STAGES")) : 4000;
  for (int fill : {0, 1}) for (int N : {192}) for (int mode = 7; mode < 10; ++mode) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      bench<<<sms, 320, smem>>>(mode, stages, d, N, fill);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    unsigned long long c0 = 0;
    cudaMemcpy(&c0, d, 8, cudaMemcpyDeviceToHost);
    const double ops = 2.0 * 128 * N * 32 * (mode >= 6 ? 22.0 / 6.0 : 4.0) * stages * sms;
    printf("fill=%d N=%d mode %d: %.1f cyc/MMA, %.0f TOPS  err=%s\n", fill, N, mode, (double)c0 / ((mode >= 6 ? 22.0 / 6.0 : 4.0) * stages),
           ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
