// Microbenchmark: issue-rate-bound tcgen05.mma throughput per SM for kind::i8 and
// kind::f16 at several N (M = 128, cta_group::1, both operands in shared memory, K-major
// SW128 descriptors over zeroed smem).  One CTA per SM, one thread issues `iters` MMAs
// into one TMEM accumulator, commit + wait at the end.  Prints TOPS over all SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_microbench tools/mma_microbench.cu
#include <cstdio>
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

__device__ volatile int g_sink;
template <int KIND>  // 0 = i8, 1 = f16 (bf16)
__global__ void __launch_bounds__(128, 1) bench(int N, int iters, unsigned long long* cyc,
                                                 int ld_iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = tid; i < 64 * 1024; i += blockDim.x) base[i] = 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  uint32_t idesc;
  if (KIND == 0)
    idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  else
    idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t da = desc_k_sw128(su32(base));
  const uint64_t db = desc_k_sw128(su32(base + 32768));
  if (tid == 0) {
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(i));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
    const unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  } else if (tid >= 32 && ld_iters > 0) {
    // concurrent TMEM reads (x16 columns per load) from warps 1-3 on columns 128.., the
    // epilogue pattern of a double-buffered GEMM
    const int w = tid >> 5;
    uint32_t acc = 0;
    for (int i = 0; i < ld_iters; ++i) {
      uint32_t r[16];
      const uint32_t ta = tmem + ((uint32_t)(w * 32) << 16) + 128 + (i & 7) * 16;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int c = 0; c < 16; ++c) acc += r[c];
    }
    if (acc == 12345) g_sink = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  for (int ld : {0, 4000}) for (int kind = 0; kind < 2; ++kind) {
    for (int N : {64, 112, 128, 224, 256}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0) bench<0><<<sms, 128, smem>>>(N, iters, d, ld);
        else bench<1><<<sms, 128, smem>>>(N, iters, d, ld);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long c0 = 0;
      cudaMemcpy(&c0, d, 8, cudaMemcpyDeviceToHost);
      const double K = kind == 0 ? 32 : 16;
      const double ops = 2.0 * 128 * N * K * iters * sms;
      printf("ld=%d %s N=%3d: %.1f cyc/MMA (SM0), %.0f TOPS (event %.3f ms)  err=%s\n", ld,
             kind == 0 ? "i8 " : "f16", N, (double)c0 / iters, ops / (ms * 1e-3) / 1e12, ms,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
