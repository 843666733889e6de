// Probe of the tcgen05.ld.16x256b register layout: TMEM lane L, column c is written
// (tcgen05.st 32x32b: thread = lane, register j = column j) with L*100 + c, then read back
// with tcgen05.ld.16x256b.x2 at lane offsets 0 and 16.  Prints (lane, col) per register.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_layout_probe tools/tmem_layout_probe.cu
#include <cstdio>
#include <cstdint>
__global__ void probe(int* out) {
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  uint32_t v[16];
  for (int j = 0; j < 16; ++j) v[j] = t * 100 + j;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(tm), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
               "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  for (int h = 0; h < 2; ++h) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tm + ((uint32_t)(16 * h) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[(h * 32 + t) * 8 + j] = (int)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}
int main() {
  int* d; cudaMalloc(&d, 2 * 32 * 8 * 4);
  probe<<<1, 32>>>(d);
  int h[512]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  for (int hh = 0; hh < 2; ++hh) for (int t = 0; t < 32; t += 1) {
    if (t > 5 && t < 30) continue;
    printf("half %d thread %2d:", hh, t);
    for (int j = 0; j < 8; ++j) printf(" (L%d,c%d)", h[(hh * 32 + t) * 8 + j] / 100, h[(hh * 32 + t) * 8 + j] % 100);
    printf("\n");
  }
  return 0;
}
