// Microbenchmark: FP32 FFMA vs packed FFMA2 vs FP64 DFMA issue throughput on the
// box's B200, used to pick the ALIF eligibility kernel's arithmetic form.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) burn(float* out, int iters, float s) {
  float a[16]; double d[8];
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 8; i++) d[i] = threadIdx.x * 1e-3 + i;
  float b = s, c = s * 0.5f;
  for (int it = 0; it < iters; it++) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; i++) a[i] = fmaf(a[i], b, c);
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        unsigned long long x = *(unsigned long long*)&a[i];
        float2 bb = make_float2(b, b), cc = make_float2(c, c);
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(*(unsigned long long*)&bb), "l"(*(unsigned long long*)&cc));
        *(unsigned long long*)&a[i] = x;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; i++) d[i] = fma(d[i], (double)b, (double)c);
    }
  }
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) acc += a[i];
#pragma unroll
  for (int i = 0; i < 8; i++) acc += (float)d[i];
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; int blocks = sms * 8;
  const char* names[3] = {"ffma", "ffma2", "dfma"};
  for (int mode = 0; mode < 3; mode++) {
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      if (mode == 0) burn<0><<<blocks, 256>>>(out, iters, 0.999f);
      if (mode == 1) burn<1><<<blocks, 256>>>(out, iters, 0.999f);
      if (mode == 2) burn<2><<<blocks, 256>>>(out, iters, 0.999f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas = (double)blocks * 256 * iters * (mode == 2 ? 8 : 16);
      if (rep == 2) printf("%s: %.2f TFLOP/s (fma counted 2)  %.3f ms\n", names[mode], 2 * fmas / ms / 1e9, ms);
    }
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms=%d clock_khz=%d\n", sms, clk);
  return 0;
}
