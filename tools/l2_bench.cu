// L2 -> SM read bandwidth on this B200, the roofline of the recurrent gather (K1rec):
//   stream: every CTA reads a 32 MB fp32 buffer (L2-resident after the first pass) with
//           16-byte loads, grid-stride, 40 passes;
//   gather: one CTA per "sample" (2 per SM, 512 threads) reads pseudo-random 4 KB rows of
//           a 4 MB matrix (the fp32 W_rec^T of n = 1024) the way K1rec gathers the rows of
//           the active presynaptic neurons (float2 per thread, 8 rows in flight).
// Prints one JSON line: {"l2_stream_gbs": ..., "l2_gather_gbs": ...}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bench tools/l2_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void stream_kernel(const float4* __restrict__ buf, long long n4, int passes,
                              float* __restrict__ sink) {
  float acc = 0.f;
  for (int p = 0; p < passes; ++p)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
      const float4 v = __ldcg(buf + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1.2345f) sink[0] = acc;
}

__global__ void __launch_bounds__(512, 2) gather_kernel(const float2* __restrict__ w, int rows,
                                                        int steps, float* __restrict__ sink) {
  // row = 1024 floats = 512 float2: one float2 per thread per row
  float2 acc = make_float2(0.f, 0.f);
  uint32_t h = 2654435761u * (blockIdx.x + 1);
  for (int s = 0; s < steps; ++s) {
    float2 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      h = h * 1664525u + 1013904223u;
      const int r = (int)(h % (uint32_t)rows);
      v[q] = __ldcg(w + (long long)r * 512 + threadIdx.x);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      acc.x += v[q].x;
      acc.y += v[q].y;
    }
  }
  if (acc.x == 1.2345f) sink[0] = acc.y;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *buf, *sink;
  const long long n_floats = 8LL << 20;  // 32 MB
  cudaMalloc(&buf, n_floats * 4);
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 0, n_floats * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f;
  const int passes = 40;
  double best_stream = 0.0, best_gather = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    stream_kernel<<<sms * 4, 512>>>(reinterpret_cast<const float4*>(buf), n_floats / 4, 1, sink);
    cudaEventRecord(e0);
    stream_kernel<<<sms * 4, 512>>>(reinterpret_cast<const float4*>(buf), n_floats / 4, passes,
                                    sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = (double)n_floats * 4 * passes / (ms * 1e-3) / 1e9;
    if (gbs > best_stream) best_stream = gbs;
  }
  const int rows = 1024, steps = 2000, ctas = 2 * sms;
  for (int rep = 0; rep < 3; ++rep) {
    gather_kernel<<<ctas, 512>>>(reinterpret_cast<const float2*>(buf), rows, 10, sink);
    cudaEventRecord(e0);
    gather_kernel<<<ctas, 512>>>(reinterpret_cast<const float2*>(buf), rows, steps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = (double)ctas * steps * 8 * 4096 / (ms * 1e-3) / 1e9;
    if (gbs > best_gather) best_gather = gbs;
  }
  printf("{\"l2_stream_gbs\": %.1f, \"l2_gather_gbs\": %.1f, \"how\": \"tools/l2_bench.cu: "
         "32 MB fp32 L2-resident stream (16-byte loads, %d CTAs x 512), and 4 KB-row gathers "
         "(2 CTAs/SM x 512 threads, 8 rows in flight), best of 3\", \"err\": \"%s\"}\n",
         best_stream, best_gather, sms * 4, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
