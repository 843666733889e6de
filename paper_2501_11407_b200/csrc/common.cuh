// Shared helpers for the sparseprop-b200 kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "sparseprop-b200 targets sm_100a (B200) only"
#endif

namespace spb {

// Last error message of the C-ABI (thread-local, read by spb_last_error()).
void set_error(const char* fmt, ...);

#define SPB_CHECK_ARG(cond, ...)            \
  do {                                      \
    if (!(cond)) {                          \
      ::spb::set_error(__VA_ARGS__);        \
      return 2;                             \
    }                                       \
  } while (0)

#define SPB_CHECK_LAUNCH(name)                                                  \
  do {                                                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess) {                                                    \
      ::spb::set_error("%s launch failed: %s", name, cudaGetErrorString(e_));   \
      return 3;                                                                 \
    }                                                                           \
  } while (0)

// Programmatic dependent launch (PDL) between the kernels of one update on the main stream:
// a kernel launched by pdl_launch may be scheduled while its predecessor drains; it calls
// pdl_enter() first thing, which waits for the predecessor grid to complete (and its memory
// to be visible) and then lets its own dependent launch early.  Both instructions are
// no-ops for kernels launched without the attribute.  SPB_PDL=0 turns the attribute off.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// explicit early trigger: the dependent grid may be scheduled before this one drains
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
template <typename... K, typename... A>
inline cudaError_t pdl_launch(void (*kernel)(K...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<A&&>(args)...);
}

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline int round_up(int a, int b) { return ceil_div(a, b) * b; }

// Packed fp32x2 FMA (sm_100: FFMA2).  d = a*b + c elementwise on float2 pairs.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

// sigma'(d) = 1 / (1 + slope*|d|)^2  (reference graph.py:40-42), fp64, no contraction.
__device__ __forceinline__ double surrogate_grad_f64(double d, double slope) {
  double t = __dadd_rn(1.0, __dmul_rn(slope, fabs(d)));
  return __ddiv_rn(1.0, __dmul_rn(t, t));
}

// Same surrogate in fp32 for the gradient path (psi only scales fp32 eligibilities):
// 1/t^2 from the hardware reciprocal (MUFU.RCP, ~1 ulp; the IEEE-rounded __frcp_rn costs
// a Newton fix-up sequence in the instruction-bound dynamics loop).
__device__ __forceinline__ float surrogate_grad_f32(float d, float slope) {
  const float t = fmaf(slope, fabsf(d), 1.0f);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
  return r * r;
}

// z = spike(d): Theta(d) = [d >= 0] (graph.py:50-52) or, with smooth=True (the reference's
// finite-difference mode, gradients.py:114-115), 0.5 + d / (1 + slope |d|) in the
// reference's operation order.
__device__ __forceinline__ double spike_value(double d, bool smooth, double slope) {
  if (!smooth) return d >= 0.0 ? 1.0 : 0.0;
  return __dadd_rn(0.5, __ddiv_rn(d, __dadd_rn(1.0, __dmul_rn(slope, fabs(d)))));
}

// bf16 hi/lo split of an fp32 value: x ~= hi + lo with |x - hi - lo| <= 2^-16 |x|.
__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// Paired split: (hi, lo) bf16x2 words of two fp32 values (cvt.rn.bf16x2.f32).
__device__ __forceinline__ void split_bf16x2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

}  // namespace spb
