// On-device optimizer steps fused after the gradient (and its allreduce): SURVEY.md 8(f)-1.
//
// Reference: sgd_update / adam_update (training.py:58-91).  The reference applies them to
// numpy arrays in the network's dtype with Python-float hyper-parameters, i.e. every
// operation is one IEEE operation in that dtype with the scalar first rounded to it
// (numpy 2 weak-scalar promotion):
//   sgd   p <- p - lr*g
//   adam  m <- b1*m + (1-b1)*g ; v <- b2*v + ((1-b2)*g)*g
//         p <- p - (lr*(m/(1-b1^t))) / (sqrt(v/(1-b2^t)) + eps)
// The kernels restate exactly that operation order with explicit round-to-nearest
// intrinsics (no FMA contraction), so a batch-1 run on the B200 applies the same update
// to the same gradient as the reference.
//
// Gradients come straight from the engine's accumulator (fp64 [rows][ld_g], or the
// packed fp32/fp64 allreduce buffer) and are scaled (1/B for a batch mean) and rounded
// to the parameter dtype first -- the reference hands the optimizer grads already cast
// to w.dtype (gradients.py:180-181).  `mirror` (optional) receives the updated parameter
// in fp64 (the readout weights the loss kernel reads).  Elementwise, HBM-bound: one
// thread per parameter, grid-stride.
#include "common.cuh"
#include "digits.cuh"

namespace spb {

template <typename T>
struct Op;
template <>
struct Op<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float sqrt(float a) { return __fsqrt_rn(a); }
};
template <>
struct Op<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt(double a) { return __dsqrt_rn(a); }
};

struct GradSrc {
  const void* g;
  int g_is_f64;
  int ld;
  double scale;
};

template <typename T>
__device__ __forceinline__ T load_grad(const GradSrc& s, long long r, long long c) {
  const long long o = r * s.ld + c;
  const double v = s.g_is_f64 ? static_cast<const double*>(s.g)[o]
                              : (double)static_cast<const float*>(s.g)[o];
  return (T)(s.scale == 1.0 ? v : __dmul_rn(v, s.scale));
}

template <typename T>
__global__ void sgd_kernel(T* __restrict__ p, GradSrc gs, int rows, int cols, T lr,
                           double* __restrict__ mirror) {
  using O = Op<T>;
  const long long total = (long long)rows * cols;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long r = idx / cols, c = idx - r * cols;
    const T g = load_grad<T>(gs, r, c);
    const T v = O::sub(p[idx], O::mul(lr, g));
    p[idx] = v;
    if (mirror) mirror[idx] = (double)v;
  }
}

template <typename T>
struct AdamScalars {
  T lr, b1, omb1, b2, omb2, bc1, bc2, eps;
};

template <typename T>
__global__ void adam_kernel(T* __restrict__ p, T* __restrict__ m, T* __restrict__ v, GradSrc gs,
                            int rows, int cols, AdamScalars<T> a, double* __restrict__ mirror) {
  using O = Op<T>;
  const long long total = (long long)rows * cols;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long r = idx / cols, c = idx - r * cols;
    const T g = load_grad<T>(gs, r, c);
    const T mn = O::add(O::mul(a.b1, m[idx]), O::mul(a.omb1, g));      // training.py:84
    const T vn = O::add(O::mul(a.b2, v[idx]), O::mul(O::mul(a.omb2, g), g));  // :85
    m[idx] = mn;
    v[idx] = vn;
    const T m_hat = O::div(mn, a.bc1);                                   // :87
    const T v_hat = O::div(vn, a.bc2);                                   // :88
    const T step = O::div(O::mul(a.lr, m_hat), O::add(O::sqrt(v_hat), a.eps));  // :89
    const T pn = O::sub(p[idx], step);
    p[idx] = pn;
    if (mirror) mirror[idx] = (double)pn;
  }
}

static int grid_for(long long total, int sm_count) {
  const long long want = (total + 255) / 256;
  const long long cap = (long long)(sm_count > 0 ? sm_count : 148) * 8;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

// ------------------------------------------------------------------------------------
// SGD on the input weights fused with their re-slicing into the INT8 projection digits
// (K2s, proj.cu / digits.cuh): CTA = one row of W.  Pass 1 applies p <- p - lr*g (the
// sgd_kernel arithmetic) and takes the row maximum; pass 2 re-reads the row (the warp's
// CTA's own fresh writes, L1-hot) and emits the P digit planes, 4 inputs per thread so every
// plane store is one 32-bit word.  do_sgd = 0 is plain slicing (spb_slice_weights).
// ------------------------------------------------------------------------------------
// scale46 = 2^(46-s) (P = 6): the product is exact, so w * scale46 == ldexp(w, 46 - s)
__device__ __forceinline__ void slice_one(double wv, int s, int P, int8_t (&q)[8],
                                          double scale46 = 0.0) {
  if (P == 6) {
    // balanced radix-256 digits of R = rint(w 2^(46-s)), |R| < 2^46, least significant
    // first: q = ((R + 128) mod 256) - 128 in [-128, 127], R <- (R - q) / 256 (exact)
    long long R = __double2ll_rn(wv * scale46);
#pragma unroll
    for (int p = 5; p >= 0; --p) {
      const long long d = ((R + 128) & 255) - 128;
      R = (R - d) >> 8;
      q[p] = (int8_t)d;
    }
  } else {  // radix-128 digits (P = 8: f64 weights; P = 7 kept for the digit tests)
    double r = ldexp(wv, -s);
    for (int p = 0; p < P; ++p) {
      const double t = r * (p == 0 ? 64.0 : 128.0);
      const double qv = rint(t);
      r = t - qv;
      q[p] = (int8_t)(int)qv;
    }
  }
}

constexpr int SS_THREADS = 256;  // one CTA per row of W

template <typename T>
__global__ void __launch_bounds__(SS_THREADS) sgd_slice_kernel(T* __restrict__ w, GradSrc gs,
                                                               int n, int k, T lr, int do_sgd,
                                                               int Kpad, int n_pad32, int P,
                                                               int8_t* __restrict__ wq,
                                                               int* __restrict__ sexp) {
  pdl_enter();
  using O = Op<T>;
  __shared__ double red[SS_THREADS / 32];
  const int i = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* row = w + (long long)i * k;
  double mx = 0.0;
  if (i < n) {
    for (int j = tid; j < k; j += SS_THREADS) {
      T v = row[j];
      if (do_sgd) {
        v = O::sub(v, O::mul(lr, load_grad<T>(gs, i, j)));
        row[j] = v;
      }
      mx = fmax(mx, fabs((double)v));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();  // also orders the row's updated values before pass 2 reads them
#pragma unroll
  for (int q = 0; q < SS_THREADS / 32; ++q) mx = fmax(mx, red[q]);
  int s = 0;
  if (mx > 0.0) frexp(mx, &s);  // mx = f * 2^s, f in [0.5, 1)  =>  |w| < 2^s
  if (tid == 0 && i < n) sexp[i] = s;
  // 2^(46-s) (f32 weights: 46 - s in [-82, 195], a normal double)
  const double sc46 = (P == 6) ? __longlong_as_double((long long)(46 - s + 1023) << 52) : 0.0;
  for (int j0 = 4 * tid; j0 < Kpad; j0 += 4 * SS_THREADS) {
    uint32_t word[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = j0 + e;
      const double wv = (i < n && j < k) ? (double)row[j] : 0.0;
      int8_t q[8];
      slice_one(wv, s, P, q, sc46);
      for (int p = 0; p < P; ++p) word[p] |= (uint32_t)(uint8_t)q[p] << (8 * e);
    }
    for (int p = 0; p < P; ++p)
      *reinterpret_cast<uint32_t*>(wq + ((long long)p * n_pad32 + wq_slot(i)) * Kpad + j0) =
          word[p];
  }
}

}  // namespace spb

using namespace spb;

// shared by spb_slice_weights (proj.cu) and spb_sgd_slice_update
extern "C" __attribute__((visibility("hidden"))) int spb_launch_sgd_slice(void* w, int w_is_f64, int n, int k, const void* g, int g_is_f64,
                         int ld_g, double g_scale, double lr, int do_sgd, int Kpad, int n_pad32,
                         int P, int8_t* wq, int* sexp, cudaStream_t stream) {
  const GradSrc gs{g, g_is_f64, ld_g, g_scale};
  const int blocks = n_pad32;
  if (w_is_f64)
    pdl_launch(sgd_slice_kernel<double>, blocks, SS_THREADS, 0, stream, static_cast<double*>(w), gs, n, k, lr,
                                                         do_sgd, Kpad, n_pad32, P, wq, sexp);
  else
    pdl_launch(sgd_slice_kernel<float>, blocks, SS_THREADS, 0, stream, static_cast<float*>(w), gs, n, k,
                                                        (float)lr, do_sgd, Kpad, n_pad32, P, wq,
                                                        sexp);
  SPB_CHECK_LAUNCH("sgd_slice");
  return 0;
}

extern "C" {

int spb_sgd_update(void* p, int p_is_f64, int rows, int cols, const void* g, int g_is_f64,
                   int ld_g, double g_scale, double lr, double* mirror, cudaStream_t stream) {
  SPB_CHECK_ARG(p && g && rows > 0 && cols > 0 && ld_g >= cols, "spb_sgd_update: bad args");
  const GradSrc gs{g, g_is_f64, ld_g, g_scale};
  const int grid = grid_for((long long)rows * cols, 148);
  if (p_is_f64)
    sgd_kernel<double><<<grid, 256, 0, stream>>>(static_cast<double*>(p), gs, rows, cols, lr,
                                                 mirror);
  else
    sgd_kernel<float><<<grid, 256, 0, stream>>>(static_cast<float*>(p), gs, rows, cols,
                                                (float)lr, mirror);
  SPB_CHECK_LAUNCH("sgd_update");
  return 0;
}

int spb_sgd_slice_update(void* w, int w_is_f64, int n, int k, const void* g, int g_is_f64,
                         int ld_g, double g_scale, double lr, int Kpad, int n_pad32, int P,
                         int8_t* wq, int* sexp, cudaStream_t stream) {
  SPB_CHECK_ARG(w && g && wq && sexp && n > 0 && k > 0 && ld_g >= k && Kpad >= k &&
                    Kpad % 128 == 0 && n_pad32 >= n && n_pad32 % 32 == 0 &&
                    (P == 6 || P == 7 || P == 8),
                "spb_sgd_slice_update: bad args");
  return spb_launch_sgd_slice(w, w_is_f64, n, k, g, g_is_f64, ld_g, g_scale, lr, 1, Kpad,
                              n_pad32, P, wq, sexp, stream);
}

int spb_adam_update(void* p, void* m, void* v, int p_is_f64, int rows, int cols, const void* g,
                    int g_is_f64, int ld_g, double g_scale, double lr, double beta1, double beta2,
                    double eps, int t, double* mirror, cudaStream_t stream) {
  SPB_CHECK_ARG(p && m && v && g && rows > 0 && cols > 0 && ld_g >= cols && t >= 1,
                "spb_adam_update: bad args");
  // Python-float scalars, computed in double exactly as the reference does, then
  // rounded once to the parameter dtype (numpy weak-scalar promotion)
  const double omb1 = 1.0 - beta1, omb2 = 1.0 - beta2;
  const double bc1 = 1.0 - pow(beta1, (double)t), bc2 = 1.0 - pow(beta2, (double)t);
  const GradSrc gs{g, g_is_f64, ld_g, g_scale};
  const int grid = grid_for((long long)rows * cols, 148);
  if (p_is_f64) {
    AdamScalars<double> a{lr, beta1, omb1, beta2, omb2, bc1, bc2, eps};
    adam_kernel<double><<<grid, 256, 0, stream>>>(static_cast<double*>(p), static_cast<double*>(m),
                                                  static_cast<double*>(v), gs, rows, cols, a,
                                                  mirror);
  } else {
    AdamScalars<float> a{(float)lr, (float)beta1, (float)omb1, (float)beta2,
                         (float)omb2, (float)bc1, (float)bc2, (float)eps};
    adam_kernel<float><<<grid, 256, 0, stream>>>(static_cast<float*>(p), static_cast<float*>(m),
                                                 static_cast<float*>(v), gs, rows, cols, a,
                                                 mirror);
  }
  SPB_CHECK_LAUNCH("adam_update");
  return 0;
}

}  // extern "C"
