// Training-step kernels (the first "next" row of the hot path: the caller of
// fno_forward / fno_backward in the reference's train_step,
// d/training.py:96-133).
//
//   k_mse_grad   one pass over (pred, target): resid = pred - target,
//                grad = scale * resid, per-CTA partial sums of resid^2 in
//                double (d/training.py:115-125); k_sum_partials adds the
//                partials in a fixed order (deterministic loss on every rank)
//   k_adam       Adam on the real view of each parameter (d/training.py:52-74)
//                with the reference's operation order and fp32 rounding of
//                every intermediate (no FMA contraction), so the updated
//                weights match numpy's float32 arithmetic bit for bit.
#include "common.cuh"

namespace dfno {

namespace {
constexpr int kTT = 256;

int sm_count_t() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}
}  // namespace

int mse_partials(long long n) {
  long long b = (n + kTT * 8 - 1) / (kTT * 8);
  const long long cap = (long long)sm_count_t() * 4;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

template <typename R>
__global__ void __launch_bounds__(kTT) k_mse_grad(long long n, const R* __restrict__ pred, const R* __restrict__ tgt,
                                                  R scale, R* __restrict__ grad, double* __restrict__ partials) {
  __shared__ double red[kTT / 32];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * kTT + threadIdx.x; i < n; i += (long long)gridDim.x * kTT) {
    const R r = pred[i] - tgt[i];
    if (grad) grad[i] = scale * r;
    acc += (double)r * (double)r;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kTT / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void k_sum_partials(int np, const double* __restrict__ partials, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < np; ++k) s += partials[k];
    out[0] = s;
  }
}

// m = b1 m + (1 - b1) g ; v = b2 v + (1 - b2) g^2 ;
// p -= lr * (m / c1) / (sqrt(v / c2) + eps)     (c1 = 1 - b1^t, c2 = 1 - b2^t)
// evaluated exactly in the reference's order with round-to-nearest on every
// operation (numpy float32 semantics: Python-float scalars rounded to R).
template <typename R>
__device__ __forceinline__ R mul_rn(R a, R b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename R>
__device__ __forceinline__ R add_rn(R a, R b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <typename R>
__device__ __forceinline__ R div_rn(R a, R b);
template <>
__device__ __forceinline__ float div_rn<float>(float a, float b) { return __fdiv_rn(a, b); }
template <>
__device__ __forceinline__ double div_rn<double>(double a, double b) { return __ddiv_rn(a, b); }
template <typename R>
__device__ __forceinline__ R sqrt_rn(R a);
template <>
__device__ __forceinline__ float sqrt_rn<float>(float a) { return __fsqrt_rn(a); }
template <>
__device__ __forceinline__ double sqrt_rn<double>(double a) { return __dsqrt_rn(a); }

template <typename R>
__global__ void __launch_bounds__(kTT) k_adam(long long n, const R* pin, R* p, const R* __restrict__ g,
                                              R* __restrict__ m, R* __restrict__ v, R lr, R b1, R one_m_b1, R b2,
                                              R one_m_b2, R c1, R c2, R eps) {
  for (long long i = (long long)blockIdx.x * kTT + threadIdx.x; i < n; i += (long long)gridDim.x * kTT) {
    const R gi = g[i];
    R mi = mul_rn(m[i], b1);                       // m *= beta1
    mi = add_rn(mi, mul_rn(one_m_b1, gi));         // m += (1 - beta1) * g
    R vi = mul_rn(v[i], b2);                       // v *= beta2
    vi = add_rn(vi, mul_rn(mul_rn(one_m_b2, gi), gi));  // v += (1 - beta2) * g * g
    const R m_hat = div_rn(mi, c1);
    const R v_hat = div_rn(vi, c2);
    const R upd = div_rn(mul_rn(lr, m_hat), add_rn(sqrt_rn(v_hat), eps));
    p[i] = add_rn(pin[i], -upd);                   // p -= lr * m_hat / (sqrt(v_hat) + eps)
    m[i] = mi;
    v[i] = vi;
  }
}

// fp32, four elements per thread per iteration (16-byte loads and stores:
// four times the bytes in flight of k_adam), same per-element arithmetic.
__device__ __forceinline__ void adam1(float& p, float gi, float& m, float& v, float lr, float b1, float one_m_b1,
                                      float b2, float one_m_b2, float c1, float c2, float eps) {
  float mi = mul_rn(m, b1);
  mi = add_rn(mi, mul_rn(one_m_b1, gi));
  float vi = mul_rn(v, b2);
  vi = add_rn(vi, mul_rn(mul_rn(one_m_b2, gi), gi));
  const float upd = div_rn(mul_rn(lr, div_rn(mi, c1)), add_rn(sqrt_rn(div_rn(vi, c2)), eps));
  p = add_rn(p, -upd);
  m = mi;
  v = vi;
}

// pin may alias p (in place) or not (the updated parameter written to a fresh
// buffer: no copy pass before the update)
__global__ void __launch_bounds__(kTT) k_adam4(long long n4, const float4* pin, float4* p, const float4* __restrict__ g,
                                               float4* __restrict__ m, float4* __restrict__ v, float lr, float b1,
                                               float one_m_b1, float b2, float one_m_b2, float c1, float c2,
                                               float eps) {
  for (long long i = (long long)blockIdx.x * kTT + threadIdx.x; i < n4; i += (long long)gridDim.x * kTT) {
    const float4 gi = __ldcs(g + i);
    float4 pi = __ldcs(pin + i), mi = __ldcs(m + i), vi = __ldcs(v + i);
    adam1(pi.x, gi.x, mi.x, vi.x, lr, b1, one_m_b1, b2, one_m_b2, c1, c2, eps);
    adam1(pi.y, gi.y, mi.y, vi.y, lr, b1, one_m_b1, b2, one_m_b2, c1, c2, eps);
    adam1(pi.z, gi.z, mi.z, vi.z, lr, b1, one_m_b1, b2, one_m_b2, c1, c2, eps);
    adam1(pi.w, gi.w, mi.w, vi.w, lr, b1, one_m_b1, b2, one_m_b2, c1, c2, eps);
    __stcs(p + i, pi);
    __stcs(m + i, mi);
    __stcs(v + i, vi);
  }
}

}  // namespace dfno

using namespace dfno;

extern "C" int dfno_mse_partials(int64_t n, int* num_partials) {
  if (!num_partials) return DFNO_ERR_NULL;
  if (n < 0) return DFNO_ERR_DIMENSION;
  *num_partials = mse_partials(n);
  return DFNO_OK;
}

extern "C" int dfno_mse_grad(const dfno_geom* g, int64_t n, const void* pred, const void* target, double grad_scale,
                             void* grad_out, void* partials, void* sse_out, void* stream) {
  if (!g || !pred || !target || !partials || !sse_out) return DFNO_ERR_NULL;
  if (n < 0) return DFNO_ERR_DIMENSION;
  cudaStream_t st = (cudaStream_t)stream;
  const int np = mse_partials(n);
  if (g->dtype == DFNO_F32)
    k_mse_grad<float><<<np, kTT, 0, st>>>(n, (const float*)pred, (const float*)target, (float)grad_scale,
                                           (float*)grad_out, (double*)partials);
  else if (g->dtype == DFNO_F64)
    k_mse_grad<double><<<np, kTT, 0, st>>>(n, (const double*)pred, (const double*)target, grad_scale,
                                            (double*)grad_out, (double*)partials);
  else
    return DFNO_ERR_DTYPE;
  DFNO_CUDA_CHECK_LAUNCH();
  k_sum_partials<<<1, 32, 0, st>>>(np, (const double*)partials, (double*)sse_out);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

namespace {
int adam_launch(const dfno_geom* g, int64_t n, const void* pin, void* param, const void* grad, void* m, void* v,
                double lr, double beta1, double beta2, double eps, int step, void* stream) {
  if (!g || !pin || !param || !grad || !m || !v) return DFNO_ERR_NULL;
  if (n < 0 || step < 1) return DFNO_ERR_DIMENSION;
  if (n == 0) return DFNO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  long long blocks = (n + kTT - 1) / kTT;
  const long long cap = (long long)sm_count_t() * 8;
  if (blocks > cap) blocks = cap;
  // scalar operands as numpy forms them: Python floats (double) rounded to
  // the array dtype at each binary op (d/training.py:66-73)
  const double c1 = 1.0 - pow(beta1, step), c2 = 1.0 - pow(beta2, step);
  const bool vec4 = g->dtype == DFNO_F32 && n % 4 == 0 &&
                    (((uintptr_t)pin | (uintptr_t)param | (uintptr_t)grad | (uintptr_t)m | (uintptr_t)v) & 15) == 0;
  if (vec4) {
    long long b4 = (n / 4 + kTT - 1) / kTT;
    if (b4 > cap) b4 = cap;
    k_adam4<<<(unsigned)b4, kTT, 0, st>>>(n / 4, (const float4*)pin, (float4*)param, (const float4*)grad,
                                          (float4*)m, (float4*)v, (float)lr, (float)beta1, (float)(1.0 - beta1),
                                          (float)beta2, (float)(1.0 - beta2), (float)c1, (float)c2, (float)eps);
  } else if (g->dtype == DFNO_F32)
    k_adam<float><<<(unsigned)blocks, kTT, 0, st>>>(n, (const float*)pin, (float*)param, (const float*)grad,
                                                    (float*)m, (float*)v, (float)lr, (float)beta1,
                                                    (float)(1.0 - beta1), (float)beta2, (float)(1.0 - beta2),
                                                    (float)c1, (float)c2, (float)eps);
  else if (g->dtype == DFNO_F64)
    k_adam<double><<<(unsigned)blocks, kTT, 0, st>>>(n, (const double*)pin, (double*)param, (const double*)grad,
                                                     (double*)m, (double*)v, lr, beta1, 1.0 - beta1, beta2,
                                                     1.0 - beta2, c1, c2, eps);
  else
    return DFNO_ERR_DTYPE;
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}
}  // namespace

extern "C" int dfno_adam(const dfno_geom* g, int64_t n, void* param, const void* grad, void* m, void* v, double lr,
                         double beta1, double beta2, double eps, int step, void* stream) {
  return adam_launch(g, n, param, param, grad, m, v, lr, beta1, beta2, eps, step, stream);
}

extern "C" int dfno_adam_out(const dfno_geom* g, int64_t n, const void* param, void* param_out, const void* grad,
                             void* m, void* v, double lr, double beta1, double beta2, double eps, int step,
                             void* stream) {
  return adam_launch(g, n, param, param_out, grad, m, v, lr, beta1, beta2, eps, step, stream);
}
