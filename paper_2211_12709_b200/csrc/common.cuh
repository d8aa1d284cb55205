// Shared device helpers for libdfno: complex arithmetic, retained-mode
// indexing, twiddle generation and the activations.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dfno.h"

namespace dfno {

template <typename R>
struct Cplx;
template <>
struct Cplx<float> {
  using T = float2;
};
template <>
struct Cplx<double> {
  using T = double2;
};
template <typename R>
using C = typename Cplx<R>::T;

template <typename R>
__device__ __forceinline__ C<R> cmk(R re, R im) {
  C<R> z;
  z.x = re;
  z.y = im;
  return z;
}

// acc += a * b
template <typename R>
__device__ __forceinline__ void cmac(C<R>& acc, const C<R>& a, const C<R>& b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

// acc += conj(a) * b
template <typename R>
__device__ __forceinline__ void cmac_conj_a(C<R>& acc, const C<R>& a, const C<R>& b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

// acc += a * conj(b)
template <typename R>
__device__ __forceinline__ void cmac_conj_b(C<R>& acc, const C<R>& a, const C<R>& b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
}

// Frequency of retained position j along a dim of extent n with m modes:
// positions {0..m-1} then {n-m..n-1}; identity when 2m >= n
// (reference d/spectral.py:55-66).
__host__ __device__ __forceinline__ int mode_freq(int j, int n, int m) {
  return (2 * m >= n) ? j : (j < m ? j : n - 2 * m + j);
}

// e^{sign * 2 pi i k x / n} with exact integer phase reduction (k*x mod n)
// evaluated in double precision, then rounded to R.
template <typename R>
__device__ __forceinline__ C<R> twiddle(int k, int x, int n, int sign) {
  long long idx = ((long long)k * (long long)x) % (long long)n;
  double s, c;
  sincospi(2.0 * (double)idx / (double)n, &s, &c);
  return cmk<R>((R)c, (R)(sign * s));
}

// Activations, reference ActivationKind d/fno.py:36-55.
__device__ __forceinline__ float erf_r(float v) { return erff(v); }
__device__ __forceinline__ double erf_r(double v) { return erf(v); }
__device__ __forceinline__ float exp_r(float v) { return expf(v); }
__device__ __forceinline__ double exp_r(double v) { return exp(v); }

// fp32 erf-GELU in ~15 instructions, |error| ~1e-7 (Abramowitz & Stegun
// 7.1.26 for erf, 1.5e-7):  erf(x) = 1 - t P(t) e^{-x^2}, t = 1 / (1 + p x).
// Phi(h) = 0.5 (1 + erf(h / sqrt 2)); e = e^{-h^2 / 2} is returned for the
// derivative gelu'(h) = Phi(h) + h e / sqrt(2 pi).  Uses the MUFU rcp / ex2
// approximations directly.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float phi_fast(float h, float& e) {
  const float x = fabsf(h) * 0.70710678118654752f;
  const float t = rcp_approx(fmaf(0.3275911f, x, 1.0f));
  // 0.5 * (a1 t + ... + a5 t^5), coefficients pre-halved
  float p = fmaf(0.5307027145f, t, -0.7265760135f);
  p = fmaf(p, t, 0.7107068705f);
  p = fmaf(p, t, -0.142248368f);
  p = fmaf(p, t, 0.127414796f);
  p *= t;
  e = ex2_approx(h * (h * -0.72134752044448170f));  // e^{-h^2/2} = 2^{-h^2 log2(e) / 2}
  const float q = p * e;                             // 0.5 (1 - erf(|x|))
  return 0.5f + copysignf(0.5f - q, h);
}

template <typename R>
__device__ __forceinline__ R act_apply(int act, R h) {
  if (act == DFNO_ACT_GELU) {
    if constexpr (sizeof(R) == 4) {
      float e;
      return h * phi_fast(h, e);
    } else {
      const R inv_sqrt2 = (R)0.70710678118654752440;
      return (R)0.5 * h * ((R)1 + erf_r(h * inv_sqrt2));
    }
  }
  if (act == DFNO_ACT_RELU) return h > (R)0 ? h : (R)0;
  return h;
}

template <typename R>
__device__ __forceinline__ R act_deriv(int act, R h) {
  if (act == DFNO_ACT_GELU) {
    if constexpr (sizeof(R) == 4) {
      float e;
      const float c = phi_fast(h, e);
      return fmaf(h * 0.3989422804014327f, e, c);
    } else {
      const R inv_sqrt2 = (R)0.70710678118654752440;
      const R inv_sqrt2pi = (R)0.39894228040143267794;
      return (R)0.5 * ((R)1 + erf_r(h * inv_sqrt2)) + h * inv_sqrt2pi * exp_r((R)-0.5 * h * h);
    }
  }
  if (act == DFNO_ACT_RELU) return h > (R)0 ? (R)1 : (R)0;
  return (R)1;
}

// Rank helpers on the geometry.
__host__ __device__ __forceinline__ int x_local(const dfno_geom& g) {
  return g.x_starts[g.rank + 1] - g.x_starts[g.rank];
}
__host__ __device__ __forceinline__ int ky_local(const dfno_geom& g) {
  return g.ky_starts[g.rank + 1] - g.ky_starts[g.rank];
}

// Owner of global ky position `ky` under the ky partition.
__device__ __forceinline__ int ky_owner(const dfno_geom& g, int ky) {
  int p = 0;
  while (ky >= g.ky_starts[p + 1]) ++p;
  return p;
}
__device__ __forceinline__ int x_owner(const dfno_geom& g, int x) {
  int p = 0;
  while (x >= g.x_starts[p + 1]) ++p;
  return p;
}

// Element offset of (bb, ch, xl, ky) row in the XK layout (this rank's
// x slab, all ky across peer chunks): chunk p starts at
// B*C*XL*RZ*RT*ky_starts[p]; inside it [b][c][xl][ky - ky_starts[p]][rz][rt].
__device__ __forceinline__ long long xk_row(const dfno_geom& g, int bb, int ch, int xl, int ky) {
  const int XL = x_local(g);
  const long long rzt = (long long)g.rz * g.rt;
  const int p = ky_owner(g, ky);
  const int kp = g.ky_starts[p + 1] - g.ky_starts[p];
  const long long base = (long long)g.batch * g.c * XL * rzt * g.ky_starts[p];
  return base + ((((long long)bb * g.c + ch) * XL + xl) * kp + (ky - g.ky_starts[p])) * rzt;
}

// Element offset of (bb, ch, x) row in the KX layout (this rank's ky pencil,
// all x across peer chunks): chunk p starts at B*C*KYL*RZ*RT*x_starts[p];
// inside it [b][c][x - x_starts[p]][ky_local][rz][rt].  Returned offset
// points at ky_local = 0, kz = 0, kt = 0; modes m = (kyl, kz, kt) follow
// contiguously.
__device__ __forceinline__ long long kx_row(const dfno_geom& g, int bb, int ch, int x) {
  const int KYL = ky_local(g);
  const long long mloc = (long long)KYL * g.rz * g.rt;
  const int p = x_owner(g, x);
  const int xp = g.x_starts[p + 1] - g.x_starts[p];
  const long long base = (long long)g.batch * g.c * mloc * g.x_starts[p];
  return base + (((long long)bb * g.c + ch) * xp + (x - g.x_starts[p])) * mloc;
}

}  // namespace dfno

#define DFNO_CUDA_CHECK_LAUNCH()                      \
  do {                                                \
    cudaError_t e__ = cudaGetLastError();             \
    if (e__ != cudaSuccess) return DFNO_ERR_CUDA;     \
  } while (0)
