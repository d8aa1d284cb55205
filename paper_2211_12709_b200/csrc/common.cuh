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
// fp32 GELU pieces: q = 0.5 erfc(|h| / sqrt 2) = p(t) e^{-h^2 / 2} with
// t = 1 / (1 + 0.3275911 |h| / sqrt 2) (A&S 7.1.26 erf, |error| <= 1.5e-7,
// coefficients pre-halved, MUFU rcp / ex2), e = e^{-h^2 / 2}.  Then
// GELU = h Phi(h) = relu(h) - |h| q and GELU' = Phi + h phi with Phi = 1 - q
// or q by the sign of h -- the same operations as the packed pair form below,
// so scalar and pair kernels agree bit for bit.
__device__ __forceinline__ float gelu_q(float h, float& nah, float& e) {
  nah = -fabsf(h);
  const float t = rcp_approx(fmaf(-0.23164188827f, nah, 1.0f));
  float p = fmaf(0.5307027145f, t, -0.7265760135f);
  p = fmaf(p, t, 0.7107068705f);
  p = fmaf(p, t, -0.142248368f);
  p = fmaf(p, t, 0.127414796f);
  p *= t;
  e = ex2_approx(h * (h * -0.72134752044448170f));  // e^{-h^2/2} = 2^{-h^2 log2(e) / 2}
  return p * e;
}

template <typename R>
__device__ __forceinline__ R act_apply(int act, R h) {
  if (act == DFNO_ACT_GELU) {
    if constexpr (sizeof(R) == 4) {
      float nah, e;
      const float q = gelu_q(h, nah, e);
      return fmaf(nah, q, fmaxf(h, 0.f));
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
      float nah, e;
      const float q = gelu_q(h, nah, e);
      return fmaf(h * 0.3989422804014327f, e, h > 0.f ? 1.f - q : q);
    } else {
      const R inv_sqrt2 = (R)0.70710678118654752440;
      const R inv_sqrt2pi = (R)0.39894228040143267794;
      return (R)0.5 * ((R)1 + erf_r(h * inv_sqrt2)) + h * inv_sqrt2pi * exp_r((R)-0.5 * h * h);
    }
  }
  if (act == DFNO_ACT_RELU) return h > (R)0 ? (R)1 : (R)0;
  return (R)1;
}

// ---- packed fp32x2 (FFMA2 / FMUL2 / FADD2 on sm_100a) ---------------------
// Two lanes of fp32 arithmetic per issued instruction: the streaming kernels
// that apply GELU / GELU' and the 3xTF32 split per element are issue-bound,
// so the converters work on element pairs.
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2s(float v) { return make_float2(v, v); }

// GELU on pairs without forming Phi: h Phi(h) = relu(h) - |h| q with
// q = 0.5 erfc(|h| / sqrt 2) = p(t) e^{-h^2 / 2} (the A&S 7.1.26 polynomial
// of gelu_q, t = 1 / (1 + 0.3275911 |h| / sqrt 2) with the two constants
// folded), and GELU' = Phi + h phi with Phi = 1 - q or q by the sign of h.
// Fewer instructions per pair than forming Phi = 0.5 + sign(h)(0.5 - q) (no
// sign copy, no 0.5 round trip); same erf approximation.
__device__ __forceinline__ void gelu_q2(float2 h, float2& nah, float2& q, float2& e) {
  nah = make_float2(-fabsf(h.x), -fabsf(h.y));
  const float2 d = f2fma(f2s(-0.23164188827f), nah, f2s(1.0f));
  const float2 t = make_float2(rcp_approx(d.x), rcp_approx(d.y));
  float2 p = f2fma(f2s(0.5307027145f), t, f2s(-0.7265760135f));
  p = f2fma(p, t, f2s(0.7107068705f));
  p = f2fma(p, t, f2s(-0.142248368f));
  p = f2fma(p, t, f2s(0.127414796f));
  p = f2mul(p, t);
  const float2 a = f2mul(h, f2mul(h, f2s(-0.72134752044448170f)));
  e = make_float2(ex2_approx(a.x), ex2_approx(a.y));
  q = f2mul(p, e);
}

__device__ __forceinline__ float2 gelu_fast2(float2 h) {
  float2 nah, q, e;
  gelu_q2(h, nah, q, e);
  return f2fma(nah, q, make_float2(fmaxf(h.x, 0.f), fmaxf(h.y, 0.f)));
}

template <int ACT>
__device__ __forceinline__ float2 act_apply2(float2 h) {
  if constexpr (ACT == DFNO_ACT_GELU) {
    return gelu_fast2(h);
  } else if constexpr (ACT == DFNO_ACT_RELU) {
    return make_float2(h.x > 0.f ? h.x : 0.f, h.y > 0.f ? h.y : 0.f);
  } else {
    return h;
  }
}

template <int ACT>
__device__ __forceinline__ float2 act_deriv2(float2 h) {
  if constexpr (ACT == DFNO_ACT_GELU) {
    // GELU' = Phi(h) + h phi(h), Phi = 1 - q or q by the sign of h (the same
    // evaluation as act_both2's derivative)
    float2 nah, q, e;
    gelu_q2(h, nah, q, e);
    const float2 c = make_float2(h.x > 0.f ? 1.f - q.x : q.x, h.y > 0.f ? 1.f - q.y : q.y);
    return f2fma(f2mul(h, f2s(0.3989422804014327f)), e, c);
  } else if constexpr (ACT == DFNO_ACT_RELU) {
    return make_float2(h.x > 0.f ? 1.f : 0.f, h.y > 0.f ? 1.f : 0.f);
  } else {
    return f2s(1.f);
  }
}

// act and act' of the same pair (one phi evaluation)
template <int ACT>
__device__ __forceinline__ void act_both2(float2 h, float2& a, float2& d) {
  if constexpr (ACT == DFNO_ACT_GELU) {
    // a exactly as act_apply2 (the weight-gradient partials must not depend on
    // which of the two the caller fused); Phi = 1 - q or q by the sign of h
    float2 nah, q, e;
    gelu_q2(h, nah, q, e);
    a = f2fma(nah, q, make_float2(fmaxf(h.x, 0.f), fmaxf(h.y, 0.f)));
    const float2 c = make_float2(h.x > 0.f ? 1.f - q.x : q.x, h.y > 0.f ? 1.f - q.y : q.y);
    d = f2fma(f2mul(h, f2s(0.3989422804014327f)), e, c);
  } else {
    a = act_apply2<ACT>(h);
    d = act_deriv2<ACT>(h);
  }
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
