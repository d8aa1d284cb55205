// Truncated DFT over (y, z, t) of one rank's x-slab and its inverse --
// generic SIMT path (fp32 and fp64, any extents).  The fp32 production path
// for the common shapes is the tcgen05 kernel in dft_fwd_tc.cu / dft_inv_tc3.cu; this file is
// the reference-precision (real64) path and the fallback envelope.
//
// Forward replaces  fft_dims(a,(y,z,t)) + truncate_modes   (reference
// d/fno.py:328-329; backward use d/fno.py:446-448): only the retained r_y x r_z
// x r_t modes are ever computed, as dense contractions against twiddle tables
// generated on the fly in shared memory (exact integer phase reduction).
// Stages per CTA (one (b, c, x) slab, y processed in chunks of YC planes):
//   t  : U[y][z][kt]  = sum_t  f(a[y][z][t]) e^{-2 pi i kt t / Nt}   (real -> complex)
//   z  : V[y][kz][kt] = sum_z  U[y][z][kt]   e^{-2 pi i kz z / Nz}
//   y  : acc[ky][kz][kt] += sum_y V[y][kz][kt] e^{-2 pi i ky y / Ny}  (registers)
// The result is written straight into the peer-major XK exchange layout.
//
// Inverse replaces pad_modes + ifft_dims(yzt) + .real (d/fno.py:338-343,
// d/fno.py:459-464): y, then z (complex), then t keeping only the real part.
#include "common.cuh"

namespace dfno {

constexpr int kYztThreads = 256;
constexpr int kYztAccMax = 16;  // complex accumulators per thread

template <typename R, int ACC>
__global__ void __launch_bounds__(kYztThreads) k_yzt_fwd(const dfno_geom g, const R* __restrict__ src,
                                                         const R* __restrict__ pre, int src_mode, R scale,
                                                         C<R>* __restrict__ out, int YC, int kyc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Ny = g.ny, Nz = g.nz, Nt = g.nt, rz = g.rz, rt = g.rt;
  const int XL = x_local(g);
  const int slab = blockIdx.x;  // (bb, ch, xl)
  const int xl = slab % XL;
  const int ch = (slab / XL) % g.c;
  const int bb = slab / (XL * g.c);
  const int ky0 = blockIdx.y * kyc;
  const int kyn = min(kyc, g.ry - ky0);

  C<R>* twt = reinterpret_cast<C<R>*>(smem_raw);  // [Nt][rt]
  C<R>* twz = twt + Nt * rt;                       // [Nz][rz]
  C<R>* twy = twz + Nz * rz;                       // [Ny][kyc]
  C<R>* U = twy + Ny * kyc;                        // [YC][Nz][rt]
  C<R>* V = U + YC * Nz * rt;                      // [YC][rz][rt]
  R* plane = reinterpret_cast<R*>(V + YC * rz * rt);  // [YC][Nz][Nt]

  const int tid = threadIdx.x;
  for (int e = tid; e < Nt * rt; e += blockDim.x) {
    const int t = e / rt, kt = e % rt;
    twt[e] = twiddle<R>(mode_freq(kt, Nt, g.mt), t, Nt, -1);
  }
  for (int e = tid; e < Nz * rz; e += blockDim.x) {
    const int z = e / rz, kz = e % rz;
    twz[e] = twiddle<R>(mode_freq(kz, Nz, g.mz), z, Nz, -1);
  }
  for (int e = tid; e < Ny * kyc; e += blockDim.x) {
    const int y = e / kyc, k = e % kyc;
    twy[e] = (k < kyn) ? twiddle<R>(mode_freq(ky0 + k, Ny, g.my), y, Ny, -1) : cmk<R>(0, 0);
  }

  C<R> acc[ACC];
#pragma unroll
  for (int j = 0; j < ACC; ++j) acc[j] = cmk<R>(0, 0);
  const int nout = kyn * rz * rt;

  const long long plane_elems = (long long)Nz * Nt;
  const long long slab_off = (((long long)bb * g.c + ch) * XL + xl) * (long long)Ny * plane_elems;
  const R* s_slab = src + slab_off;
  const R* p_slab = pre ? pre + slab_off : nullptr;

  for (int y0 = 0; y0 < Ny; y0 += YC) {
    const int yc = min(YC, Ny - y0);
    __syncthreads();
    // stage the plane chunk (contiguous in global memory), input transform fused
    const long long n = (long long)yc * plane_elems;
    const R* s = s_slab + (long long)y0 * plane_elems;
    const R* pp = p_slab ? p_slab + (long long)y0 * plane_elems : nullptr;
    for (long long e = tid; e < n; e += blockDim.x) {
      R v = __ldg(s + e);
      if (src_mode == DFNO_SRC_ACT) v = act_apply<R>(g.act, v);
      else if (src_mode == DFNO_SRC_GRAD) v = v * act_deriv<R>(g.act, __ldg(pp + e));
      plane[e] = v;
    }
    __syncthreads();
    // t stage (real -> complex)
    for (int e = tid; e < yc * Nz * rt; e += blockDim.x) {
      const int row = e / rt, kt = e % rt;
      const R* pr = plane + (long long)row * Nt;
      C<R> u = cmk<R>(0, 0);
      for (int t = 0; t < Nt; ++t) {
        const R a = pr[t];
        const C<R> w = twt[t * rt + kt];
        u.x = fma(a, w.x, u.x);
        u.y = fma(a, w.y, u.y);
      }
      U[e] = u;
    }
    __syncthreads();
    // z stage
    for (int e = tid; e < yc * rz * rt; e += blockDim.x) {
      const int kt = e % rt;
      const int kz = (e / rt) % rz;
      const int y = e / (rt * rz);
      const C<R>* ur = U + (long long)y * Nz * rt + kt;
      C<R> v = cmk<R>(0, 0);
      for (int z = 0; z < Nz; ++z) cmac<R>(v, ur[z * rt], twz[z * rz + kz]);
      V[e] = v;
    }
    __syncthreads();
    // y stage: accumulate into registers
#pragma unroll
    for (int j = 0; j < ACC; ++j) {
      const int o = tid + j * kYztThreads;
      if (o < nout) {
        const int kzt = o % (rz * rt);
        const int k = o / (rz * rt);
        for (int y = 0; y < yc; ++y) cmac<R>(acc[j], V[y * rz * rt + kzt], twy[(y0 + y) * kyc + k]);
      }
    }
  }
  // write into the XK exchange layout
#pragma unroll
  for (int j = 0; j < ACC; ++j) {
    const int o = tid + j * kYztThreads;
    if (o < nout) {
      const int kzt = o % (rz * rt);
      const int k = o / (rz * rt);
      C<R> v = acc[j];
      v.x *= scale;
      v.y *= scale;
      out[xk_row(g, bb, ch, xl, ky0 + k) + kzt] = v;
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(kYztThreads) k_yzt_inv(const dfno_geom g, const C<R>* __restrict__ in, R scale,
                                                         R* __restrict__ out, int YC) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Ny = g.ny, Nz = g.nz, Nt = g.nt, ry = g.ry, rz = g.rz, rt = g.rt;
  const int XL = x_local(g);
  const int slab = blockIdx.x;
  const int xl = slab % XL;
  const int ch = (slab / XL) % g.c;
  const int bb = slab / (XL * g.c);
  const int rzt = rz * rt;

  C<R>* twy = reinterpret_cast<C<R>*>(smem_raw);  // [Ny][ry]  e^{+i}
  C<R>* twz = twy + Ny * ry;                       // [Nz][rz]
  C<R>* twt = twz + Nz * rz;                       // [rt][Nt]
  C<R>* Vs = twt + rt * Nt;                        // [ry][rz][rt]
  C<R>* W1 = Vs + ry * rzt;                        // [YC][rz][rt]
  C<R>* W2 = W1 + YC * rzt;                        // [YC][Nz][rt]

  const int tid = threadIdx.x;
  for (int e = tid; e < Ny * ry; e += blockDim.x) {
    const int y = e / ry, k = e % ry;
    twy[e] = twiddle<R>(mode_freq(k, Ny, g.my), y, Ny, +1);
  }
  for (int e = tid; e < Nz * rz; e += blockDim.x) {
    const int z = e / rz, k = e % rz;
    twz[e] = twiddle<R>(mode_freq(k, Nz, g.mz), z, Nz, +1);
  }
  for (int e = tid; e < rt * Nt; e += blockDim.x) {
    const int k = e / Nt, t = e % Nt;
    twt[e] = twiddle<R>(mode_freq(k, Nt, g.mt), t, Nt, +1);
  }
  for (int e = tid; e < ry * rzt; e += blockDim.x) {
    const int ky = e / rzt, kzt = e % rzt;
    Vs[e] = in[xk_row(g, bb, ch, xl, ky) + kzt];
  }
  const long long plane_elems = (long long)Nz * Nt;
  R* o_slab = out + (((long long)bb * g.c + ch) * XL + xl) * (long long)Ny * plane_elems;

  for (int y0 = 0; y0 < Ny; y0 += YC) {
    const int yc = min(YC, Ny - y0);
    __syncthreads();
    for (int e = tid; e < yc * rzt; e += blockDim.x) {
      const int kzt = e % rzt, y = e / rzt;
      const C<R>* tw = twy + (y0 + y) * ry;
      C<R> a = cmk<R>(0, 0);
      for (int k = 0; k < ry; ++k) cmac<R>(a, Vs[k * rzt + kzt], tw[k]);
      W1[e] = a;
    }
    __syncthreads();
    for (int e = tid; e < yc * Nz * rt; e += blockDim.x) {
      const int kt = e % rt;
      const int z = (e / rt) % Nz;
      const int y = e / (rt * Nz);
      const C<R>* w1 = W1 + y * rzt + kt;
      const C<R>* tw = twz + z * rz;
      C<R> a = cmk<R>(0, 0);
      for (int k = 0; k < rz; ++k) cmac<R>(a, w1[k * rt], tw[k]);
      W2[e] = a;
    }
    __syncthreads();
    const long long n = (long long)yc * plane_elems;
    R* o = o_slab + (long long)y0 * plane_elems;
    for (long long e = tid; e < n; e += blockDim.x) {
      const int t = (int)(e % Nt);
      const long long row = e / Nt;  // (y, z)
      const C<R>* w2 = W2 + row * rt;
      R s = (R)0;
      for (int k = 0; k < rt; ++k) {
        const C<R> a = w2[k];
        const C<R> w = twt[k * Nt + t];
        s = fma(a.x, w.x, s);
        s = fma(-a.y, w.y, s);
      }
      o[e] = s * scale;
    }
  }
}

template <typename R>
static size_t yzt_fwd_smem(const dfno_geom& g, int YC, int kyc) {
  const size_t cplx = (size_t)g.nt * g.rt + (size_t)g.nz * g.rz + (size_t)g.ny * kyc + (size_t)YC * g.nz * g.rt +
                      (size_t)YC * g.rz * g.rt;
  return cplx * 2 * sizeof(R) + (size_t)YC * g.nz * g.nt * sizeof(R);
}

template <typename R>
static size_t yzt_inv_smem(const dfno_geom& g, int YC) {
  const size_t cplx = (size_t)g.ny * g.ry + (size_t)g.nz * g.rz + (size_t)g.rt * g.nt + (size_t)g.ry * g.rz * g.rt +
                      (size_t)YC * g.rz * g.rt + (size_t)YC * g.nz * g.rt;
  return cplx * 2 * sizeof(R);
}

static constexpr size_t kSmemBudget = 200 * 1024;

template <typename R, int ACC>
static int launch_yzt_fwd_acc(const dfno_geom& g, const void* src, const void* pre, int mode, R scale, void* out,
                              int YC, int kyc, size_t smem, cudaStream_t st) {
  auto kern = k_yzt_fwd<R, ACC>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int slabs = g.batch * g.c * x_local(g);
  dim3 grid(slabs, (g.ry + kyc - 1) / kyc);
  kern<<<grid, kYztThreads, smem, st>>>(g, (const R*)src, (const R*)pre, mode, scale, (C<R>*)out, YC, kyc);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

template <typename R>
int yzt_fwd_simt(const dfno_geom& g, const void* src, const void* pre, int mode, double scale, void* out,
                 cudaStream_t st) {
  const int rzt = g.rz * g.rt;
  const int max_out = kYztThreads * kYztAccMax;
  if (rzt > max_out) return DFNO_ERR_UNSUPPORTED;
  int kyc = max_out / rzt;
  if (kyc > g.ry) kyc = g.ry;
  // balance the ky chunks
  const int nchunk = (g.ry + kyc - 1) / kyc;
  kyc = (g.ry + nchunk - 1) / nchunk;
  int YC = 8;
  while (YC > 1 && yzt_fwd_smem<R>(g, YC, kyc) > kSmemBudget) --YC;
  const size_t smem = yzt_fwd_smem<R>(g, YC, kyc);
  if (smem > kSmemBudget) return DFNO_ERR_UNSUPPORTED;
  const int acc = (kyc * rzt + kYztThreads - 1) / kYztThreads;
  const R s = (R)scale;
  if (acc <= 1) return launch_yzt_fwd_acc<R, 1>(g, src, pre, mode, s, out, YC, kyc, smem, st);
  if (acc <= 2) return launch_yzt_fwd_acc<R, 2>(g, src, pre, mode, s, out, YC, kyc, smem, st);
  if (acc <= 4) return launch_yzt_fwd_acc<R, 4>(g, src, pre, mode, s, out, YC, kyc, smem, st);
  if (acc <= 8) return launch_yzt_fwd_acc<R, 8>(g, src, pre, mode, s, out, YC, kyc, smem, st);
  return launch_yzt_fwd_acc<R, 16>(g, src, pre, mode, s, out, YC, kyc, smem, st);
}

template <typename R>
int yzt_inv_simt(const dfno_geom& g, const void* in, double scale, void* out, cudaStream_t st) {
  int YC = 8;
  while (YC > 1 && yzt_inv_smem<R>(g, YC) > kSmemBudget) --YC;
  const size_t smem = yzt_inv_smem<R>(g, YC);
  if (smem > kSmemBudget) return DFNO_ERR_UNSUPPORTED;
  auto kern = k_yzt_inv<R>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int slabs = g.batch * g.c * x_local(g);
  kern<<<slabs, kYztThreads, smem, st>>>(g, (const C<R>*)in, (R)scale, (R*)out, YC);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

template int yzt_fwd_simt<float>(const dfno_geom&, const void*, const void*, int, double, void*, cudaStream_t);
template int yzt_fwd_simt<double>(const dfno_geom&, const void*, const void*, int, double, void*, cudaStream_t);
template int yzt_inv_simt<float>(const dfno_geom&, const void*, double, void*, cudaStream_t);
template int yzt_inv_simt<double>(const dfno_geom&, const void*, double, void*, cudaStream_t);

}  // namespace dfno
