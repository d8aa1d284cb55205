// x-spectral stage on one rank's ky pencil: truncated DFT along x over the
// full Nx, the per-mode complex channel contraction with the spectral weight
// shard, and the inverse DFT back to x -- fused in one kernel so the
// truncated spectrum never leaves shared memory.
//
// Forward replaces fft_dims(x) + truncate(kx) + einsum_spectral + pad(kx) +
// ifft_dims(kx)  (reference d/fno.py:331-336, d/tensor.py:231-255).
// Backward replaces the adjoint chain d/fno.py:450-457 with
// _spectral_weight_grad / _spectral_input_grad (d/fno.py:415-423).
//
// One CTA owns MT consecutive local modes m = (ky_local, kz, kt) (the
// innermost, contiguous index of every operand, so all global accesses are
// MT-wide contiguous runs) and all (b, c, kx) for them:
//   A  X[b][i][kx][m] = s1 * sum_x Z[b][i][x][m] e^{-2 pi i kx x / Nx}   (Z gathered
//      straight from the peer-major KX exchange buffer -- unpack fused)
//   B  fwd: Y[b][o][kx][m] = sum_i X[b][i][kx][m] W[i][o][kx][m]     (+ spec cache)
//      bwd: gW[i][o][kx][m] = sum_b conj(S[b][i][kx][m]) X[b][o][kx][m]
//           Y[b][i][kx][m]  = sum_o X[b][o][kx][m] conj(W[i][o][kx][m])
//   C  U[b][o][x][m] = s2 * sum_kx Y[b][o][kx][m] e^{+2 pi i kx x / Nx}  written
//      straight into the peer-major KX layout (pack fused)
// Truncation / zero padding along kx are implicit: only retained kx rows of
// the twiddle table exist.  The op is bound by the weight stream (8 c^2 R B per
// block), so SIMT FMA is sufficient here.
#include "common.cuh"

namespace dfno {

constexpr int kXspecThreads = 256;

template <typename R, bool BWD>
__global__ void __launch_bounds__(kXspecThreads) k_xspec(const dfno_geom g, const C<R>* __restrict__ kx_in,
                                                         const C<R>* __restrict__ w, C<R>* __restrict__ spec,
                                                         C<R>* __restrict__ gw, C<R>* __restrict__ kx_out, int MT,
                                                         R s1, R s2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Nx = g.nx, rx = g.rx, c = g.c, nb = g.batch;
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long m0 = (long long)blockIdx.x * MT;
  const int mt = (int)min((long long)MT, mloc - m0);

  C<R>* twx = reinterpret_cast<C<R>*>(smem_raw);  // [Nx][rx] e^{-i}
  C<R>* Z = twx + Nx * rx;                         // [Nx][MT]
  C<R>* X = Z + Nx * MT;                           // [b][c][rx][MT]
  C<R>* Y = X + (long long)nb * c * rx * MT;       // [b][c][rx][MT]
  const int tid = threadIdx.x;

  for (int e = tid; e < Nx * rx; e += blockDim.x) {
    const int x = e / rx, k = e % rx;
    twx[e] = twiddle<R>(mode_freq(k, Nx, g.mx), x, Nx, -1);
  }
  for (long long e = tid; e < (long long)nb * c * rx * MT; e += blockDim.x) Y[e] = cmk<R>(0, 0);

  // ---- A: forward DFT along x, one (b, i) channel column at a time
  for (int bc = 0; bc < nb * c; ++bc) {
    const int bb = bc / c, i = bc % c;
    __syncthreads();
    for (int e = tid; e < Nx * MT; e += blockDim.x) {
      const int x = e / MT, mm = e % MT;
      Z[e] = (mm < mt) ? kx_in[kx_row(g, bb, i, x) + m0 + mm] : cmk<R>(0, 0);
    }
    __syncthreads();
    for (int e = tid; e < rx * MT; e += blockDim.x) {
      const int kx = e / MT, mm = e % MT;
      C<R> a = cmk<R>(0, 0);
      for (int x = 0; x < Nx; ++x) cmac<R>(a, Z[x * MT + mm], twx[x * rx + kx]);
      a.x *= s1;
      a.y *= s1;
      X[(long long)bc * rx * MT + e] = a;
      if (!BWD && spec && mm < mt) spec[((long long)bc * rx + kx) * mloc + m0 + mm] = a;
    }
  }
  __syncthreads();

  // ---- B: per-mode channel contraction (thread owns one (kx, m) column)
  for (int e = tid; e < rx * MT; e += blockDim.x) {
    const int kx = e / MT, mm = e % MT;
    if (mm >= mt) continue;
    const long long mg = m0 + mm;
    if (!BWD) {
      for (int i = 0; i < c; ++i) {
        for (int o = 0; o < c; ++o) {
          const C<R> wv = __ldg(w + (((long long)i * c + o) * rx + kx) * mloc + mg);
          for (int bb = 0; bb < nb; ++bb)
            cmac<R>(Y[((long long)(bb * c + o) * rx) * MT + e], X[((long long)(bb * c + i) * rx) * MT + e], wv);
        }
      }
    } else {
      for (int i = 0; i < c; ++i) {
        for (int o = 0; o < c; ++o) {
          const C<R> wv = __ldg(w + (((long long)i * c + o) * rx + kx) * mloc + mg);
          C<R> gacc = cmk<R>(0, 0);
          for (int bb = 0; bb < nb; ++bb) {
            const C<R> d = X[((long long)(bb * c + o) * rx) * MT + e];
            const C<R> s = __ldg(spec + (((long long)(bb * c + i)) * rx + kx) * mloc + mg);
            cmac_conj_a<R>(gacc, s, d);
            cmac_conj_b<R>(Y[((long long)(bb * c + i) * rx) * MT + e], d, wv);
          }
          gw[(((long long)i * c + o) * rx + kx) * mloc + mg] = gacc;
        }
      }
    }
  }
  __syncthreads();

  // ---- C: inverse DFT along x, pack into the KX exchange layout
  for (int bc = 0; bc < nb * c; ++bc) {
    const int bb = bc / c, o = bc % c;
    const C<R>* yr = Y + (long long)bc * rx * MT;
    for (int e = tid; e < Nx * MT; e += blockDim.x) {
      const int x = e / MT, mm = e % MT;
      if (mm >= mt) continue;
      const C<R>* tw = twx + x * rx;
      C<R> a = cmk<R>(0, 0);
      for (int k = 0; k < rx; ++k) cmac_conj_b<R>(a, yr[k * MT + mm], tw[k]);
      a.x *= s2;
      a.y *= s2;
      kx_out[kx_row(g, bb, o, x) + m0 + mm] = a;
    }
  }
}

template <typename R>
static size_t xspec_smem(const dfno_geom& g, int MT) {
  const size_t cplx = (size_t)g.nx * g.rx + (size_t)g.nx * MT + 2 * (size_t)g.batch * g.c * g.rx * MT;
  return cplx * 2 * sizeof(R);
}

template <typename R, bool BWD>
static int launch_xspec(const dfno_geom& g, const void* kx_in, const void* w, void* spec, void* gw, void* kx_out,
                        R s1, R s2, cudaStream_t st) {
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t budget = 200 * 1024;
  int MT = 32;
  while (MT > 1 && (xspec_smem<R>(g, MT) > budget || ((mloc + MT - 1) / MT < 2LL * sms && MT > 4))) MT /= 2;
  const size_t smem = xspec_smem<R>(g, MT);
  if (smem > budget) return DFNO_ERR_UNSUPPORTED;
  auto kern = k_xspec<R, BWD>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const long long blocks = (mloc + MT - 1) / MT;
  kern<<<(unsigned)blocks, kXspecThreads, smem, st>>>(g, (const C<R>*)kx_in, (const C<R>*)w, (C<R>*)spec,
                                                      (C<R>*)gw, (C<R>*)kx_out, MT, s1, s2);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

template <typename R>
int xspec_fwd_simt(const dfno_geom& g, const void* kx_in, const void* w, void* spec, void* kx_out, cudaStream_t st) {
  // forward: fft_x unnormalised, ifft_x carries 1/Nx (d/spectral.py:1-9)
  return launch_xspec<R, false>(g, kx_in, w, spec, nullptr, kx_out, (R)1, (R)(1.0 / g.nx), st);
}

template <typename R>
int xspec_bwd_simt(const dfno_geom& g, const void* kx_in, const void* spec, const void* w, void* gw, void* kx_out,
                   cudaStream_t st) {
  // backward: fft_x / Nx, then ifft_x * Nx = unnormalised inverse (d/fno.py:450-457)
  return launch_xspec<R, true>(g, kx_in, w, const_cast<void*>(spec), gw, kx_out, (R)(1.0 / g.nx), (R)1, st);
}

template int xspec_fwd_simt<float>(const dfno_geom&, const void*, const void*, void*, void*, cudaStream_t);
template int xspec_fwd_simt<double>(const dfno_geom&, const void*, const void*, void*, void*, cudaStream_t);
template int xspec_bwd_simt<float>(const dfno_geom&, const void*, const void*, const void*, void*, void*,
                                   cudaStream_t);
template int xspec_bwd_simt<double>(const dfno_geom&, const void*, const void*, const void*, void*, void*,
                                    cudaStream_t);

}  // namespace dfno
