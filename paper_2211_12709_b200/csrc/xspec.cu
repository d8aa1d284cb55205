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

template <typename R, bool BWD, int CM, int BM, int RXM>
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
  C<R>* X = twx + Nx * rx;                         // [b][c][rx][MT]
  C<R>* Y = X + (long long)nb * c * rx * MT;       // [b][c][rx][MT]
  const int tid = threadIdx.x;

  for (int e = tid; e < Nx * rx; e += blockDim.x) {
    const int x = e / rx, k = e % rx;
    twx[e] = twiddle<R>(mode_freq(k, Nx, g.mx), x, Nx, -1);
  }
  __syncthreads();

  // ---- A: forward DFT along x.  A thread owns one (b, i, m) column and
  //      streams all Nx samples (independent loads, gathered straight from the
  //      peer-major KX exchange buffer), accumulating every retained kx.
  for (int e = tid; e < nb * c * MT; e += blockDim.x) {
    const int mm = e % MT, bc = e / MT;
    const int bb = bc / c, i = bc % c;
    if (mm >= mt) continue;
    C<R> acc[RXM];
#pragma unroll
    for (int k = 0; k < RXM; ++k) acc[k] = cmk<R>(0, 0);
    int p = 0, pend = g.x_starts[1];
    long long row = kx_row(g, bb, i, 0) + m0 + mm;
    const long long step = (long long)ky_local(g) * g.rz * g.rt;  // next x inside a peer chunk
#pragma unroll 4
    for (int x = 0; x < Nx; ++x) {
      if (x == pend) {  // next peer chunk
        ++p;
        pend = g.x_starts[p + 1];
        row = kx_row(g, bb, i, x) + m0 + mm;
      }
      const C<R> z = __ldg(kx_in + row);
      row += step;
      const C<R>* tw = twx + x * rx;
#pragma unroll
      for (int k = 0; k < RXM; ++k)
        if (k < rx) cmac<R>(acc[k], z, tw[k]);
    }
#pragma unroll
    for (int k = 0; k < RXM; ++k) {
      if (k < rx) {
        C<R> a = acc[k];
        a.x *= s1;
        a.y *= s1;
        X[((long long)bc * rx + k) * MT + mm] = a;
        if (!BWD && spec) spec[((long long)bc * rx + k) * mloc + m0 + mm] = a;
      }
    }
  }
  __syncthreads();

  // ---- B: per-mode channel contraction (thread owns one (kx, m) column);
  //      accumulators in registers, the CM weights of a row loaded back to back
  for (int e = tid; e < rx * MT; e += blockDim.x) {
    const int kx = e / MT, mm = e % MT;
    if (mm >= mt) continue;
    const long long mg = m0 + mm;
    const C<R>* wcol = w + (long long)kx * mloc + mg;  // + ((i * c + o) * rx) * mloc
    const long long wstride_o = (long long)rx * mloc;
    for (int b0 = 0; b0 < nb; b0 += BM) {
      if (!BWD) {
        C<R> acc[CM][BM];
#pragma unroll
        for (int o = 0; o < CM; ++o)
#pragma unroll
          for (int bb = 0; bb < BM; ++bb) acc[o][bb] = cmk<R>(0, 0);
        for (int i = 0; i < c; ++i) {
          C<R> xv[BM];
#pragma unroll
          for (int bb = 0; bb < BM; ++bb)
            xv[bb] = (b0 + bb < nb) ? X[((long long)((b0 + bb) * c + i) * rx) * MT + e] : cmk<R>(0, 0);
          const C<R>* wr = wcol + (long long)i * c * wstride_o;
          C<R> wv[CM];
#pragma unroll
          for (int o = 0; o < CM; ++o) wv[o] = (o < c) ? __ldg(wr + o * wstride_o) : cmk<R>(0, 0);
#pragma unroll
          for (int o = 0; o < CM; ++o)
#pragma unroll
            for (int bb = 0; bb < BM; ++bb) cmac<R>(acc[o][bb], xv[bb], wv[o]);
        }
#pragma unroll
        for (int o = 0; o < CM; ++o)
#pragma unroll
          for (int bb = 0; bb < BM; ++bb)
            if (o < c && b0 + bb < nb) Y[((long long)((b0 + bb) * c + o) * rx) * MT + e] = acc[o][bb];
      } else {
        // D[b][o] = X (the scaled truncated fft of the upstream gradient)
        C<R> dv[CM][BM];
#pragma unroll
        for (int o = 0; o < CM; ++o)
#pragma unroll
          for (int bb = 0; bb < BM; ++bb)
            dv[o][bb] = (o < c && b0 + bb < nb) ? X[((long long)((b0 + bb) * c + o) * rx) * MT + e] : cmk<R>(0, 0);
        for (int i = 0; i < c; ++i) {
          const C<R>* wr = wcol + (long long)i * c * wstride_o;
          C<R> wv[CM];
#pragma unroll
          for (int o = 0; o < CM; ++o) wv[o] = (o < c) ? __ldg(wr + o * wstride_o) : cmk<R>(0, 0);
          C<R> sv[BM];
#pragma unroll
          for (int bb = 0; bb < BM; ++bb)
            sv[bb] = (b0 + bb < nb) ? __ldg(spec + ((long long)((b0 + bb) * c + i) * rx + kx) * mloc + mg)
                                    : cmk<R>(0, 0);
          // dX[b][i] = sum_o D[b][o] conj(W[i][o])
#pragma unroll
          for (int bb = 0; bb < BM; ++bb) {
            C<R> y = cmk<R>(0, 0);
#pragma unroll
            for (int o = 0; o < CM; ++o) cmac_conj_b<R>(y, dv[o][bb], wv[o]);
            if (b0 + bb < nb) Y[((long long)((b0 + bb) * c + i) * rx) * MT + e] = y;
          }
          // gW[i][o] (+)= sum_b conj(S[b][i]) D[b][o]
          C<R>* gwr = gw + ((long long)i * c * rx + kx) * mloc + mg;
#pragma unroll
          for (int o = 0; o < CM; ++o) {
            if (o < c) {
              C<R> gacc = (b0 > 0) ? gwr[o * wstride_o] : cmk<R>(0, 0);
#pragma unroll
              for (int bb = 0; bb < BM; ++bb) cmac_conj_a<R>(gacc, sv[bb], dv[o][bb]);
              gwr[o * wstride_o] = gacc;
            }
          }
        }
      }
    }
  }
  __syncthreads();

  // ---- C: inverse DFT along x, packed into the KX exchange layout: a thread
  //      owns one (b, o, m) column and writes all Nx outputs.
  for (int e = tid; e < nb * c * MT; e += blockDim.x) {
    const int mm = e % MT, bc = e / MT;
    const int bb = bc / c, o = bc % c;
    if (mm >= mt) continue;
    C<R> yv[RXM];
#pragma unroll
    for (int k = 0; k < RXM; ++k) yv[k] = (k < rx) ? Y[((long long)bc * rx + k) * MT + mm] : cmk<R>(0, 0);
    int p = 0, pend = g.x_starts[1];
    long long row = kx_row(g, bb, o, 0) + m0 + mm;
    const long long step = (long long)ky_local(g) * g.rz * g.rt;
#pragma unroll 4
    for (int x = 0; x < Nx; ++x) {
      if (x == pend) {
        ++p;
        pend = g.x_starts[p + 1];
        row = kx_row(g, bb, o, x) + m0 + mm;
      }
      const C<R>* tw = twx + x * rx;
      C<R> a = cmk<R>(0, 0);
#pragma unroll
      for (int k = 0; k < RXM; ++k)
        if (k < rx) cmac_conj_b<R>(a, yv[k], tw[k]);
      a.x *= s2;
      a.y *= s2;
      kx_out[row] = a;
      row += step;
    }
  }
}

template <typename R>
static size_t xspec_smem(const dfno_geom& g, int MT) {
  const size_t cplx = (size_t)g.nx * g.rx + 2 * (size_t)g.batch * g.c * g.rx * MT;
  return cplx * 2 * sizeof(R);
}

template <typename R, bool BWD, int CM, int BM>
static int launch_xspec_t(const dfno_geom& g, const void* kx_in, const void* w, void* spec, void* gw, void* kx_out,
                          R s1, R s2, int MT, size_t smem, cudaStream_t st) {
  auto kern = g.rx <= 16 ? k_xspec<R, BWD, CM, BM, 16> : k_xspec<R, BWD, CM, BM, 32>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long blocks = (mloc + MT - 1) / MT;
  kern<<<(unsigned)blocks, kXspecThreads, smem, st>>>(g, (const C<R>*)kx_in, (const C<R>*)w, (C<R>*)spec, (C<R>*)gw,
                                                      (C<R>*)kx_out, MT, s1, s2);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
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
  const int c = g.c;
  if (g.rx > 32) return DFNO_ERR_UNSUPPORTED;  // envelope: m_x <= 16
  // register accumulators: CM output channels x BM batch entries per thread
  constexpr int BM = sizeof(R) == 4 ? 2 : 1;
  if (c <= 4) return launch_xspec_t<R, BWD, 4, BM>(g, kx_in, w, spec, gw, kx_out, s1, s2, MT, smem, st);
  if (c <= 8) return launch_xspec_t<R, BWD, 8, BM>(g, kx_in, w, spec, gw, kx_out, s1, s2, MT, smem, st);
  if (c <= 16) return launch_xspec_t<R, BWD, 16, 1>(g, kx_in, w, spec, gw, kx_out, s1, s2, MT, smem, st);
  if (c <= 20) return launch_xspec_t<R, BWD, 20, 1>(g, kx_in, w, spec, gw, kx_out, s1, s2, MT, smem, st);
  if (c <= 32) return launch_xspec_t<R, BWD, 32, 1>(g, kx_in, w, spec, gw, kx_out, s1, s2, MT, smem, st);
  return DFNO_ERR_UNSUPPORTED;
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
