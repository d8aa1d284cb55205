// x-spectral stage as three bandwidth-shaped kernels (fp32), the path used
// when the caller supplies a workspace (dfno_xspec_fwd_ws / _bwd_ws):
//
//   k_xdft    X[b][c][kx][m] = s1 * sum_x Z[b][c][x][m] e^{-2 pi i kx x/Nx}
//             (Z gathered straight from the peer-major KX exchange buffer:
//             unpack fused; truncation implicit -- only retained kx rows of
//             the twiddle table exist)                     d/fno.py:331-332
//   k_xmix    forward  Y[b][o][kx][m] = sum_i X[b][i][kx][m] W[i][o][kx][m]
//             (d/tensor.py:231-255): a batched small GEMM per (kx, m), bound
//             by the weight stream (8 flop per 8 B at b = 1), so each thread
//             owns one (o group, kx, m) column: every W load is a coalesced
//             256-byte warp transaction and every W byte is read once.
//   k_xmix_bwd gW[i][o][kx][m] = sum_b conj(S[b][i]) D[b][o]
//             dX[b][i][kx][m]  = sum_o D[b][o] conj(W[i][o])  (d/fno.py:415-423)
//   k_xidft   U[b][c][x][m] = s2 * sum_kx Y[b][c][kx][m] e^{+2 pi i kx x/Nx}
//             written straight into the KX layout (pack fused; zero padding
//             of the missing kx implicit)                  d/fno.py:335-336
//
// Compared with the fused one-CTA-per-mode-block kernel (xspec.cu) this
// streams the weights with full occupancy and no block-wide phases; the
// extra traffic is the 2 x b c r_x (ky) r_z r_t spectrum round trip
// (21 MB at C2 against 210 MB of weights).
#include <stdlib.h>

#include "common.cuh"

namespace dfno {

int xdft_tc(const dfno_geom&, const void*, float, void*, cudaStream_t);
int xidft_tc(const dfno_geom&, const void*, float, void*, cudaStream_t);

namespace {
constexpr int kXT = 256;  // threads per block
constexpr int kOG = 4;    // output channels per thread in k_xmix / input channels in k_xmix_bwd
constexpr int kBMax = 4;  // batch entries held in registers by k_xmix_bwd

__device__ __forceinline__ long long mloc_of(const dfno_geom& g) { return (long long)ky_local(g) * g.rz * g.rt; }

// twiddle table tw[x][kx] = e^{-2 pi i f(kx) x / Nx} in shared memory
__device__ void fill_tw(float2* tw, const dfno_geom& g) {
  for (int e = threadIdx.x; e < g.nx * g.rx; e += blockDim.x) {
    const int x = e / g.rx, k = e % g.rx;
    tw[e] = twiddle<float>(mode_freq(k, g.nx, g.mx), x, g.nx, -1);
  }
  __syncthreads();
}
}  // namespace

// one thread per (b, c, m) column and kx share: KS threads split the r_x
// outputs of a column (RXM each) for parallelism; the shared Z loads hit L1.
template <int RXM, int KS>
__global__ void __launch_bounds__(kXT) k_xdft(const dfno_geom g, const float2* __restrict__ kx_in, float s1,
                                              float2* __restrict__ X) {
  extern __shared__ float2 tw[];
  fill_tw(tw, g);
  const long long mloc = mloc_of(g);
  const long long n = (long long)g.batch * g.c * mloc * KS;
  const int rx = g.rx;
  for (long long e = (long long)blockIdx.x * kXT + threadIdx.x; e < n; e += (long long)gridDim.x * kXT) {
    const long long m = e % mloc, q = e / mloc;
    const int h = (int)(q % KS);
    const long long bc = q / KS;
    const int c = (int)(bc % g.c), bb = (int)(bc / g.c);
    const int k0 = h * RXM;
    float2 acc[RXM];
#pragma unroll
    for (int k = 0; k < RXM; ++k) acc[k] = make_float2(0.f, 0.f);
    for (int p = 0; p < g.nranks; ++p) {  // peer chunks of the KX layout (d/partition.py:135-188)
      const int x0 = g.x_starts[p], x1 = g.x_starts[p + 1];
      const float2* src = kx_in + kx_row(g, bb, c, x0) + m;
#pragma unroll 4
      for (int x = x0; x < x1; ++x) {
        const float2 z = __ldg(src);
        src += mloc;
        const float2* t = tw + x * rx + k0;
#pragma unroll
        for (int k = 0; k < RXM; ++k)
          if (k0 + k < rx) cmac<float>(acc[k], z, t[k]);
      }
    }
    float2* dst = X + (bc * rx + k0) * mloc + m;
#pragma unroll
    for (int k = 0; k < RXM; ++k)
      if (k0 + k < rx) dst[(long long)k * mloc] = make_float2(s1 * acc[k].x, s1 * acc[k].y);
  }
}

// one thread per (b, c, m) column and x share: XS threads split the Nx
// outputs of a column for parallelism.
template <int RXM, int XS>
__global__ void __launch_bounds__(kXT) k_xidft(const dfno_geom g, const float2* __restrict__ Y, float s2,
                                               float2* __restrict__ kx_out) {
  extern __shared__ float2 tw[];
  fill_tw(tw, g);
  const long long mloc = mloc_of(g);
  const long long n = (long long)g.batch * g.c * mloc * XS;
  const int rx = g.rx, Nx = g.nx;
  for (long long e = (long long)blockIdx.x * kXT + threadIdx.x; e < n; e += (long long)gridDim.x * kXT) {
    const long long m = e % mloc, q = e / mloc;
    const int h = (int)(q % XS);
    const long long bc = q / XS;
    const int c = (int)(bc % g.c), bb = (int)(bc / g.c);
    float2 yv[RXM];
    const float2* src = Y + (bc * rx) * mloc + m;
#pragma unroll
    for (int k = 0; k < RXM; ++k) yv[k] = (k < rx) ? src[(long long)k * mloc] : make_float2(0.f, 0.f);
    const int xa = (int)(((long long)Nx * h) / XS), xb = (int)(((long long)Nx * (h + 1)) / XS);
    int p = 0;
    while (xa >= g.x_starts[p + 1]) ++p;
    float2* dst = kx_out + kx_row(g, bb, c, xa) + m;
#pragma unroll 2
    for (int x = xa; x < xb; ++x) {
      if (x == g.x_starts[p + 1]) {  // next peer chunk of the KX layout
        ++p;
        dst = kx_out + kx_row(g, bb, c, x) + m;
      }
      const float2* t = tw + x * rx;
      float2 a = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < RXM; ++k)
        if (k < rx) cmac_conj_b<float>(a, yv[k], t[k]);  // e^{+i} = conj(e^{-i})
      __stcs(dst, make_float2(s2 * a.x, s2 * a.y));
      dst += mloc;
    }
  }
}

// forward contraction: one thread per (o group, kx, m), all batch entries
__global__ void __launch_bounds__(kXT) k_xmix(const dfno_geom g, const float2* __restrict__ X,
                                              const float2* __restrict__ W, float2* __restrict__ Y) {
  const long long mloc = mloc_of(g);
  const int rx = g.rx, C = g.c, nog = (C + kOG - 1) / kOG;
  const long long cols = (long long)rx * mloc;  // (kx, m)
  const long long n = (long long)nog * cols;
  const long long wo = cols;                    // W stride between consecutive o
  for (long long e = (long long)blockIdx.x * kXT + threadIdx.x; e < n; e += (long long)gridDim.x * kXT) {
    const long long col = e % cols;
    const int o0 = (int)(e / cols) * kOG;
    for (int bb = 0; bb < g.batch; ++bb) {
      float2 acc[kOG];
#pragma unroll
      for (int j = 0; j < kOG; ++j) acc[j] = make_float2(0.f, 0.f);
      const float2* xp = X + ((long long)bb * C) * cols + col;
      const float2* wp = W + ((long long)o0) * wo + col;
#pragma unroll 2
      for (int i = 0; i < C; ++i) {
        const float2 xv = xp[(long long)i * cols];
        const float2* wr = wp + (long long)i * C * wo;
        float2 wv[kOG];
#pragma unroll
        for (int j = 0; j < kOG; ++j) wv[j] = (o0 + j < C) ? __ldcs(wr + j * wo) : make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < kOG; ++j) cmac<float>(acc[j], xv, wv[j]);
      }
      float2* yp = Y + ((long long)bb * C + o0) * cols + col;
#pragma unroll
      for (int j = 0; j < kOG; ++j)
        if (o0 + j < C) yp[j * cols] = acc[j];
    }
  }
}

// backward contraction: one thread per (i group, kx, m); batch <= BM <= kBMax
template <int BM>
__global__ void __launch_bounds__(kXT) k_xmix_bwd(const dfno_geom g, const float2* __restrict__ S,
                                                  const float2* __restrict__ D, const float2* __restrict__ W,
                                                  float2* __restrict__ gW, float2* __restrict__ dX) {
  const long long mloc = mloc_of(g);
  const int rx = g.rx, C = g.c, nig = (C + kOG - 1) / kOG, B = g.batch;
  const long long cols = (long long)rx * mloc;
  const long long n = (long long)nig * cols;
  for (long long e = (long long)blockIdx.x * kXT + threadIdx.x; e < n; e += (long long)gridDim.x * kXT) {
    const long long col = e % cols;
    const int i0 = (int)(e / cols) * kOG;
    float2 sv[BM][kOG], dx[BM][kOG];
#pragma unroll
    for (int bb = 0; bb < BM; ++bb)
#pragma unroll
      for (int j = 0; j < kOG; ++j) {
        sv[bb][j] = (bb < B && i0 + j < C) ? S[((long long)bb * C + i0 + j) * cols + col] : make_float2(0.f, 0.f);
        dx[bb][j] = make_float2(0.f, 0.f);
      }
#pragma unroll 2
    for (int o = 0; o < C; ++o) {
      float2 dv[BM];
#pragma unroll
      for (int bb = 0; bb < BM; ++bb) dv[bb] = (bb < B) ? D[((long long)bb * C + o) * cols + col] : make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < kOG; ++j) {
        if (i0 + j >= C) continue;
        const long long wi = ((long long)(i0 + j) * C + o) * cols + col;
        const float2 wv = __ldcs(W + wi);
        float2 gacc = make_float2(0.f, 0.f);
#pragma unroll
        for (int bb = 0; bb < BM; ++bb) {
          cmac_conj_a<float>(gacc, sv[bb][j], dv[bb]);   // conj(S) D
          cmac_conj_b<float>(dx[bb][j], dv[bb], wv);     // D conj(W)
        }
        __stcs(gW + wi, gacc);
      }
    }
#pragma unroll
    for (int bb = 0; bb < BM; ++bb)
#pragma unroll
      for (int j = 0; j < kOG; ++j)
        if (bb < B && i0 + j < C) dX[((long long)bb * C + i0 + j) * cols + col] = dx[bb][j];
  }
}

// Two (kx, m) columns per thread (16-byte loads and stores): the contractions
// are weight-stream bound and latency-limited at the occupancy their register
// blocking allows, so doubling the bytes per request doubles the bytes in
// flight.  Requires an even column count (r_x * modes).
__device__ __forceinline__ void cmac2(float4& acc, const float4& a, const float4& b) {
  acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y); acc.y = fmaf(a.y, b.x, acc.y);
  acc.z = fmaf(a.z, b.z, acc.z); acc.z = fmaf(-a.w, b.w, acc.z);
  acc.w = fmaf(a.z, b.w, acc.w); acc.w = fmaf(a.w, b.z, acc.w);
}
__device__ __forceinline__ void cmac2_conj_a(float4& acc, const float4& a, const float4& b) {  // conj(a) b
  acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y); acc.y = fmaf(-a.y, b.x, acc.y);
  acc.z = fmaf(a.z, b.z, acc.z); acc.z = fmaf(a.w, b.w, acc.z);
  acc.w = fmaf(a.z, b.w, acc.w); acc.w = fmaf(-a.w, b.z, acc.w);
}
__device__ __forceinline__ void cmac2_conj_b(float4& acc, const float4& a, const float4& b) {  // a conj(b)
  acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.y, b.x, acc.y); acc.y = fmaf(-a.x, b.y, acc.y);
  acc.z = fmaf(a.z, b.z, acc.z); acc.z = fmaf(a.w, b.w, acc.z);
  acc.w = fmaf(a.w, b.z, acc.w); acc.w = fmaf(-a.z, b.w, acc.w);
}

template <int OG>
__global__ void __launch_bounds__(kXT) k_xmix2(const dfno_geom g, const float4* __restrict__ X,
                                               const float4* __restrict__ W, float4* __restrict__ Y) {
  const long long mloc = mloc_of(g);
  const int C = g.c, nog = (C + OG - 1) / OG;
  const long long cols = (long long)g.rx * mloc / 2;  // column pairs
  const long long n = (long long)nog * cols;
  for (long long e = (long long)blockIdx.x * kXT + threadIdx.x; e < n; e += (long long)gridDim.x * kXT) {
    const long long col = e % cols;
    const int o0 = (int)(e / cols) * OG;
    for (int bb = 0; bb < g.batch; ++bb) {
      float4 acc[OG];
#pragma unroll
      for (int j = 0; j < OG; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4* xp = X + ((long long)bb * C) * cols + col;
#pragma unroll 2
      for (int i = 0; i < C; ++i) {
        const float4 xv = xp[(long long)i * cols];
        const float4* wr = W + ((long long)i * C + o0) * cols + col;
#pragma unroll
        for (int j = 0; j < OG; ++j) {
          const float4 wv = (o0 + j < C) ? __ldcs(wr + j * cols) : make_float4(0.f, 0.f, 0.f, 0.f);
          cmac2(acc[j], xv, wv);
        }
      }
      float4* yp = Y + ((long long)bb * C + o0) * cols + col;
#pragma unroll
      for (int j = 0; j < OG; ++j)
        if (o0 + j < C) yp[j * cols] = acc[j];
    }
  }
}

template <int BM, int OG>
__global__ void __launch_bounds__(kXT) k_xmix_bwd2(const dfno_geom g, const float4* __restrict__ S,
                                                   const float4* __restrict__ D, const float4* __restrict__ W,
                                                   float4* __restrict__ gW, float4* __restrict__ dX) {
  const long long mloc = mloc_of(g);
  const int C = g.c, nig = (C + OG - 1) / OG, B = g.batch;
  const long long cols = (long long)g.rx * mloc / 2;
  const long long n = (long long)nig * cols;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long e = (long long)blockIdx.x * kXT + threadIdx.x; e < n; e += (long long)gridDim.x * kXT) {
    const long long col = e % cols;
    const int i0 = (int)(e / cols) * OG;
    float4 sv[BM][OG], dx[BM][OG];
#pragma unroll
    for (int bb = 0; bb < BM; ++bb)
#pragma unroll
      for (int j = 0; j < OG; ++j) {
        sv[bb][j] = (bb < B && i0 + j < C) ? S[((long long)bb * C + i0 + j) * cols + col] : z4;
        dx[bb][j] = z4;
      }
#pragma unroll 2
    for (int o = 0; o < C; ++o) {
      float4 dv[BM];
#pragma unroll
      for (int bb = 0; bb < BM; ++bb) dv[bb] = (bb < B) ? D[((long long)bb * C + o) * cols + col] : z4;
#pragma unroll
      for (int j = 0; j < OG; ++j) {
        if (i0 + j >= C) continue;
        const long long wi = ((long long)(i0 + j) * C + o) * cols + col;
        const float4 wv = __ldcs(W + wi);
        float4 gacc = z4;
#pragma unroll
        for (int bb = 0; bb < BM; ++bb) {
          cmac2_conj_a(gacc, sv[bb][j], dv[bb]);  // conj(S) D
          cmac2_conj_b(dx[bb][j], dv[bb], wv);    // D conj(W)
        }
        __stcs(gW + wi, gacc);
      }
    }
#pragma unroll
    for (int bb = 0; bb < BM; ++bb)
#pragma unroll
      for (int j = 0; j < OG; ++j)
        if (bb < B && i0 + j < C) dX[((long long)bb * C + i0 + j) * cols + col] = dx[bb][j];
  }
}


namespace {
int sms_x() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ---------------------------------------------------------------------------
// Register-blocked x-DFTs (SIMT, any N_x, r_x <= 16).  Both are small complex
// GEMMs (16 x N_x by N_x x modes) that the FFMA issue rate bounds, so each
// thread owns two modes (m, m + 32: coalesced across the warp) and eight kx
// (forward) or all sixteen kx (inverse): every twiddle read from shared memory
// (broadcast float4 = 2 twiddles) feeds 8 complex MACs, every data load 8 or
// 16.  A block covers 256 / XS modes of one (b, c); when the modes per rank are
// few (P = 8 ky pencils: 2 x 16 x 16) the x range is split XS ways across the
// block's warps (forward: partial sums reduced through shared memory) so the
// grid still fills the GPU.  Twiddles are fp32 sincospif (<= 1 ulp) with the
// exact integer phase reduction.
constexpr int kXB = 256;  // threads per block

__device__ __forceinline__ void fill_tw16(float2* tw, long long* rows, const dfno_geom& g, int bb, int c) {
  for (int e = threadIdx.x; e < g.nx * 16; e += blockDim.x) {
    const int x = e >> 4, k = e & 15;
    float sn = 0.f, cs = 0.f;
    if (k < g.rx) {
      const long long f = mode_freq(k, g.nx, g.mx);
      const long long idx = ((f % g.nx + g.nx) % g.nx) * x % g.nx;
      sincospif(2.0f * (float)idx / (float)g.nx, &sn, &cs);
    }
    tw[e] = make_float2(cs, -sn);  // e^{-2 pi i f x / Nx}
  }
  for (int x = threadIdx.x; x < g.nx; x += blockDim.x) rows[x] = kx_row(g, bb, c, x);
}

// warps: kh = w & 1 (kx half), q = w >> 1 = (x part xs, mode group mg)
template <int XS>
__global__ void __launch_bounds__(kXB) k_xdft_s(const dfno_geom g, const float2* __restrict__ kx_in, float s1,
                                                float2* __restrict__ X) {
  constexpr int MG = 4 / XS, kM = 64 * MG;
  extern __shared__ __align__(16) unsigned char xs_raw[];
  const int Nx = g.nx;
  float2* tw = reinterpret_cast<float2*>(xs_raw);  // [Nx][16]
  long long* rows = reinterpret_cast<long long*>(tw + Nx * 16);
  const long long mloc = mloc_of(g);
  const long long mtiles = (mloc + kM - 1) / kM;
  const long long bc = blockIdx.x / mtiles, m0 = (blockIdx.x - bc * mtiles) * kM;
  const int c = (int)(bc % g.c), bb = (int)(bc / g.c);
  fill_tw16(tw, rows, g, bb, c);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, kh = w & 1, q = w >> 1;
  const int mg = q % MG, xs = q / MG;
  const long long ma = m0 + mg * 64 + lane, mb = ma + 32;
  const bool oka = ma < mloc, okb = mb < mloc;
  const int xlo = (int)((long long)Nx * xs / XS), xhi = (int)((long long)Nx * (xs + 1) / XS);
  float2 acc[2][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[0][j] = acc[1][j] = make_float2(0.f, 0.f);
  const float4* t4 = reinterpret_cast<const float4*>(tw) + 4 * kh;
  // loads run four x ahead of the MACs (register double buffer)
  constexpr int kPf = 4;
  float2 za[kPf], zb[kPf];
  auto fetch = [&](int x0) {
#pragma unroll
    for (int u = 0; u < kPf; ++u) {
      const int x = x0 + u;
      const float2* src = kx_in + rows[x < xhi ? x : xlo];
      za[u] = (oka && x < xhi) ? __ldcs(src + ma) : make_float2(0.f, 0.f);
      zb[u] = (okb && x < xhi) ? __ldcs(src + mb) : make_float2(0.f, 0.f);
    }
  };
  fetch(xlo);
#pragma unroll 1
  for (int x0 = xlo; x0 < xhi; x0 += kPf) {
    float2 ca[kPf], cb[kPf];
#pragma unroll
    for (int u = 0; u < kPf; ++u) {
      ca[u] = za[u];
      cb[u] = zb[u];
    }
    fetch(x0 + kPf);
#pragma unroll
    for (int u = 0; u < kPf; ++u) {
      const int x = min(x0 + u, xhi - 1);  // x >= xhi carries zero data
#pragma unroll
      for (int j2 = 0; j2 < 4; ++j2) {
        const float4 t = t4[x * 8 + j2];
        const float2 t0 = make_float2(t.x, t.y), t1 = make_float2(t.z, t.w);
        cmac<float>(acc[0][2 * j2], ca[u], t0);
        cmac<float>(acc[0][2 * j2 + 1], ca[u], t1);
        cmac<float>(acc[1][2 * j2], cb[u], t0);
        cmac<float>(acc[1][2 * j2 + 1], cb[u], t1);
      }
    }
  }
  if constexpr (XS > 1) {
    // partial sums of x parts 1.. -> shared (aliases the twiddles), x part 0 adds them in order
    __syncthreads();
    float2* red = tw;  // [xs - 1][kh][mg][j][half][lane]
    if (xs > 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float2* r = red + ((((xs - 1) * 2 + kh) * MG + mg) * 8 + j) * 64 + lane;
        r[0] = acc[0][j];
        r[32] = acc[1][j];
      }
    }
    __syncthreads();
    if (xs > 0) return;
#pragma unroll
    for (int p = 1; p < XS; ++p)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2* r = red + ((((p - 1) * 2 + kh) * MG + mg) * 8 + j) * 64 + lane;
        acc[0][j].x += r[0].x;
        acc[0][j].y += r[0].y;
        acc[1][j].x += r[32].x;
        acc[1][j].y += r[32].y;
      }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int kx = 8 * kh + j;
    if (kx < g.rx) {
      float2* dst = X + (bc * g.rx + kx) * mloc;
      if (oka) dst[ma] = make_float2(s1 * acc[0][j].x, s1 * acc[0][j].y);
      if (okb) dst[mb] = make_float2(s1 * acc[1][j].x, s1 * acc[1][j].y);
    }
  }
}

// warps: xt = w % (2 XS) (x part), mg = w / (2 XS) (mode group)
template <int XS>
__global__ void __launch_bounds__(kXB) k_xidft_s(const dfno_geom g, const float2* __restrict__ Y, float s2,
                                                 float2* __restrict__ kx_out) {
  constexpr int MG = 4 / XS, XT = 2 * XS, kM = 64 * MG;
  extern __shared__ __align__(16) unsigned char xs_raw[];
  const int Nx = g.nx;
  float2* tw = reinterpret_cast<float2*>(xs_raw);  // [Nx][16]
  long long* rows = reinterpret_cast<long long*>(tw + Nx * 16);
  const long long mloc = mloc_of(g);
  const long long mtiles = (mloc + kM - 1) / kM;
  const long long bc = blockIdx.x / mtiles, m0 = (blockIdx.x - bc * mtiles) * kM;
  const int c = (int)(bc % g.c), bb = (int)(bc / g.c);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, xt = w % XT, mg = w / XT;
  const long long ma = m0 + mg * 64 + lane, mb = ma + 32;
  const bool oka = ma < mloc, okb = mb < mloc;
  float2 ya[16], yb[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const float2* src = Y + (bc * g.rx + k) * mloc;
    ya[k] = (oka && k < g.rx) ? __ldg(src + ma) : make_float2(0.f, 0.f);
    yb[k] = (okb && k < g.rx) ? __ldg(src + mb) : make_float2(0.f, 0.f);
  }
  fill_tw16(tw, rows, g, bb, c);
  __syncthreads();
  const float4* t4 = reinterpret_cast<const float4*>(tw);
  const int xa = (int)((long long)Nx * xt / XT), xb = (int)((long long)Nx * (xt + 1) / XT);
#pragma unroll 2
  for (int x = xa; x < xb; ++x) {
    float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) {
      const float4 t = t4[x * 8 + k2];
      const float2 t0 = make_float2(t.x, t.y), t1 = make_float2(t.z, t.w);
      cmac_conj_b<float>(a, ya[2 * k2], t0);  // e^{+i} = conj(e^{-i})
      cmac_conj_b<float>(a, ya[2 * k2 + 1], t1);
      cmac_conj_b<float>(b, yb[2 * k2], t0);
      cmac_conj_b<float>(b, yb[2 * k2 + 1], t1);
    }
    float2* dst = kx_out + rows[x];
    if (oka) __stcs(dst + ma, make_float2(s2 * a.x, s2 * a.y));
    if (okb) __stcs(dst + mb, make_float2(s2 * b.x, s2 * b.y));
  }
}

bool tiled_ok(const dfno_geom& g) {
  return g.dtype == DFNO_F32 && g.rx <= 16 && (size_t)g.nx * (16 * sizeof(float2) + sizeof(long long)) <= 200 * 1024;
}

unsigned grid_for(long long n, int per_sm = 8) {
  long long b = (n + kXT - 1) / kXT;
  const long long cap = (long long)sms_x() * per_sm;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

// x split: the smallest XS whose grid (b c ceil(modes / (256 / XS)) blocks)
// covers two blocks per SM
int x_split(const dfno_geom& g) {
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt, bc = (long long)g.batch * g.c;
  for (int xs = 1; xs < 4; xs *= 2)
    if (bc * ((mloc + 256 / xs - 1) / (256 / xs)) >= 2LL * sms_x()) return xs;
  return 4;
}

template <typename K>
int launch_tiled(K kern, const dfno_geom& g, int xs, const void* in, float s, void* out, cudaStream_t st) {
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long blocks = (long long)g.batch * g.c * ((mloc + 256 / xs - 1) / (256 / xs));
  size_t smem = (size_t)g.nx * (16 * sizeof(float2) + sizeof(long long));
  if (smem < 32 * 1024) smem = 32 * 1024;  // the forward's x-split reduction aliases the twiddles
  if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  kern<<<(unsigned)blocks, kXB, smem, st>>>(g, (const float2*)in, s, (float2*)out);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

int launch_dft(const dfno_geom& g, const void* kx_in, float s1, void* X, cudaStream_t st) {
  const int rt = xdft_tc(g, kx_in, s1, X, st);  // tcgen05 (xdft_tc.cu); SIMT outside its envelope
  if (rt != DFNO_ERR_UNSUPPORTED) return rt;
  if (tiled_ok(g)) {
    const int xs = x_split(g);
    const int rc = xs == 1 ? launch_tiled(k_xdft_s<1>, g, 1, kx_in, s1, X, st)
                   : xs == 2 ? launch_tiled(k_xdft_s<2>, g, 2, kx_in, s1, X, st)
                             : launch_tiled(k_xdft_s<4>, g, 4, kx_in, s1, X, st);
    if (rc != DFNO_ERR_UNSUPPORTED) return rc;
  }
  const size_t smem = (size_t)g.nx * g.rx * sizeof(float2);
  const long long n = (long long)g.batch * g.c * (long long)ky_local(g) * g.rz * g.rt * 2;
  auto k = g.rx <= 16 ? k_xdft<8, 2> : k_xdft<16, 2>;
  if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  k<<<grid_for(n, 4), kXT, smem, st>>>(g, (const float2*)kx_in, s1, (float2*)X);  // fewer CTAs: twiddle setup amortised
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

int launch_idft(const dfno_geom& g, const void* Y, float s2, void* kx_out, cudaStream_t st) {
  const int rt = xidft_tc(g, Y, s2, kx_out, st);
  if (rt != DFNO_ERR_UNSUPPORTED) return rt;
  if (tiled_ok(g)) {
    const int xs = x_split(g);
    const int rc = xs == 1 ? launch_tiled(k_xidft_s<1>, g, 1, Y, s2, kx_out, st)
                   : xs == 2 ? launch_tiled(k_xidft_s<2>, g, 2, Y, s2, kx_out, st)
                             : launch_tiled(k_xidft_s<4>, g, 4, Y, s2, kx_out, st);
    if (rc != DFNO_ERR_UNSUPPORTED) return rc;
  }
  const size_t smem = (size_t)g.nx * g.rx * sizeof(float2);
  const long long n = (long long)g.batch * g.c * (long long)ky_local(g) * g.rz * g.rt;
  auto k = g.rx <= 16 ? k_xidft<16, 1> : k_xidft<32, 1>;
  if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  k<<<grid_for(n, 4), kXT, smem, st>>>(g, (const float2*)Y, s2, (float2*)kx_out);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

bool stream_ok(const dfno_geom& g) {
  return g.dtype == DFNO_F32 && g.rx <= 32 && (size_t)g.nx * g.rx * sizeof(float2) <= 200 * 1024 &&
         g.batch <= kBMax;
}
}  // namespace

size_t xspec_stream_workspace(const dfno_geom& g) {
  return 2 * (size_t)g.batch * g.c * g.rx * ky_local(g) * g.rz * g.rt * sizeof(float2);
}

// the three stages on their own (channel-group pipelining in the Python
// layer launches the x-DFTs per channel group around the exchanges)
int xdft_stage(const dfno_geom& g, const void* kx_in, float s1, void* X, cudaStream_t st) {
  if (!stream_ok(g)) return DFNO_ERR_UNSUPPORTED;
  return launch_dft(g, kx_in, s1, X, st);
}

int xidft_stage(const dfno_geom& g, const void* Y, float s2, void* kx_out, cudaStream_t st) {
  if (!stream_ok(g)) return DFNO_ERR_UNSUPPORTED;
  return launch_idft(g, Y, s2, kx_out, st);
}

// Channel grouping of the weight-stream contractions.  A thread owns OG
// channels of one column pair and streams C x OG weight pairs; the grid is the
// resident block count and the kernels stride over it, so a launch takes
// ceil(items / resident threads) rounds.  With OG = 4 at C2 (5 x 32768 items,
// 444 resident blocks) that is 1.44 -> 2 rounds and a third of the GPU idles in
// the second; the pick minimises rounds x requests per item (one shared column
// load per channel plus OG weight loads, and OG gradient stores backward).
// Measured at C2 (ncu, profiles/r02_ab_xmix_og.txt): OG = 1 / 2 / 4 forward
// 45.5 / 61.0 / 78.9 us, backward 80.4 / 98.1 / 159.2 us (the earlier fixed
// OG = 4 with an oversubscribed grid: 44.6 / 115 us).
template <typename K>
struct OgPick {
  int og;
  K kern;
  unsigned grid;
};

template <typename K>
OgPick<K> pick_og(const K (&ks)[3], int (&occ)[3], int C, long long cols2, int reqs_per_og) {
  static const int ogs[3] = {1, 2, 4};
  OgPick<K> best{0, nullptr, 0};
  double best_cost = 0;
  for (int i = 0; i < 3; ++i) {
#ifdef DFNO_XMIX_OG  // A/B experiments only (tools/og_probe.sh)
    if (ogs[i] != DFNO_XMIX_OG) continue;
#endif
    if (!occ[i]) {  // resident blocks per SM, queried once per kernel (same value from every thread)
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks[i], kXT, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
      occ[i] = per_sm;
    }
    const int per_sm = occ[i];
    const long long slots = (long long)per_sm * sms_x();
    const long long items = (long long)((C + ogs[i] - 1) / ogs[i]) * cols2;
    const long long blocks = (items + kXT - 1) / kXT;
    const long long rounds = (items + slots * kXT - 1) / (slots * kXT);
    const double cost = (double)rounds * C * (1 + reqs_per_og * ogs[i]);
    if (!best.kern || cost < best_cost) {
      best = {ogs[i], ks[i], (unsigned)(blocks < slots ? blocks : slots)};
      best_cost = cost;
    }
  }
  return best;
}

int xmix_fwd_stage(const dfno_geom& g, const void* X, const void* w, void* Y, cudaStream_t st) {
  if (!stream_ok(g)) return DFNO_ERR_UNSUPPORTED;
  const long long cols = (long long)g.rx * ky_local(g) * g.rz * g.rt;
  if (cols % 2 == 0) {
    using K = void (*)(const dfno_geom, const float4*, const float4*, float4*);
    static const K ks[3] = {k_xmix2<1>, k_xmix2<2>, k_xmix2<4>};
    static int occ[3];
    const auto p = pick_og(ks, occ, g.c, cols / 2, 1);
    p.kern<<<p.grid, kXT, 0, st>>>(g, (const float4*)X, (const float4*)w, (float4*)Y);
  } else {
    k_xmix<<<grid_for((long long)((g.c + kOG - 1) / kOG) * cols), kXT, 0, st>>>(g, (const float2*)X,
                                                                                (const float2*)w, (float2*)Y);
  }
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

int xmix_bwd_stage(const dfno_geom& g, const void* spec, const void* D, const void* w, void* gw, void* dX,
                   cudaStream_t st) {
  if (!stream_ok(g)) return DFNO_ERR_UNSUPPORTED;
  const long long cols = (long long)g.rx * ky_local(g) * g.rz * g.rt;
  if (cols % 2 == 0 && g.batch == 1) {
    using K = void (*)(const dfno_geom, const float4*, const float4*, const float4*, float4*, float4*);
    static const K ks[3] = {k_xmix_bwd2<1, 1>, k_xmix_bwd2<1, 2>, k_xmix_bwd2<1, 4>};
    static int occ[3];
    const auto p = pick_og(ks, occ, g.c, cols / 2, 2);
    p.kern<<<p.grid, kXT, 0, st>>>(g, (const float4*)spec, (const float4*)D, (const float4*)w, (float4*)gw,
                                   (float4*)dX);
  } else {
    auto kb = g.batch == 1 ? k_xmix_bwd<1> : (g.batch == 2 ? k_xmix_bwd<2> : k_xmix_bwd<kBMax>);
    kb<<<grid_for((long long)((g.c + kOG - 1) / kOG) * cols), kXT, 0, st>>>(
        g, (const float2*)spec, (const float2*)D, (const float2*)w, (float2*)gw, (float2*)dX);
  }
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

int xspec_fwd_stream(const dfno_geom& g, const void* kx_in, const void* w, void* spec, void* kx_out, void* work,
                     cudaStream_t st) {
  if (!stream_ok(g)) return DFNO_ERR_UNSUPPORTED;
  const size_t half = xspec_stream_workspace(g) / 2;
  void* X = spec ? spec : work;
  void* Y = static_cast<char*>(work) + half;
  int rc = launch_dft(g, kx_in, 1.f, X, st);  // fft_x unnormalised (d/spectral.py:36)
  if (rc) return rc;
  rc = xmix_fwd_stage(g, X, w, Y, st);
  if (rc) return rc;
  return launch_idft(g, Y, (float)(1.0 / g.nx), kx_out, st);  // ifft_x carries 1/Nx (d/spectral.py:49)
}

int xspec_bwd_stream(const dfno_geom& g, const void* kx_in, const void* spec, const void* w, void* gw, void* kx_out,
                     void* work, cudaStream_t st) {
  if (!stream_ok(g)) return DFNO_ERR_UNSUPPORTED;
  const size_t half = xspec_stream_workspace(g) / 2;
  void* D = work;
  void* dX = static_cast<char*>(work) + half;
  int rc = launch_dft(g, kx_in, (float)(1.0 / g.nx), D, st);  // fft_x / Nx (d/fno.py:450-452)
  if (rc) return rc;
  rc = xmix_bwd_stage(g, spec, D, w, gw, dX, st);
  if (rc) return rc;
  return launch_idft(g, dX, 1.f, kx_out, st);  // ifft_x * Nx = unnormalised inverse (d/fno.py:455-457)
}

}  // namespace dfno
