// Truncated DFT along x on the tcgen05 tensor cores (3xTF32), the two ends of
// the streamed x-spectral stage (xspec_stream.cu):
//
//   k_xdft_tc   X[b][c][kx][m] = s1 * sum_x Z[b][c][x][m] e^{-2 pi i f(kx) x / Nx}
//               (d/fno.py:331-332; Z gathered from the peer-major KX buffer)
//               one CTA tile = 128 modes m of one (b, c): A = Z^T (128 m x
//               (x re | x im), 16 x per chunk) split hi / lo into TMEM by the
//               owning thread, B = realified twiddles [[C, S]; [-S, C]] in
//               shared memory, D (128 m x (kx re | kx im)) accumulated over
//               the x chunks, read back by the owning thread.
//   k_xidft_tc  U[b][c][x][m] = s2 * sum_kx Y[b][c][kx][m] e^{+2 pi i f(kx) x / Nx}
//               (d/fno.py:335-336; zero padding implicit) written into the KX
//               layout: A = Y^T (128 m x (kx re | kx im)) in TMEM, N = 64 x
//               (re | im) per MMA group.
// The data operand is the M = 128 side (TMEM, no shared-memory re-reads); the
// twiddles are the small B operand.  Two CTAs per SM; each CTA loads the
// next chunk while its MMAs run.  Envelope: fp32, r_x <= 16, N_x <= 128.
#include "common.cuh"
#include "tc.cuh"

namespace dfno {

namespace {
constexpr int kXTh = 128;
constexpr int kXC = 16;                   // x per chunk in the forward (K' = 32)
constexpr int kIXC = 64;                  // x per MMA group in the inverse (N = 128)

__device__ __forceinline__ int kmajx(int r, int k, int sbo) {
  return (r >> 3) * sbo + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ void put_split_x(unsigned char* b, int plane, int off, double v) {
  const float hi = tc::round_tf32((float)v);
  const float lo = tc::round_tf32((float)(v - (double)hi));
  *reinterpret_cast<float*>(b + off) = hi;
  *reinterpret_cast<float*>(b + plane + off) = lo;
}

__device__ __forceinline__ void csx(int k, int x, const dfno_geom& g, double& c, double& s) {
  c = s = 0.0;
  if (k < g.rx && x < g.nx) {
    const long long idx = ((long long)mode_freq(k, g.nx, g.mx) * x) % g.nx;
    sincospi(2.0 * (double)idx / g.nx, &s, &c);
  }
}
}  // namespace

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kXTh, 4) k_xdft_tc(const dfno_geom g, const float2* __restrict__ kx_in, float s1,
                                                     float2* __restrict__ X) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int Nx = g.nx, nch = (Nx + kXC - 1) / kXC;
  const int sbo = 8 * 128;                 // K' = 32 -> 8 core matrices per 8-row group
  const int plane = nch * 4 * sbo;         // rows (chunk, n 0..31) x K' 32, hi then lo
  // B rows (chunk q, n): n < 16 out re(kx = n), n >= 16 out im; K' = (x re | x im)
  // of chunk q.  One sincospi per (kx, x) pair feeds its four realified entries.
  for (int e = threadIdx.x; e < nch * kXC * 16; e += kXTh) {
    const int kx = e % 16, x = e / 16, q = x / kXC, xl = x % kXC;
    double c, s;
    csx(kx, x, g, c, s);  // e^{-i}: re = zr C + zi S ; im = zi C - zr S
    const int r0 = q * 32 + kx, r1 = r0 + 16;
    put_split_x(smem, plane, kmajx(r0, xl, sbo), c);
    put_split_x(smem, plane, kmajx(r0, 16 + xl, sbo), s);
    put_split_x(smem, plane, kmajx(r1, xl, sbo), -s);
    put_split_x(smem, plane, kmajx(r1, 16 + xl, sbo), c);
  }
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc<128>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base, d = tmem, ah = tmem + 32, al = tmem + 64;
  const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long mtiles = (mloc + kXTh - 1) / kXTh;
  const long long ntiles = (long long)g.batch * g.c * mtiles;
  const uint32_t sb = tc::smem_u32(smem), id = tc::idesc_tf32(128, 32);
  int it = 0;  // MMA groups issued by this CTA (mbarrier phases)

  float2 zv[kXC];
  auto load = [&](long long tile, int q) {
    const long long bc = tile / mtiles;
    const long long m = (tile - bc * mtiles) * kXTh + tid;
    const bool ok = tile < ntiles && m < mloc;
    const int c = (int)(bc % g.c), bb = (int)(bc / g.c);
    // row pointer advanced by mloc per x inside a peer chunk; recomputed at
    // chunk boundaries of the peer-major KX layout
    const int x0 = q * kXC;
    int p = x_owner(g, min(x0, Nx - 1)), pend = g.x_starts[p + 1];
    const float2* src = kx_in + kx_row(g, bb, c, min(x0, Nx - 1)) + m;
#pragma unroll
    for (int j = 0; j < kXC; ++j) {
      const int x = x0 + j;
      if (x == pend && x < Nx) {
        ++p;
        pend = g.x_starts[p + 1];
        src = kx_in + kx_row(g, bb, c, x) + m;
      }
      zv[j] = (ok && x < Nx) ? __ldcs(src) : make_float2(0.f, 0.f);
      src += mloc;
    }
  };
  long long tile = blockIdx.x;
  if (tile < ntiles) load(tile, 0);
#pragma unroll 1
  for (; tile < ntiles; tile += gridDim.x) {
    for (int q = 0; q < nch; ++q, ++it) {
      float h[32], l[32];
#pragma unroll
      for (int j = 0; j < kXC; ++j) {
        tc::split_hl(zv[j].x, h[j], l[j]);
        tc::split_hl(zv[j].y, h[16 + j], l[16 + j]);
      }
      // prefetch the next chunk (or the next tile's first chunk)
      if (q + 1 < nch) load(tile, q + 1);
      else load(tile + gridDim.x, 0);
      if (it > 0) {
        tc::mbar_wait(&bar, (it - 1) & 1);
        tc::fence_after();
      }
      tc::tmem_st32(ah + lane_off, h);
      tc::tmem_st32(al + lane_off, l);
      tc::tmem_st_wait();
      tc::fence_before();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint32_t kb = (uint32_t)q * 4 * sbo + s * 256;
          const uint64_t bh = tc::desc(sb + kb, 128, sbo), bl = tc::desc(sb + plane + kb, 128, sbo);
          tc::mma_tf32_ts(d, ah + 8 * s, bh, id, (q | s) ? 1u : 0u);
          tc::mma_tf32_ts(d, al + 8 * s, bh, id, 1u);
          tc::mma_tf32_ts(d, ah + 8 * s, bl, id, 1u);
        }
        tc::commit(&bar);
      }
    }
    // tile done: D -> X
    tc::mbar_wait(&bar, (it - 1) & 1);
    tc::fence_after();
    uint32_t r[32];
    tc::tmem_ld32_nowait(d + lane_off, r);
    tc::tmem_ld_wait();
    tc::fence_before();
    __syncthreads();  // every thread has read D before the next tile's first MMA overwrites it
    const long long bc = tile / mtiles;
    const long long m = (tile - bc * mtiles) * kXTh + tid;
    if (m < mloc) {
      float2* dst = X + (bc * g.rx) * mloc + m;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < g.rx) __stcs(dst + (long long)k * mloc, make_float2(s1 * __uint_as_float(r[k]), s1 * __uint_as_float(r[16 + k])));
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<128>(tmem);
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kXTh, 2) k_xidft_tc(const dfno_geom g, const float2* __restrict__ Y, float s2,
                                                      float2* __restrict__ kx_out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int Nx = g.nx, ngr = (Nx + kIXC - 1) / kIXC;
  const int sbo = 8 * 128;                 // K' = 32 (kx re | kx im)
  const int plane = ngr * 16 * sbo;        // rows (group, n 0..127) x K' 32
  // B rows (group p, n): n < 64 out re(x = 64 p + n), n >= 64 out im; e^{+i}:
  // re = yr C - yi S ; im = yr S + yi C.  One sincospi per (kx, x) pair.
  for (int e = threadIdx.x; e < ngr * kIXC * 16; e += kXTh) {
    const int kx = e % 16, x = e / 16, p = x / kIXC, xl = x % kIXC;
    double c, s;
    csx(kx, x, g, c, s);
    const int r0 = p * 128 + xl, r1 = r0 + 64;
    put_split_x(smem, plane, kmajx(r0, kx, sbo), c);
    put_split_x(smem, plane, kmajx(r0, 16 + kx, sbo), -s);
    put_split_x(smem, plane, kmajx(r1, kx, sbo), s);
    put_split_x(smem, plane, kmajx(r1, 16 + kx, sbo), c);
  }
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base, d = tmem, ah = tmem + 128, al = tmem + 160;
  const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long mtiles = (mloc + kXTh - 1) / kXTh;
  const long long ntiles = (long long)g.batch * g.c * mtiles;
  const uint32_t sb = tc::smem_u32(smem), id = tc::idesc_tf32(128, 128);
  int it = 0;

  float2 yv[16];
  auto load = [&](long long tile) {
    const long long bc = tile / mtiles;
    const long long m = (tile - bc * mtiles) * kXTh + tid;
    const bool ok = tile < ntiles && m < mloc;
    const float2* src = Y + (bc * g.rx) * mloc + m;
#pragma unroll
    for (int k = 0; k < 16; ++k) yv[k] = (ok && k < g.rx) ? __ldcs(src + (long long)k * mloc) : make_float2(0.f, 0.f);
  };
  long long tile = blockIdx.x;
  if (tile < ntiles) load(tile);
#pragma unroll 1
  for (; tile < ntiles; tile += gridDim.x) {
    float h[32], l[32];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      tc::split_hl(yv[k].x, h[k], l[k]);
      tc::split_hl(yv[k].y, h[16 + k], l[16 + k]);
    }
    load(tile + gridDim.x);
    const long long bc = tile / mtiles;
    const long long m = (tile - bc * mtiles) * kXTh + tid;
    const int c = (int)(bc % g.c), bb = (int)(bc / g.c);
    tc::tmem_st32(ah + lane_off, h);
    tc::tmem_st32(al + lane_off, l);
    tc::tmem_st_wait();
    tc::fence_before();
    __syncthreads();
    for (int p = 0; p < ngr; ++p, ++it) {
      if (tid == 0) {
        tc::fence_after();
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint32_t kb = (uint32_t)p * 16 * sbo + s * 256;
          const uint64_t bh = tc::desc(sb + kb, 128, sbo), bl = tc::desc(sb + plane + kb, 128, sbo);
          tc::mma_tf32_ts(d, ah + 8 * s, bh, id, s ? 1u : 0u);
          tc::mma_tf32_ts(d, al + 8 * s, bh, id, 1u);
          tc::mma_tf32_ts(d, ah + 8 * s, bl, id, 1u);
        }
        tc::commit(&bar);
      }
      tc::mbar_wait(&bar, it & 1);
      tc::fence_after();
      // D row m: cols 0..63 re(x), 64..127 im(x) of this x group
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t re[32], im[32];
        tc::tmem_ld32_nowait(d + lane_off + 32 * h2, re);
        tc::tmem_ld32_nowait(d + lane_off + 64 + 32 * h2, im);
        tc::tmem_ld_wait();
        if (m < mloc) {
#pragma unroll
          const int xa = p * kIXC + 32 * h2;
          int q = x_owner(g, min(xa, Nx - 1)), qend = g.x_starts[q + 1];
          float2* dst = kx_out + kx_row(g, bb, c, min(xa, Nx - 1)) + m;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int x = xa + j;
            if (x == qend && x < Nx) {
              ++q;
              qend = g.x_starts[q + 1];
              dst = kx_out + kx_row(g, bb, c, x) + m;
            }
            if (x < Nx) __stcs(dst, make_float2(s2 * __uint_as_float(re[j]), s2 * __uint_as_float(im[j])));
            dst += mloc;
          }
        }
      }
      tc::fence_before();
      __syncthreads();  // D consumed before the next group's MMAs; A free after the last group
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

// ---------------------------------------------------------------------------
namespace {
int sms_xt() {
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

int xdft_tc(const dfno_geom& g, const void* kx_in, float s1, void* X, cudaStream_t st) {
  if (g.dtype != DFNO_F32 || g.rx > 16 || g.nx > 128) return DFNO_ERR_UNSUPPORTED;
  const int nch = (g.nx + kXC - 1) / kXC;
  const int smem = 2 * nch * 4 * 8 * 128;
  if (cudaFuncSetAttribute(k_xdft_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long tiles = (long long)g.batch * g.c * ((mloc + kXTh - 1) / kXTh);
  const long long grid = tiles < 4LL * sms_xt() ? tiles : 4LL * sms_xt();  // 128 TMEM columns: 4 CTAs / SM
  k_xdft_tc<<<(unsigned)grid, kXTh, smem, st>>>(g, (const float2*)kx_in, s1, (float2*)X);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

int xidft_tc(const dfno_geom& g, const void* Y, float s2, void* kx_out, cudaStream_t st) {
  if (g.dtype != DFNO_F32 || g.rx > 16 || g.nx > 128) return DFNO_ERR_UNSUPPORTED;
  const int ngr = (g.nx + kIXC - 1) / kIXC;
  const int smem = 2 * ngr * 16 * 8 * 128;
  if (cudaFuncSetAttribute(k_xidft_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long tiles = (long long)g.batch * g.c * ((mloc + kXTh - 1) / kXTh);
  const long long grid = tiles < 2LL * sms_xt() ? tiles : 2LL * sms_xt();
  k_xidft_tc<<<(unsigned)grid, kXTh, smem, st>>>(g, (const float2*)Y, s2, (float2*)kx_out);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

}  // namespace dfno
