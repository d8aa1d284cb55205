// Truncated DFT along x on the tcgen05 tensor cores (3xTF32): the two ends of
// the streamed x-spectral stage (xspec_stream.cu), any N_x, r_x <= 16.
//
//   k_xdft_tc   X[b][c][kx][m] = s1 * sum_x Z[b][c][x][m] e^{-2 pi i f(kx) x / Nx}
//               (reference d/fno.py:331-332, backward d/fno.py:450-452; Z is
//               gathered straight from the peer-major KX exchange buffer)
//   k_xidft_tc  U[b][c][x][m] = s2 * sum_kx Y[b][c][kx][m] e^{+2 pi i f(kx) x / Nx}
//               written straight into the KX layout (d/fno.py:335-336,
//               d/fno.py:455-457; the zero padding of the missing kx is implicit)
//
// Both are GEMMs with the 128 modes m of a tile as M (TMEM lane = thread =
// mode, so every global access is a coalesced run of consecutive modes), the
// realified complex x (or kx) as K = 32 per chunk of 16, and the realified
// twiddles of the retained kx (or of 16 x) as the small B operand, stacked
// [hi ; lo] so one N = 64 MMA yields hi.hi and hi.lo and a second N = 32 MMA
// adds lo.hi (3xTF32, the accumulator halves are summed on read-out).
//
//   forward   per chunk of 16 x: each thread loads its 16 complex Z (one chunk
//             ahead in registers), splits hi / lo into a double-buffered A in
//             TMEM, thread 0 issues 8 MMAs into one accumulator per tile.  When
//             the x extent is long and the (b c, mode) tiles few -- P = 8 ky
//             pencils have 2 x 16 x 16 modes per (b, c) -- the x range is split
//             over the CTAs of a cluster and the partial spectra are summed in
//             a fixed rank order through distributed shared memory.
//   inverse   per tile the 16 complex Y of each mode go to TMEM once; per chunk
//             of 16 x one N = 64 + one N = 32 MMA group per K step into a
//             double-buffered accumulator whose read-out (16 complex outputs
//             per mode) overlaps the next chunk's MMAs.  Long x extents are
//             split over independent CTAs (no reduction needed).
//
// Twiddles: exact integer phase reduction (f x mod N_x) into a double-precision
// table, split hi / lo round-to-nearest; the CTA's twiddle chunks for its x
// range stay resident in shared memory across the tiles it walks (persistent).
#include <cooperative_groups.h>

#include "common.cuh"
#include "tc.cuh"

namespace cg = cooperative_groups;

namespace dfno {

namespace {

constexpr int kT = 128;                    // threads = modes per tile = TMEM lanes
constexpr int kC = 16;                     // x per chunk (K = 32 reals)
constexpr int kBChunk = 64 * 32 * 4;       // one chunk of [B_hi ; B_lo]: 64 rows x K 32, K-major, SBO 1024
constexpr int kTmemCols = 256;

__device__ __forceinline__ int kmajb(int r, int k) { return (r >> 3) * 1024 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4; }

struct XLay {
  int xcnt, nch;         // x in this CTA's range, chunks
  int off_ph, off_rows, off_b, off_red, total;
};

// offsets sized for the longest x range of the split (xmax), so every CTA of
// a cluster has the same layout (the reduction reads peers' buffers at its
// own offset); xcnt is this CTA's own range
__host__ __device__ inline XLay make_xlay(int nx, int xmax, int xcnt, bool red) {
  XLay L;
  const int nch_max = (xmax + kC - 1) / kC;
  L.xcnt = xcnt;
  L.nch = (xcnt + kC - 1) / kC;
  int o = 0;
  L.off_ph = o; o += 16 * nx;                         // float4 (cos hi, cos lo, sin hi, sin lo) of 2 pi j / N_x
  L.off_rows = o; o += 2 * 8 * nch_max * kC;          // per x of the range: KX row offset at (b c) = 0, (b c) stride
  o = (o + 1023) & ~1023;
  L.off_b = o; o += nch_max * kBChunk;
  L.off_red = o; o += red ? kT * 33 * 4 : 0;         // cluster reduction: [mode][32 (+1)] partial sums
  L.total = o;
  return L;
}

// phase table and the resident twiddle chunks of x in [x0, x0 + xcnt): one
// (x, kx) pair per step -- one integer phase reduction (f x mod N_x) feeds
// its eight entries (re / im row, two K parts, hi / lo plane).
// Forward (e^{-i}): rows = kx (re 0-15, im 16-31), K = (x, part):
//   re = zr c + zi s ; im = zi c - zr s.
// Inverse (e^{+i}): rows = x of the chunk, K = (kx, part):
//   re = yr c - yi s ; im = yi c + yr s.
template <bool INV>
__device__ void build_twiddles(const dfno_geom& g, const XLay& L, unsigned char* smem, int x0) {
  float4* ph = reinterpret_cast<float4*>(smem + L.off_ph);
  // fp32 sincospif (<= 1 ulp, exact phase reduction already done) then the
  // hi / lo split of the fp32 value: the pair carries the twiddle to ~2^-24
  for (int j = threadIdx.x; j < g.nx; j += blockDim.x) {
    float s, c;
    sincospif(2.0f * (float)j / (float)g.nx, &s, &c);
    const float ch = tc::round_tf32(c), sh = tc::round_tf32(s);
    ph[j] = make_float4(ch, tc::round_tf32(c - ch), sh, tc::round_tf32(s - sh));
  }
  __syncthreads();
  float* b = reinterpret_cast<float*>(smem + L.off_b);
  const int nx = g.nx;
  for (int e = threadIdx.x; e < L.nch * kC * 16; e += blockDim.x) {
    const int slot = e >> 4, kx = e & 15, ch = slot / kC, xi = slot % kC;
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    if (kx < g.rx && slot < L.xcnt) {
      const int f = ((mode_freq(kx, nx, g.mx) % nx) + nx) % nx;
      t = ph[(f * (x0 + slot)) % nx];
    }
    const int row = INV ? xi : kx, kk = INV ? kx : xi;
    unsigned char* bc = reinterpret_cast<unsigned char*>(b) + ch * kBChunk;
#pragma unroll
    for (int pl = 0; pl < 2; ++pl) {  // hi, lo planes
      const float cv = pl ? t.y : t.x, sv = pl ? t.w : t.z;
      const int r_re = 32 * pl + row, r_im = r_re + 16;
      *reinterpret_cast<float*>(bc + kmajb(r_re, 2 * kk)) = cv;
      *reinterpret_cast<float*>(bc + kmajb(r_re, 2 * kk + 1)) = INV ? -sv : sv;
      *reinterpret_cast<float*>(bc + kmajb(r_im, 2 * kk)) = INV ? sv : -sv;
      *reinterpret_cast<float*>(bc + kmajb(r_im, 2 * kk + 1)) = cv;
    }
  }
}

// KX layout (common.cuh kx_row): row(bc, x) = r0[x] + bc * rs[x], tables for
// the CTA's x range built once (no per-tile row table, no per-tile barrier)
__device__ void build_rows(const dfno_geom& g, long long* r0, long long* rs, int x0, int xcnt) {
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  for (int i = threadIdx.x; i < xcnt; i += blockDim.x) {
    const int x = x0 + i;
    const int p = x_owner(g, x);
    const long long xp = g.x_starts[p + 1] - g.x_starts[p];
    r0[i] = kx_row(g, 0, 0, x);
    rs[i] = xp * mloc;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// forward: grid = (clusters of XS CTAs) x (tile walkers); CTA rank r of a
// cluster owns x range r.
__global__ void __launch_bounds__(kT, 2) k_xdft_tc(const dfno_geom g, const float2* __restrict__ kx_in, float s1,
                                                   float2* __restrict__ X, int xs) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t done[2];
  __shared__ uint32_t tmem_base;
  const int Nx = g.nx, tid = threadIdx.x, warp = tid >> 5;
  const int rank = xs > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int x0 = (int)((long long)Nx * rank / xs), x1 = (int)((long long)Nx * (rank + 1) / xs);
  const XLay L = make_xlay(Nx, (Nx + xs - 1) / xs, x1 - x0, xs > 1);
  build_twiddles<false>(g, L, smem, x0);
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&done[0], 1);
    tc::mbar_init(&done[1], 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base, lane_off = (uint32_t)(32 * warp) << 16;
  const uint32_t cA = 0, cD = 128;  // A: 2 x (hi 32 | lo 32); D: 2 x 64
  long long* r0 = reinterpret_cast<long long*>(smem + L.off_rows);
  long long* rs = r0 + L.nch * kC;
  build_rows(g, r0, rs, x0, L.xcnt);
  __syncthreads();
  const uint32_t sb = tc::smem_u32(smem + L.off_b);
  const uint32_t id64 = tc::idesc_tf32(128, 64), id32 = tc::idesc_tf32(128, 32);

  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long mtiles = (mloc + kT - 1) / kT;
  const long long ntiles = (long long)g.batch * g.c * mtiles;
  const long long walkers = gridDim.x / xs, w0 = blockIdx.x / xs;
  int q = 0;  // running chunk counter: A / D buffer parity
  // the loads run one chunk ahead, across tile boundaries
  float2 z[kC];
  auto fetch = [&](long long tile, int ch) {
    const long long bc = tile / mtiles, m = (tile - bc * mtiles) * kT + tid;
    const bool ok = tile < ntiles && m < mloc;
#pragma unroll
    for (int i = 0; i < kC; ++i) {
      const int xi = ch * kC + i;
      z[i] = (ok && xi < L.xcnt) ? __ldcs(kx_in + r0[xi] + bc * rs[xi] + m) : make_float2(0.f, 0.f);
    }
  };
  fetch(w0, 0);
  for (long long tile = w0; tile < ntiles; tile += walkers) {
    const long long bc = tile / mtiles, m = (tile - bc * mtiles) * kT + tid;
    const bool ok = m < mloc;
    // Each chunk accumulates in a fresh TMEM accumulator (double-buffered with
    // A) and the chunk sums are added in registers with round-to-nearest
    // fp32 adds: the tensor core's accumulator adds truncate, and a long
    // x extent (N_x / 16 chunks x 4 K steps) would otherwise build a biased
    // error into the spectrum.
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = 0.f;
    auto drain = [&](int qq) {
      const int db = qq & 1;
      tc::mbar_wait(&done[db], (qq >> 1) & 1);
      tc::fence_after();
      uint32_t r0[32], r1[32];
      tc::tmem_ld32_nowait(tmem + cD + 64 * db + lane_off, r0);
      tc::tmem_ld32_nowait(tmem + cD + 64 * db + 32 + lane_off, r1);
      tc::tmem_ld_wait();
      tc::fence_before();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += __uint_as_float(r0[j]) + __uint_as_float(r1[j]);
    };
    for (int ch = 0; ch < L.nch; ++ch, ++q) {
      float h[32], l[32];
#pragma unroll
      for (int i = 0; i < kC; ++i) tc::split_hl2(z[i], h[2 * i], h[2 * i + 1], l[2 * i], l[2 * i + 1]);
      if (ch + 1 < L.nch) fetch(tile, ch + 1);
      else fetch(tile + walkers, 0);
      const int ab = q & 1;
      // buffer ab (A and D) was last used by chunk q - 2, drained by this
      // thread one iteration ago (or in the previous tile)
      tc::tmem_st32(tmem + cA + 64 * ab + lane_off, h);
      tc::tmem_st32(tmem + cA + 64 * ab + 32 + lane_off, l);
      tc::tmem_st_wait();
      tc::fence_before();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after();
        const uint32_t a = tmem + cA + 64 * ab, d = tmem + cD + 64 * ab, bch = sb + ch * kBChunk;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint64_t bd = tc::desc(bch + s * 256, 128, 1024);
          tc::mma_tf32_ts(d, a + 8 * s, bd, id64, s ? 1u : 0u);  // hi.[hi | lo]
          tc::mma_tf32_ts(d + 32, a + 32 + 8 * s, bd, id32, 1u);  // lo.hi
        }
        tc::commit(&done[ab]);
      }
      __syncwarp();
      if (ch > 0) drain(q - 1);
    }
    drain(q - 1);
    float2* dst = X + (bc * g.rx) * mloc;
    if (xs == 1) {
      if (ok)
#pragma unroll
        for (int kx = 0; kx < 16; ++kx)
          if (kx < g.rx) dst[(long long)kx * mloc + m] = make_float2(s1 * v[kx], s1 * v[16 + kx]);
      continue;
    }
    // partial spectra of the cluster's x ranges, summed in rank order
    float* red = reinterpret_cast<float*>(smem + L.off_red);
#pragma unroll
    for (int j = 0; j < 32; ++j) red[tid * 33 + j] = v[j];
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int per = kT / xs;  // modes reduced by this rank
    for (int e = tid; e < per * 16; e += kT) {
      const int row = rank * per + e % per, kx = e / per;
      float re = 0.f, im = 0.f;
      for (int p = 0; p < xs; ++p) {
        const float* rr = cl.map_shared_rank(red, p);
        re += rr[row * 33 + kx];
        im += rr[row * 33 + 16 + kx];
      }
      const long long mm = (tile - bc * mtiles) * kT + row;
      if (kx < g.rx && mm < mloc) dst[(long long)kx * mloc + mm] = make_float2(s1 * re, s1 * im);
    }
    cl.sync();  // every rank has read every partial before they are overwritten / freed
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTmemCols>(tmem);
}

// ---------------------------------------------------------------------------
// inverse: CTA = (x part) x (tile walker); independent CTAs.
__global__ void __launch_bounds__(kT, 2) k_xidft_tc(const dfno_geom g, const float2* __restrict__ Y, float s2,
                                                    float2* __restrict__ kx_out, int xs) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t dfull[2], dfree[2];
  __shared__ uint32_t tmem_base;
  const int Nx = g.nx, tid = threadIdx.x, warp = tid >> 5;
  const int part = blockIdx.x % xs;
  const int x0 = (int)((long long)Nx * part / xs), x1 = (int)((long long)Nx * (part + 1) / xs);
  const XLay L = make_xlay(Nx, (Nx + xs - 1) / xs, x1 - x0, false);
  build_twiddles<true>(g, L, smem, x0);
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&tmem_base);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&dfull[b], 1);
      tc::mbar_init(&dfree[b], kT);
    }
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base, lane_off = (uint32_t)(32 * warp) << 16;
  const uint32_t cA = 0, cD = 64;  // A: hi 32 | lo 32; D: 2 x 64
  long long* r0t = reinterpret_cast<long long*>(smem + L.off_rows);
  long long* rst = r0t + L.nch * kC;
  build_rows(g, r0t, rst, x0, L.xcnt);
  __syncthreads();
  const uint32_t sb = tc::smem_u32(smem + L.off_b);
  const uint32_t id64 = tc::idesc_tf32(128, 64), id32 = tc::idesc_tf32(128, 32);

  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  const long long mtiles = (mloc + kT - 1) / kT;
  const long long ntiles = (long long)g.batch * g.c * mtiles;
  const long long walkers = gridDim.x / xs, w0 = blockIdx.x / xs;
  int q = 0;  // running chunk counter (D buffer parity)
  auto issue = [&](int ch, int qq) {
    const int db = qq & 1;
    if (qq >= 2) tc::mbar_wait(&dfree[db], ((qq >> 1) & 1) ^ 1);
    tc::fence_after();
    const uint32_t d = tmem + cD + 64 * db, bch = sb + ch * kBChunk;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint64_t bd = tc::desc(bch + s * 256, 128, 1024);
      tc::mma_tf32_ts(d, tmem + cA + 8 * s, bd, id64, s ? 1u : 0u);      // hi.[hi | lo]
      tc::mma_tf32_ts(d + 32, tmem + cA + 32 + 8 * s, bd, id32, 1u);     // lo.hi
    }
    tc::commit(&dfull[db]);
  };
  // the next tile's Y is loaded while this tile's chunks run
  float2 yv[16];
  auto load_y = [&](long long tile) {
    const long long bc = tile / mtiles, m = (tile - bc * mtiles) * kT + tid;
    const bool ok = tile < ntiles && m < mloc;
    const float2* src = Y + (bc * g.rx) * mloc + m;
#pragma unroll
    for (int kx = 0; kx < 16; ++kx)
      yv[kx] = (ok && kx < g.rx) ? __ldg(src + (long long)kx * mloc) : make_float2(0.f, 0.f);
  };
  load_y(w0);
  for (long long tile = w0; tile < ntiles; tile += walkers) {
    const long long bc = tile / mtiles, m = (tile - bc * mtiles) * kT + tid;
    const bool ok = m < mloc;
    float h[32], l[32];
#pragma unroll
    for (int kx = 0; kx < 16; ++kx) tc::split_hl2(yv[kx], h[2 * kx], h[2 * kx + 1], l[2 * kx], l[2 * kx + 1]);
    load_y(tile + walkers);
    // the previous tile's MMAs (which read A) are done: this thread waited
    // on that tile's last accumulator, committed after all of them
    tc::tmem_st32(tmem + cA + lane_off, h);
    tc::tmem_st32(tmem + cA + 32 + lane_off, l);
    tc::tmem_st_wait();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) issue(0, q);
    __syncwarp();
    for (int ch = 0; ch < L.nch; ++ch, ++q) {
      if (tid == 0 && ch + 1 < L.nch) issue(ch + 1, q + 1);
      __syncwarp();
      const int db = q & 1;
      tc::mbar_wait(&dfull[db], (q >> 1) & 1);
      tc::fence_after();
      uint32_t r0[32], r1[32];
      tc::tmem_ld32_nowait(tmem + cD + 64 * db + lane_off, r0);
      tc::tmem_ld32_nowait(tmem + cD + 64 * db + 32 + lane_off, r1);
      tc::tmem_ld_wait();
      tc::fence_before();
      tc::mbar_arrive(&dfree[db]);
      if (ok) {
#pragma unroll
        for (int i = 0; i < kC; ++i) {
          const int xi = ch * kC + i;
          if (xi < L.xcnt) {
            const float re = __uint_as_float(r0[i]) + __uint_as_float(r1[i]);
            const float im = __uint_as_float(r0[16 + i]) + __uint_as_float(r1[16 + i]);
            __stcs(kx_out + r0t[xi] + bc * rst[xi] + m, make_float2(s2 * re, s2 * im));
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTmemCols>(tmem);
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

long long xtiles(const dfno_geom& g) {
  const long long mloc = (long long)ky_local(g) * g.rz * g.rt;
  return (long long)g.batch * g.c * ((mloc + kT - 1) / kT);
}

// x split: the smallest power of two (<= 8) giving two CTAs per SM, also
// keeping every part at least one chunk long
int xsplit(const dfno_geom& g) {
  const long long t = xtiles(g);
  int xs = 1;
  while (xs < 8 && t * xs < 2LL * sms_xt() && g.nx / (2 * xs) >= kC) xs *= 2;
  return xs;
}
}  // namespace

int xdft_tc(const dfno_geom& g, const void* kx_in, float s1, void* X, cudaStream_t st) {
  if (g.dtype != DFNO_F32 || g.rx > 16) return DFNO_ERR_UNSUPPORTED;
  const int xs = xsplit(g);
  const int xmax = (g.nx + xs - 1) / xs;
  const XLay L = make_xlay(g.nx, xmax, xmax, xs > 1);
  const int smem = L.total + 1024;
  if (smem > 200 * 1024) return DFNO_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(k_xdft_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const long long t = xtiles(g);
  long long walkers = 2LL * sms_xt() / xs;
  if (walkers > t) walkers = t;
  if (walkers < 1) walkers = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(walkers * xs));
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = xs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k_xdft_tc, g, (const float2*)kx_in, s1, (float2*)X, xs) != cudaSuccess)
    return DFNO_ERR_CUDA;
  return DFNO_OK;
}

int xidft_tc(const dfno_geom& g, const void* Y, float s2, void* kx_out, cudaStream_t st) {
  if (g.dtype != DFNO_F32 || g.rx > 16) return DFNO_ERR_UNSUPPORTED;
  // the inverse's x parts are independent CTAs (no reduction), so splitting
  // even a well-filled grid in two shortens each CTA's serial chunk chain:
  // C2 26.5 -> 23.9 us, C3 45.4 -> 39.2 us (a split of 4: 26.8 / 40.5); the
  // forward's cluster split only pays when tiles are scarce (C2 22.5 -> 56 us)
  int xs = xsplit(g);
  if (xs < 2 && g.nx / 4 >= kC) xs = 2;
  const int xmax = (g.nx + xs - 1) / xs;
  const XLay L = make_xlay(g.nx, xmax, xmax, false);
  const int smem = L.total + 1024;
  if (smem > 200 * 1024) return DFNO_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(k_xidft_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const long long t = xtiles(g);
  long long walkers = 2LL * sms_xt() / xs;
  if (walkers > t) walkers = t;
  if (walkers < 1) walkers = 1;
  k_xidft_tc<<<(unsigned)(walkers * xs), kT, smem, st>>>(g, (const float2*)Y, s2, (float2*)kx_out, xs);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

}  // namespace dfno
