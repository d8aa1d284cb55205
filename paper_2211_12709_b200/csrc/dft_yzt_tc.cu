// Truncated (y, z, t) DFTs on the 5th-generation tensor cores (tcgen05,
// kind::tf32, fp32 accumulation in TMEM) with 3xTF32 operand splitting
// (hi*hi + lo*hi + hi*lo, round-to-nearest split), so results carry
// fp32-level accuracy; tests/test_gpu_kernels.py checks them against numpy
// real64.
//
// FORWARD (replaces fft_dims(a,(y,z,t)) + truncate_modes, reference
// d/fno.py:328-329; backward use d/fno.py:446-448).  A persistent CTA walks
// (b, c, x) slabs; each slab is consumed in tiles of 8 y-planes x 16 z-rows x
// 32 t, streamed into a ring of raw shared-memory stages with cp.async
// (several tiles in flight per SM), then converted (activation or
// grad*act' fused, 3xTF32 split) into the stage-T operand:
//
//   stage T  D1[(y,z)][kt re|im] = sum_t f(a)[y][z][t] {cos,-sin}      M=128 N=32 K=32
//   stage Z  D2[(kt,y)][kz]     += sum_z D1 e^{-i kz z} (planar re/im)  M=128 N=16 K=16 per tile
//   stage Y  D3[(kz,kt)][ky]    += sum_y D2 e^{-i ky y}  (per 8 y)      M=2x128 N=16 K=8
//
// INVERSE (replaces pad_modes + ifft_dims(yzt) + .real, d/fno.py:338-343 /
// d/fno.py:459-464), per slab, per 16-y chunk:
//
//   stage Y' D1[(kz,kt)][y]  = sum_ky V e^{+i ky y}                    M=2x128 N=16 K=16
//   stage Z' D2[(y,kt)][z]   = sum_kz D1 e^{+i kz z}                   M=2x128 N<=64 K=16
//   stage T' D3[(y,z)][t]    = Re sum_kt D2 e^{+i kt t}  (real output)  M=2x128 N=32 K=16
//
// The transposes between stages go TMEM -> registers -> shared memory into
// SWIZZLE_NONE K-major tiles whose LBO / SBO paddings make the stores
// bank-conflict free.  Twiddles are generated per CTA with exact integer
// phase reduction (double precision) and split hi / lo.  The forward writes
// straight into the peer-major XK exchange layout; the inverse reads it.
//
// Envelope: r_y, r_z, r_t <= 16 (m <= 8 per dim -- every BASELINE config);
// other geometries use the SIMT kernels (dft_yzt.cu).
#include <type_traits>

#include "common.cuh"
#include "tc.cuh"

namespace dfno {

namespace {

constexpr int kThreads = 256;
constexpr int kTileT = 32;                         // t per stage-T K block
// forward operand tiles (bytes)
constexpr int kLboT = 144, kSboT = 1152, kATBytes = 16 * kSboT;
constexpr int kLboZ = 160, kSboZ = 608, kAZBytes = 16 * kSboZ;
constexpr int kLboY = 192, kSboY = 320, kTileYBytes = 16 * kSboY;
constexpr int kAYBytes = 8 * kTileYBytes;          // (re, im) x (hi, lo) x 2 tiles
// inverse operand tiles: 128 rows x K = 16, LBO 128, SBO 528
constexpr int kSbo16 = 528, kTile16 = 16 * kSbo16;
constexpr int kBSbo16 = 512;                       // twiddle B with K = 16
constexpr uint32_t kFwdTmemCols = 256, kInvTmemCols = 512;

__host__ __device__ inline int rup(int a, int b) { return (a + b - 1) / b * b; }

__device__ __forceinline__ int kmaj(int r, int k, int lbo, int sbo) {
  return (r >> 3) * sbo + (k >> 2) * lbo + (r & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ void st_split(unsigned char* hi, unsigned char* lo, int off, float v) {
  float h, l;
  tc::split_rn(v, h, l);
  *reinterpret_cast<float*>(hi + off) = h;
  *reinterpret_cast<float*>(lo + off) = l;
}

// hi / lo of a double-precision twiddle
__device__ __forceinline__ void split_d(double v, float& hi, float& lo) {
  hi = tc::round_tf32((float)v);
  lo = tc::round_tf32((float)(v - (double)hi));
}

__device__ __forceinline__ void sincos_idx(long long k, int n, int N, double& s, double& c) {
  const long long idx = (k * n) % N;
  sincospi(2.0 * (double)idx / N, &s, &c);
}

template <int MODE>
__device__ __forceinline__ float transform(float v, float p, int act) {
  if (MODE == DFNO_SRC_ACT) return act_apply<float>(act, v);
  if (MODE == DFNO_SRC_GRAD) return v * act_deriv<float>(act, p);
  return v;
}

// Twiddle matrix B[n][k] (rows n, K-major, LBO 128) with 4 planes
// (C hi, C lo, S hi, S lo): C = cos(2 pi f(n or k) ...), filled by fn(n, k, c, s).
template <typename F>
__device__ void fill_cs(unsigned char* b, int rows, int kdim, int sbo, F fn) {
  const int plane = (rows / 8) * sbo;
  for (int e = threadIdx.x; e < rows * kdim; e += blockDim.x) {
    const int n = e / kdim, k = e % kdim;
    double c = 0.0, s = 0.0;
    fn(n, k, c, s);
    float ch, cl, sh, sl;
    split_d(c, ch, cl);
    split_d(s, sh, sl);
    const int off = kmaj(n, k, 128, sbo);
    *reinterpret_cast<float*>(b + 0 * plane + off) = ch;
    *reinterpret_cast<float*>(b + 1 * plane + off) = cl;
    *reinterpret_cast<float*>(b + 2 * plane + off) = sh;
    *reinterpret_cast<float*>(b + 3 * plane + off) = sl;
  }
}

// 3xTF32 complex-planar MMA group:  D += A * B  for one K step where
// A = a_{hi,lo}, B = b_{hi,lo}:  hi*hi + lo*hi + hi*lo.
__device__ __forceinline__ void mma3(uint32_t d, uint64_t a_hi, uint64_t a_lo, uint64_t b_hi, uint64_t b_lo,
                                     uint32_t idesc, uint32_t acc) {
  tc::mma_tf32(d, a_hi, b_hi, idesc, acc);
  tc::mma_tf32(d, a_lo, b_hi, idesc, 1u);
  tc::mma_tf32(d, a_hi, b_lo, idesc, 1u);
}

struct FwdLayout {
  int KT, NZ16, NY8, sbo_bt, sbo_bz, sbo_by;
  int off_at, off_az, off_ay, off_bt, off_bz, off_by, total;
};

__host__ __device__ inline FwdLayout fwd_layout(int ny, int nz, int nt) {
  FwdLayout L;
  L.KT = rup(nt, kTileT);
  L.NZ16 = rup(nz, 16);
  L.NY8 = rup(ny, 8);
  L.sbo_bt = (L.KT / 4) * 128;
  L.sbo_bz = (L.NZ16 / 4) * 128;
  L.sbo_by = (L.NY8 / 4) * 128;
  int o = 0;
  L.off_at = o; o += 4 * kATBytes;  // 2 buffers x (hi, lo)
  L.off_az = o; o += 4 * kAZBytes;
  L.off_ay = o; o += kAYBytes;
  L.off_bt = o; o += 2 * 4 * L.sbo_bt;
  L.off_bz = o; o += 4 * 2 * L.sbo_bz;
  L.off_by = o; o += 4 * 2 * L.sbo_by;
  L.total = o;
  return L;
}

// Walks the tiles (slab, y chunk, z block, t block) of one CTA in order.
struct TileCursor {
  int slab, yc, zb, tb;
  long long base;  // element offset of the slab ((b, c, x) slabs are contiguous)
  __device__ void start(int s, long long slab_elems) {
    slab = s;
    yc = zb = tb = 0;
    base = (long long)s * slab_elems;
  }
  __device__ void advance(int n_yc, int n_zb, int n_tb, long long slab_elems) {
    if (++tb < n_tb) return;
    tb = 0;
    if (++zb < n_zb) return;
    zb = 0;
    if (++yc < n_yc) return;
    start(slab + (int)gridDim.x, slab_elems);
  }
};

// (slab, y chunk, z block) group walk
struct GroupCursor {
  int slab, yc, zb;
  __device__ void advance(int n_yc, int n_zb) {
    if (++zb < n_zb) return;
    zb = 0;
    if (++yc < n_yc) return;
    yc = 0;
    slab += (int)gridDim.x;
  }
};

constexpr int kConvWarps = 8, kEpiWarps = 4;
constexpr int kFwdThreads = (kConvWarps + kEpiWarps + 1) * 32;  // + 1 MMA warp

}  // namespace

// ===========================================================================
// forward: warp-specialised
//   warps 0-7  converters : global -> registers (PF tiles ahead) -> act /
//                           grad*act' -> 3xTF32 split -> A_T[2] ring
//   warps 8-11 epilogue   : D1 (TMEM) -> A_Z ; D2 -> A_Y ; D3 -> XK output
//   warp 12    MMA issuer : stage T / Z / Y tcgen05.mma, commits to mbarriers
// Every hand-off is an mbarrier full / empty pair; no block-wide barrier in
// the steady state.
// ===========================================================================
template <int MODE, bool VEC, int PF>
__global__ void __launch_bounds__(kFwdThreads, 1) k_yzt_fwd_tc(const dfno_geom g, const float* __restrict__ src,
                                                               const float* __restrict__ pre, float scale,
                                                               float2* __restrict__ out) {
  constexpr bool GRAD = (MODE == DFNO_SRC_GRAD);
  constexpr int NV = VEC ? 4 : 16;  // loads per converter thread per tile
  using LT = typename std::conditional<VEC, float4, float>::type;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t at_full[2], at_empty[2], d1_full[2], d1_empty[2];
  __shared__ uint64_t az_full, az_empty, d2_full, d2_empty, ay_full, ay_empty, d3_full, d3_empty;
  __shared__ uint32_t tmem_base;

  const int Ny = g.ny, Nz = g.nz, Nt = g.nt;
  const int XL = x_local(g);
  const FwdLayout L = fwd_layout(Ny, Nz, Nt);
  unsigned char* at = smem + L.off_at;
  unsigned char* az = smem + L.off_az;
  unsigned char* ay = smem + L.off_ay;
  unsigned char* bt = smem + L.off_bt;
  unsigned char* bz = smem + L.off_bz;
  unsigned char* by = smem + L.off_by;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- twiddles ---------------------------------------------------------
  {
    const int plane = 4 * L.sbo_bt;  // 32 rows
    for (int e = tid; e < 32 * L.KT; e += blockDim.x) {
      const int n = e / L.KT, t = e % L.KT, kt = n & 15;
      double c = 0.0, s = 0.0;
      if (kt < g.rt && t < Nt) sincos_idx(mode_freq(kt, Nt, g.mt), t, Nt, s, c);
      float hi, lo;
      split_d(n < 16 ? c : -s, hi, lo);
      const int off = kmaj(n, t, 128, L.sbo_bt);
      *reinterpret_cast<float*>(bt + off) = hi;
      *reinterpret_cast<float*>(bt + plane + off) = lo;
    }
  }
  fill_cs(bz, 16, L.NZ16, L.sbo_bz, [&](int n, int z, double& c, double& s) {
    if (n < g.rz && z < Nz) sincos_idx(mode_freq(n, Nz, g.mz), z, Nz, s, c);
  });
  fill_cs(by, 16, L.NY8, L.sbo_by, [&](int n, int y, double& c, double& s) {
    if (n < g.ry && y < Ny) sincos_idx(mode_freq(n, Ny, g.my), y, Ny, s, c);
  });
  if (warp == 0) tc::tmem_alloc<kFwdTmemCols>(&tmem_base);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&at_full[b], kConvWarps * 32);
      tc::mbar_init(&at_empty[b], 1);
      tc::mbar_init(&d1_full[b], 1);
      tc::mbar_init(&d1_empty[b], kEpiWarps * 32);
    }
    tc::mbar_init(&az_full, kEpiWarps * 32);
    tc::mbar_init(&az_empty, 1);
    tc::mbar_init(&d2_full, 1);
    tc::mbar_init(&d2_empty, kEpiWarps * 32);
    tc::mbar_init(&ay_full, kEpiWarps * 32);
    tc::mbar_init(&ay_empty, 1);
    tc::mbar_init(&d3_full, 1);
    tc::mbar_init(&d3_empty, kEpiWarps * 32);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t d2 = tmem + 64, d3 = tmem + 96;  // D1 double buffer at 0 / 32

  const int n_yc = (Ny + 7) / 8, n_zb = (Nz + 15) / 16, n_tb = L.KT / kTileT;
  const int slabs = g.batch * g.c * XL;
  const int my_slabs = (slabs - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int n_groups = my_slabs * n_yc * n_zb;
  const int n_tiles = n_groups * n_tb;
  const long long plane = (long long)Nz * Nt;
  const long long slab_elems = (long long)Ny * plane;

  if (warp < kConvWarps) {
    // ======================= converters =======================
    const int ct = tid;  // 0 .. 255
    const int tt = VEC ? 4 * (ct & 7) : (ct & 31);
    LT buf[PF][NV];
    LT pbuf[GRAD ? PF : 1][GRAD ? NV : 1];
    auto load_tile = [&](const TileCursor& c, LT (&b)[NV], LT (&pb)[GRAD ? NV : 1]) {
      const int y0 = c.yc * 8, z0 = c.zb * 16, t = c.tb * kTileT + tt;
      const bool t_ok = t < Nt;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        // VEC:    row = (ct >> 3) + 32 j -> y = (ct >> 7) + 2 j, z = (ct >> 3) & 15
        // scalar: row = (ct >> 5) + 8 j  -> y = j >> 1,          z = (ct >> 5) + 8 (j & 1)
        const int y = VEC ? y0 + (ct >> 7) + 2 * j : y0 + (j >> 1);
        const int z = VEC ? z0 + ((ct >> 3) & 15) : z0 + (ct >> 5) + 8 * (j & 1);
        const bool ok = t_ok && (z < Nz) && (y < Ny);
        const long long off = c.base + (long long)y * plane + (long long)z * Nt + t;
        if constexpr (VEC) {
          b[j] = ok ? __ldg(reinterpret_cast<const float4*>(src + off)) : make_float4(0.f, 0.f, 0.f, 0.f);
          if constexpr (GRAD)
            pb[j] = ok ? __ldg(reinterpret_cast<const float4*>(pre + off)) : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          b[j] = ok ? __ldg(src + off) : 0.f;
          if constexpr (GRAD) pb[j] = ok ? __ldg(pre + off) : 0.f;
        }
      }
    };
    auto convert_tile = [&](LT (&b)[NV], LT (&pb)[GRAD ? NV : 1], unsigned char* hi, unsigned char* lo) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if constexpr (VEC) {
          float4 v = b[j];
          const float4 p = GRAD ? pb[j] : make_float4(0.f, 0.f, 0.f, 0.f);
          v.x = transform<MODE>(v.x, p.x, g.act);
          v.y = transform<MODE>(v.y, p.y, g.act);
          v.z = transform<MODE>(v.z, p.z, g.act);
          v.w = transform<MODE>(v.w, p.w, g.act);
          float4 h, l;
          tc::split_hl(v.x, h.x, l.x);
          tc::split_hl(v.y, h.y, l.y);
          tc::split_hl(v.z, h.z, l.z);
          tc::split_hl(v.w, h.w, l.w);
          const int row = (ct >> 3) + 32 * j;
          const int off = (row >> 3) * kSboT + (ct & 7) * kLboT + (row & 7) * 16;
          *reinterpret_cast<float4*>(hi + off) = h;
          *reinterpret_cast<float4*>(lo + off) = l;
        } else {
          const float v = transform<MODE>(b[j], GRAD ? pb[j] : 0.f, g.act);
          const int row = (ct >> 5) + 8 * j;
          float h, l;
          tc::split_hl(v, h, l);
          const int off = kmaj(row, ct & 31, kLboT, kSboT);
          *reinterpret_cast<float*>(hi + off) = h;
          *reinterpret_cast<float*>(lo + off) = l;
        }
      }
    };
    TileCursor lc;
    lc.start(blockIdx.x, slab_elems);
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      if (k < n_tiles) {
        if constexpr (GRAD) load_tile(lc, buf[k], pbuf[k]);
        else load_tile(lc, buf[k], pbuf[0]);
        lc.advance(n_yc, n_zb, n_tb, slab_elems);
      }
    }
#pragma unroll 1
    for (int i0 = 0; i0 < n_tiles; i0 += PF) {
#pragma unroll
      for (int k = 0; k < PF; ++k) {
        const int i = i0 + k;
        if (i < n_tiles) {
          const int ab = i & 1;
          tc::mbar_wait(&at_empty[ab], ((i >> 1) & 1) ^ 1);
          unsigned char* hi = at + ab * 2 * kATBytes;
          if constexpr (GRAD) convert_tile(buf[k], pbuf[k], hi, hi + kATBytes);
          else convert_tile(buf[k], pbuf[0], hi, hi + kATBytes);
          if (i + PF < n_tiles) {
            if constexpr (GRAD) load_tile(lc, buf[k], pbuf[k]);
            else load_tile(lc, buf[k], pbuf[0]);
            lc.advance(n_yc, n_zb, n_tb, slab_elems);
          }
          tc::fence_proxy_async();
          tc::mbar_arrive(&at_full[ab]);
        }
      }
    }
  } else if (warp < kConvWarps + kEpiWarps) {
    // ======================= epilogue =======================
    const int quarter = warp & 3;
    const int m = 32 * quarter + lane;  // TMEM lane / operand row
    const uint32_t lane_off = (uint32_t)(32 * quarter) << 16;
    GroupCursor gc{(int)blockIdx.x, 0, 0};
    int chunk = 0, slab_i = 0;
#pragma unroll 1
    for (int G = 0; G < n_groups; ++G) {
      const int d1b = G & 1;
      tc::mbar_wait(&d1_full[d1b], (G >> 1) & 1);
      tc::fence_after();
      float v[32];
      tc::tmem_ld32(tmem + 32 * d1b + lane_off, v);  // row (y, zl): re[kt] 0..15, im[kt] 16..31
      tc::fence_before();
      tc::mbar_arrive(&d1_empty[d1b]);
      tc::mbar_wait(&az_empty, (G & 1) ^ 1);
      {
        const int y = m >> 4, zl = m & 15;
        const int base = (zl >> 2) * kLboZ + y * 16 + (zl & 3) * 4;  // A_Z row = (kt, y), k = zl
#pragma unroll
        for (int kt = 0; kt < 16; ++kt) {
          st_split(az + 0 * kAZBytes, az + 1 * kAZBytes, kt * kSboZ + base, v[kt]);
          st_split(az + 2 * kAZBytes, az + 3 * kAZBytes, kt * kSboZ + base, v[16 + kt]);
        }
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&az_full);
      if (gc.zb == n_zb - 1) {
        // ---- chunk end: D2 -> A_Y
        tc::mbar_wait(&d2_full, chunk & 1);
        tc::fence_after();
        tc::tmem_ld32(d2 + lane_off, v);  // row (kt, y): re[kz] 0..15, im[kz] 16..31
        tc::fence_before();
        tc::mbar_arrive(&d2_empty);
        tc::mbar_wait(&ay_empty, (chunk & 1) ^ 1);
        {
          const int kt = m >> 3, y = m & 7;
          const int base = (kt >> 3) * kSboY + (y >> 2) * kLboY + (kt & 7) * 16 + (y & 3) * 4;
#pragma unroll
          for (int kz = 0; kz < 16; ++kz) {  // A_Y row = (kz % 8, kt) of tile kz / 8, k = y
            const int off = (kz >> 3) * kTileYBytes + (kz & 7) * 2 * kSboY + base;
            st_split(ay + 0 * kTileYBytes, ay + 2 * kTileYBytes, off, v[kz]);
            st_split(ay + 4 * kTileYBytes, ay + 6 * kTileYBytes, off, v[16 + kz]);
          }
        }
        tc::fence_proxy_async();
        tc::mbar_arrive(&ay_full);
        ++chunk;
        if (gc.yc == n_yc - 1) {
          // ---- slab end: D3 -> XK exchange layout
          tc::mbar_wait(&d3_full, slab_i & 1);
          tc::fence_after();
          const int slab = gc.slab, xl = slab % XL, ch = (slab / XL) % g.c, bb = slab / (XL * g.c);
#pragma unroll
          for (int tile = 0; tile < 2; ++tile) {
            tc::tmem_ld32(d3 + 32 * tile + lane_off, v);
            const int kz = 8 * tile + (m >> 4), kt = m & 15;
            if (kz < g.rz && kt < g.rt) {
#pragma unroll
              for (int ky = 0; ky < 16; ++ky)
                if (ky < g.ry)
                  out[xk_row(g, bb, ch, xl, ky) + kz * g.rt + kt] = make_float2(scale * v[ky], scale * v[16 + ky]);
            }
          }
          tc::fence_before();
          tc::mbar_arrive(&d3_empty);
          ++slab_i;
        }
      }
      gc.advance(n_yc, n_zb);
    }
  } else if (lane == 0) {
    // ======================= MMA issuer =======================
    const uint32_t id_t = tc::idesc_tf32(128, 32);
    const uint32_t id16 = tc::idesc_tf32(128, 16);
    const uint32_t id16n = tc::idesc_tf32(128, 16, false, true);
    const uint32_t s_at = tc::smem_u32(at), s_az = tc::smem_u32(az), s_ay = tc::smem_u32(ay);
    const uint32_t s_bt = tc::smem_u32(bt), s_bz = tc::smem_u32(bz), s_by = tc::smem_u32(by);
    GroupCursor gT{(int)blockIdx.x, 0, 0}, gZ = gT, gY = gT;  // groups for the T, Z and Y jobs
    int tile = 0, zchunk = 0, yslab = 0, ygroup = 0;
#pragma unroll 1
    for (int G = 0; G < n_groups + 2; ++G) {
      if (G < n_groups) {
        // ---- stage T for all t blocks of group G -> D1[G & 1]
        const int d1b = G & 1;
        tc::mbar_wait(&d1_empty[d1b], ((G >> 1) & 1) ^ 1);
        for (int tb = 0; tb < n_tb; ++tb, ++tile) {
          const int ab = tile & 1;
          tc::mbar_wait(&at_full[ab], (tile >> 1) & 1);
          tc::fence_after();
          const uint32_t a0 = s_at + ab * 2 * kATBytes;
#pragma unroll
          for (int s = 0; s < kTileT / 8; ++s) {
            const uint32_t ka = 2 * s * kLboT, kb = (uint32_t)(tb * (kTileT / 4) + 2 * s) * 128;
            mma3(tmem + 32 * d1b, tc::desc(a0 + ka, kLboT, kSboT), tc::desc(a0 + kATBytes + ka, kLboT, kSboT),
                 tc::desc(s_bt + kb, 128, L.sbo_bt), tc::desc(s_bt + 4 * L.sbo_bt + kb, 128, L.sbo_bt), id_t,
                 (tb > 0 || s > 0) ? 1u : 0u);
          }
          tc::commit(&at_empty[ab]);
        }
        tc::commit(&d1_full[d1b]);
        gT.advance(n_yc, n_zb);
      }
      // order: Y(G-2) before Z(G-1) -- the epilogue's slab end waits for
      // Y(G-2) before it can hand over A_Z of group G-1
      if (G >= 2 && G - 2 < n_groups) {
        const bool chunk_end = (gY.zb == n_zb - 1);
        if (chunk_end) {
          // ---- stage Y for the chunk that group G - 2 completed -> D3
          tc::mbar_wait(&ay_full, ygroup & 1);
          if (gY.yc == 0) tc::mbar_wait(&d3_empty, (yslab & 1) ^ 1);
          tc::fence_after();
          const uint32_t kb = (uint32_t)(gY.yc * 2) * 128, pl = 2 * L.sbo_by;
          const uint64_t c_h = tc::desc(s_by + 0 * pl + kb, 128, L.sbo_by);
          const uint64_t c_l = tc::desc(s_by + 1 * pl + kb, 128, L.sbo_by);
          const uint64_t s_h = tc::desc(s_by + 2 * pl + kb, 128, L.sbo_by);
          const uint64_t s_l = tc::desc(s_by + 3 * pl + kb, 128, L.sbo_by);
          const uint32_t first = (gY.yc == 0) ? 0u : 1u;
#pragma unroll
          for (int t2 = 0; t2 < 2; ++t2) {
            const uint32_t a0 = s_ay + t2 * kTileYBytes;
            const uint64_t re_h = tc::desc(a0 + 0 * kTileYBytes, kLboY, kSboY);
            const uint64_t re_l = tc::desc(a0 + 2 * kTileYBytes, kLboY, kSboY);
            const uint64_t im_h = tc::desc(a0 + 4 * kTileYBytes, kLboY, kSboY);
            const uint64_t im_l = tc::desc(a0 + 6 * kTileYBytes, kLboY, kSboY);
            const uint32_t dre = d3 + 32 * t2, dim = dre + 16;
            mma3(dre, re_h, re_l, c_h, c_l, id16, first);
            mma3(dre, im_h, im_l, s_h, s_l, id16, 1u);
            mma3(dim, im_h, im_l, c_h, c_l, id16, first);
            mma3(dim, re_h, re_l, s_h, s_l, id16n, 1u);
          }
          tc::commit(&ay_empty);
          ++ygroup;
          if (gY.yc == n_yc - 1) {
            tc::commit(&d3_full);
            ++yslab;
          }
        }
        gY.advance(n_yc, n_zb);
      }
      if (G >= 1 && G - 1 < n_groups) {
        // ---- stage Z for group G - 1 (K block zb) -> D2
        tc::mbar_wait(&az_full, (G - 1) & 1);
        if (gZ.zb == 0) tc::mbar_wait(&d2_empty, (zchunk & 1) ^ 1);
        tc::fence_after();
        const uint32_t pl = 2 * L.sbo_bz;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const uint32_t ka = 2 * s * kLboZ, kb = (uint32_t)(gZ.zb * 4 + 2 * s) * 128;
          const uint64_t re_h = tc::desc(s_az + 0 * kAZBytes + ka, kLboZ, kSboZ);
          const uint64_t re_l = tc::desc(s_az + 1 * kAZBytes + ka, kLboZ, kSboZ);
          const uint64_t im_h = tc::desc(s_az + 2 * kAZBytes + ka, kLboZ, kSboZ);
          const uint64_t im_l = tc::desc(s_az + 3 * kAZBytes + ka, kLboZ, kSboZ);
          const uint64_t c_h = tc::desc(s_bz + 0 * pl + kb, 128, L.sbo_bz);
          const uint64_t c_l = tc::desc(s_bz + 1 * pl + kb, 128, L.sbo_bz);
          const uint64_t s_h = tc::desc(s_bz + 2 * pl + kb, 128, L.sbo_bz);
          const uint64_t s_l = tc::desc(s_bz + 3 * pl + kb, 128, L.sbo_bz);
          const uint32_t first = (gZ.zb == 0 && s == 0) ? 0u : 1u;
          // e^{-i}: re += A_re C + A_im S ;  im += A_im C - A_re S
          mma3(d2, re_h, re_l, c_h, c_l, id16, first);
          mma3(d2, im_h, im_l, s_h, s_l, id16, 1u);
          mma3(d2 + 16, im_h, im_l, c_h, c_l, id16, first);
          mma3(d2 + 16, re_h, re_l, s_h, s_l, id16n, 1u);
        }
        tc::commit(&az_empty);
        if (gZ.zb == n_zb - 1) {
          tc::commit(&d2_full);
          ++zchunk;
        }
        gZ.advance(n_yc, n_zb);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kFwdTmemCols>(tmem);
}

// ===========================================================================
// inverse
// ===========================================================================
struct InvLayout {
  int NY16, NZ16, KT, sbo_by, sbo_bz, sbo_bt;
  int off_v, off_azt, off_by, off_bz, off_bt, total;
};

__host__ __device__ inline InvLayout inv_layout(int ny, int nz, int nt) {
  InvLayout L;
  L.NY16 = rup(ny, 16);
  L.NZ16 = rup(nz, 16);
  L.KT = rup(nt, kTileT);
  int o = 0;
  L.off_v = o;   o += 8 * kTile16;                // V: (re, im) x (hi, lo) x 2 tiles
  L.off_azt = o; o += 8 * kTile16;                // A_Z' then A_T' (aliased)
  L.off_by = o;  o += 4 * (L.NY16 / 8) * kBSbo16;  // rows y, K = ky
  L.off_bz = o;  o += 4 * (L.NZ16 / 8) * kBSbo16;  // rows z, K = kz
  L.off_bt = o;  o += 4 * (L.KT / 8) * kBSbo16;    // rows t, K = kt
  L.total = o;
  return L;
}

__global__ void __launch_bounds__(kThreads, 1) k_yzt_inv_tc(const dfno_geom g, const float2* __restrict__ in,
                                                            float scale, float* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  // one barrier per D3 buffer: a commit is never outstanding twice on the
  // same barrier when it is waited on (phase parity would alias)
  __shared__ uint64_t bar_y, bar_z, bar_t[2];
  __shared__ uint32_t tmem_base;
  const int Ny = g.ny, Nz = g.nz, Nt = g.nt;
  const int XL = x_local(g);
  const InvLayout L = inv_layout(Ny, Nz, Nt);
  unsigned char* av = smem + L.off_v;
  unsigned char* azt = smem + L.off_azt;  // A_Z' (2 tiles) -- later A_T' buffers 0 / 1 (1 tile each)
  unsigned char* by = smem + L.off_by;
  unsigned char* bz = smem + L.off_bz;
  unsigned char* bt = smem + L.off_bt;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, part = warp >> 2;

  fill_cs(by, L.NY16, 16, kBSbo16, [&](int y, int k, double& c, double& s) {
    if (y < Ny && k < g.ry) sincos_idx(mode_freq(k, Ny, g.my), y, Ny, s, c);
  });
  fill_cs(bz, L.NZ16, 16, kBSbo16, [&](int z, int k, double& c, double& s) {
    if (z < Nz && k < g.rz) sincos_idx(mode_freq(k, Nz, g.mz), z, Nz, s, c);
  });
  fill_cs(bt, L.KT, 16, kBSbo16, [&](int t, int k, double& c, double& s) {
    if (t < Nt && k < g.rt) sincos_idx(mode_freq(k, Nt, g.mt), t, Nt, s, c);
  });
  if (warp == 0) tc::tmem_alloc<kInvTmemCols>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&bar_y, 1);
    tc::mbar_init(&bar_z, 1);
    tc::mbar_init(&bar_t[0], 1);
    tc::mbar_init(&bar_t[1], 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t d1 = tmem, d2 = tmem + 64, d3 = tmem + 320;  // D3 double buffer at 320 / 352
  uint32_t ph_y = 0, ph_z = 0, ph_t0 = 0, ph_t1 = 0;
  const uint32_t id16 = tc::idesc_tf32(128, 16), id16n = tc::idesc_tf32(128, 16, false, true);
  const uint32_t id32 = tc::idesc_tf32(128, 32), id32n = tc::idesc_tf32(128, 32, false, true);
  const uint32_t s_av = tc::smem_u32(av), s_azt = tc::smem_u32(azt);
  const uint32_t s_by = tc::smem_u32(by), s_bz = tc::smem_u32(bz), s_bt = tc::smem_u32(bt);
  const uint32_t pl_by = (L.NY16 / 8) * kBSbo16, pl_bz = (L.NZ16 / 8) * kBSbo16, pl_bt = (L.KT / 8) * kBSbo16;
  const int slabs = g.batch * g.c * XL;
  const int n_yc = (Ny + 15) / 16, n_zc = (Nz + 63) / 64, n_tb = L.KT / kTileT;
  const bool vec_out = (Nt % 4 == 0) && (((uintptr_t)out & 15) == 0);
  const long long plane = (long long)Nz * Nt;

  // stage Y' for y chunk yc (reads V, writes D1)
  auto issue_y = [&](int yc) {
    if (tid != 0) return;
    tc::fence_after();
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const uint32_t kb = (uint32_t)(yc * 2) * kBSbo16 + 2 * s * 128;
      const uint64_t c_h = tc::desc(s_by + 0 * pl_by + kb, 128, kBSbo16);
      const uint64_t c_l = tc::desc(s_by + 1 * pl_by + kb, 128, kBSbo16);
      const uint64_t s_h = tc::desc(s_by + 2 * pl_by + kb, 128, kBSbo16);
      const uint64_t s_l = tc::desc(s_by + 3 * pl_by + kb, 128, kBSbo16);
#pragma unroll
      for (int tile = 0; tile < 2; ++tile) {
        const uint32_t a0 = s_av + tile * kTile16 + 2 * s * 128;
        const uint64_t re_h = tc::desc(a0 + 0 * kTile16, 128, kSbo16);
        const uint64_t re_l = tc::desc(a0 + 2 * kTile16, 128, kSbo16);
        const uint64_t im_h = tc::desc(a0 + 4 * kTile16, 128, kSbo16);
        const uint64_t im_l = tc::desc(a0 + 6 * kTile16, 128, kSbo16);
        const uint32_t dre = d1 + 32 * tile, dim = dre + 16, acc = s ? 1u : 0u;
        // e^{+i}: re = A_re C - A_im S ; im = A_im C + A_re S
        mma3(dre, re_h, re_l, c_h, c_l, id16, acc);
        mma3(dre, im_h, im_l, s_h, s_l, id16n, 1u);
        mma3(dim, im_h, im_l, c_h, c_l, id16, acc);
        mma3(dim, re_h, re_l, s_h, s_l, id16, 1u);
      }
    }
    tc::commit(&bar_y);
  };

  for (int slab = blockIdx.x; slab < slabs; slab += gridDim.x) {
    const int xl = slab % XL, ch = (slab / XL) % g.c, bb = slab / (XL * g.c);
    float* o_slab = out + (((long long)bb * g.c + ch) * XL + xl) * (long long)Ny * plane;
    // ---- V (XK layout) -> stage-Y' operand: row (kz % 8, kt) of tile kz / 8, k = ky
    for (int e = tid; e < 16 * 16 * 16; e += kThreads) {
      const int ky = e >> 8, kz = (e >> 4) & 15, kt = e & 15;
      float2 v = make_float2(0.f, 0.f);
      if (ky < g.ry && kz < g.rz && kt < g.rt) v = in[xk_row(g, bb, ch, xl, ky) + kz * g.rt + kt];
      const int off = (kz >> 3) * kTile16 + kmaj((kz & 7) * 16 + kt, ky, 128, kSbo16);
      st_split(av + 0 * kTile16, av + 2 * kTile16, off, v.x);
      st_split(av + 4 * kTile16, av + 6 * kTile16, off, v.y);
    }
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    issue_y(0);
    for (int yc = 0; yc < n_yc; ++yc) {
      for (int zc = 0; zc < n_zc; ++zc) {
        const int nz_c = min(64, L.NZ16 - 64 * zc);
        if (zc > 0) {  // recompute stage Y' for the next z chunk (D1 was consumed)
          issue_y(yc);
        }
        // ---- D1 -> A_Z': row (y % 8, kt) of tile y / 8, k = kz
        tc::mbar_wait(&bar_y, ph_y);
        ph_y ^= 1;
        tc::fence_after();
        {
          float v[32];
          const int tile = part;  // D1 tile = kz / 8
          tc::tmem_ld32(d1 + ((uint32_t)(32 * quarter) << 16) + 32 * tile, v);
          const int m = 32 * quarter + lane, kz = 8 * tile + (m >> 4), kt = m & 15;
#pragma unroll
          for (int y = 0; y < 16; ++y) {
            const int off = (y >> 3) * kTile16 + kmaj((y & 7) * 16 + kt, kz, 128, kSbo16);
            st_split(azt + 0 * kTile16, azt + 2 * kTile16, off, v[y]);
            st_split(azt + 4 * kTile16, azt + 6 * kTile16, off, v[16 + y]);
          }
        }
        tc::fence_proxy_async();
        tc::fence_before();
        __syncthreads();
        // ---- stage Z' (and, early, stage Y' of the next y chunk)
        if (tid == 0) {
          tc::fence_after();
          const uint32_t idn = tc::idesc_tf32(128, nz_c), idnn = tc::idesc_tf32(128, nz_c, false, true);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const uint32_t kb = (uint32_t)(zc * 8) * kBSbo16 + 2 * s * 128;
            const uint64_t c_h = tc::desc(s_bz + 0 * pl_bz + kb, 128, kBSbo16);
            const uint64_t c_l = tc::desc(s_bz + 1 * pl_bz + kb, 128, kBSbo16);
            const uint64_t s_h = tc::desc(s_bz + 2 * pl_bz + kb, 128, kBSbo16);
            const uint64_t s_l = tc::desc(s_bz + 3 * pl_bz + kb, 128, kBSbo16);
#pragma unroll
            for (int tile = 0; tile < 2; ++tile) {
              const uint32_t a0 = s_azt + tile * kTile16 + 2 * s * 128;
              const uint64_t re_h = tc::desc(a0 + 0 * kTile16, 128, kSbo16);
              const uint64_t re_l = tc::desc(a0 + 2 * kTile16, 128, kSbo16);
              const uint64_t im_h = tc::desc(a0 + 4 * kTile16, 128, kSbo16);
              const uint64_t im_l = tc::desc(a0 + 6 * kTile16, 128, kSbo16);
              const uint32_t dre = d2 + 128 * tile, dim = dre + 64, acc = s ? 1u : 0u;
              mma3(dre, re_h, re_l, c_h, c_l, idn, acc);
              mma3(dre, im_h, im_l, s_h, s_l, idnn, 1u);
              mma3(dim, im_h, im_l, c_h, c_l, idn, acc);
              mma3(dim, re_h, re_l, s_h, s_l, idn, 1u);
            }
          }
          tc::commit(&bar_z);
        }
        if (zc == n_zc - 1 && yc + 1 < n_yc) issue_y(yc + 1);
        tc::mbar_wait(&bar_z, ph_z);
        ph_z ^= 1;
        tc::fence_after();
        // ---- stage T' steps over (z block, y tile, t block), software pipelined:
        //      write A_T'[tile] -> MMA into D3[s & 1] -> store D3 of the previous step
        const int n_steps = (nz_c / 16) * 2 * n_tb;
        int prev_y = -1, prev_z = 0, prev_t0 = 0;
        for (int st = 0; st <= n_steps; ++st) {
          if (st < n_steps) {
            const int tb = st % n_tb, tile = (st / n_tb) & 1, zb = st / (2 * n_tb);
            if (tb == 0) {
              // D2 (tile rows (y % 8, kt), cols z of block zb) -> A_T'[tile]: row (y % 8, zl), k = kt
              float v[16];
              const uint32_t a = d2 + ((uint32_t)(32 * quarter) << 16) + 128 * tile + 64 * part + 16 * zb;
              tc::tmem_ld16(a, v);  // part 0: re, part 1: im
              const int m = 32 * quarter + lane, y8 = m >> 4, kt = m & 15;
              unsigned char* hi = azt + tile * 4 * kTile16 + part * 2 * kTile16;
              unsigned char* lo = hi + kTile16;
#pragma unroll
              for (int zl = 0; zl < 16; ++zl) st_split(hi, lo, kmaj(y8 * 16 + zl, kt, 128, kSbo16), v[zl]);
              tc::fence_proxy_async();
            }
            tc::fence_before();
            __syncthreads();
            if (tid == 0) {
              tc::fence_after();
              const uint32_t a0 = s_azt + tile * 4 * kTile16;
              const uint32_t d = d3 + 32 * (st & 1);
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                const uint32_t kb = (uint32_t)(tb * 4) * kBSbo16 + 2 * s * 128;
                const uint64_t c_h = tc::desc(s_bt + 0 * pl_bt + kb, 128, kBSbo16);
                const uint64_t c_l = tc::desc(s_bt + 1 * pl_bt + kb, 128, kBSbo16);
                const uint64_t s_h = tc::desc(s_bt + 2 * pl_bt + kb, 128, kBSbo16);
                const uint64_t s_l = tc::desc(s_bt + 3 * pl_bt + kb, 128, kBSbo16);
                const uint64_t re_h = tc::desc(a0 + 0 * kTile16 + 2 * s * 128, 128, kSbo16);
                const uint64_t re_l = tc::desc(a0 + 1 * kTile16 + 2 * s * 128, 128, kSbo16);
                const uint64_t im_h = tc::desc(a0 + 2 * kTile16 + 2 * s * 128, 128, kSbo16);
                const uint64_t im_l = tc::desc(a0 + 3 * kTile16 + 2 * s * 128, 128, kSbo16);
                mma3(d, re_h, re_l, c_h, c_l, id32, s ? 1u : 0u);
                mma3(d, im_h, im_l, s_h, s_l, id32n, 1u);
              }
              tc::commit(&bar_t[st & 1]);
            }
          }
          if (prev_y >= 0) {
            // ---- store D3 of the previous step: rows (y % 8, zl) -> (y, z), 32 t
            if ((st - 1) & 1) {
              tc::mbar_wait(&bar_t[1], ph_t1);
              ph_t1 ^= 1;
            } else {
              tc::mbar_wait(&bar_t[0], ph_t0);
              ph_t0 ^= 1;
            }
            tc::fence_after();
            if (part == 0) {
              float v[32];
              tc::tmem_ld32(d3 + 32 * ((st - 1) & 1) + ((uint32_t)(32 * quarter) << 16), v);
              const int m = 32 * quarter + lane;
              const int y = prev_y + (m >> 4), z = prev_z + (m & 15);
              if (y < Ny && z < Nz) {
                float* row = o_slab + (long long)y * plane + (long long)z * Nt + prev_t0;
                if (vec_out && prev_t0 + kTileT <= Nt) {
#pragma unroll
                  for (int q = 0; q < 8; ++q)
                    __stcs(reinterpret_cast<float4*>(row + 4 * q),
                           make_float4(scale * v[4 * q], scale * v[4 * q + 1], scale * v[4 * q + 2],
                                       scale * v[4 * q + 3]));
                } else {
#pragma unroll
                  for (int t = 0; t < 32; ++t)
                    if (prev_t0 + t < Nt) row[t] = scale * v[t];
                }
              }
            }
          }
          if (st < n_steps) {
            const int tb = st % n_tb, tile = (st / n_tb) & 1, zb = st / (2 * n_tb);
            prev_y = yc * 16 + tile * 8;
            prev_z = zc * 64 + zb * 16;
            prev_t0 = tb * kTileT;
          }
        }
        tc::fence_before();
        __syncthreads();
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kInvTmemCols>(tmem);
}

// ===========================================================================
// host side
// ===========================================================================
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static bool supported(const dfno_geom& g) {
  return g.dtype == DFNO_F32 && g.ry <= 16 && g.rz <= 16 && g.rt <= 16;
}

static constexpr int kSmemCap = 225 * 1024;

template <int MODE, bool VEC>
static int launch_fwd(const dfno_geom& g, const void* src, const void* pre, double scale, void* out,
                      cudaStream_t st) {
  // tiles held in registers ahead of use by each converter thread
  constexpr int PF = 2;
  const FwdLayout L = fwd_layout(g.ny, g.nz, g.nt);
  if (L.total > kSmemCap) return DFNO_ERR_UNSUPPORTED;
  auto kern = k_yzt_fwd_tc<MODE, VEC, PF>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int slabs = g.batch * g.c * x_local(g);
  const int grid = sm_count() < slabs ? sm_count() : slabs;
  kern<<<grid, kFwdThreads, L.total, st>>>(g, (const float*)src, (const float*)pre, (float)scale, (float2*)out);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

int yzt_fwd_tc(const dfno_geom& g, const void* src, const void* pre, int mode, double scale, void* out,
               cudaStream_t st) {
  if (!supported(g)) return DFNO_ERR_UNSUPPORTED;
  const bool vec = (g.nt % 4 == 0) && ((uintptr_t)src % 16 == 0) && (pre == nullptr || (uintptr_t)pre % 16 == 0);
  switch (mode) {
    case DFNO_SRC_ACT:
      return vec ? launch_fwd<DFNO_SRC_ACT, true>(g, src, pre, scale, out, st)
                 : launch_fwd<DFNO_SRC_ACT, false>(g, src, pre, scale, out, st);
    case DFNO_SRC_GRAD:
      return vec ? launch_fwd<DFNO_SRC_GRAD, true>(g, src, pre, scale, out, st)
                 : launch_fwd<DFNO_SRC_GRAD, false>(g, src, pre, scale, out, st);
    default:
      return vec ? launch_fwd<DFNO_SRC_RAW, true>(g, src, pre, scale, out, st)
                 : launch_fwd<DFNO_SRC_RAW, false>(g, src, pre, scale, out, st);
  }
}

int yzt_inv_tc(const dfno_geom& g, const void* in, double scale, void* out, cudaStream_t st) {
  if (!supported(g)) return DFNO_ERR_UNSUPPORTED;
  const InvLayout L = inv_layout(g.ny, g.nz, g.nt);
  if (L.total > kSmemCap) return DFNO_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(k_yzt_inv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int slabs = g.batch * g.c * x_local(g);
  const int grid = sm_count() < slabs ? sm_count() : slabs;
  k_yzt_inv_tc<<<grid, kThreads, L.total, st>>>(g, (const float2*)in, (float)scale, (float*)out);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

}  // namespace dfno
