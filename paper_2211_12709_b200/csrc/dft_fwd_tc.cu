// Truncated forward (y, z, t) DFT of one rank's x-slab on the tcgen05 tensor
// cores: every contraction runs with its data operand A in TENSOR MEMORY
// (tcgen05.mma ... [d], [a_tmem], b_desc) so the tensor core never re-reads
// the data from shared memory, the twiddles are the small B operand in shared
// memory, and fp32 accuracy comes from 3xTF32 (hi*hi + lo*hi + hi*lo).
//
// Replaces fft_dims(a, (y,z,t)) + truncate_modes (reference d/fno.py:328-329;
// the backward use d/fno.py:446-448 with scale 1/N_yzt).  Output is written
// straight into the peer-major XK exchange layout (include/dfno.h).
//
// Per slab (b, c, x) the input [Ny][Nz][Nt] is walked in groups
// (y chunk of 8, z block of 16) of 128 rows (y, z) x 32 t tiles:
//
//   producer       4-D tensor-map loads (SWIZZLE_128B) of each tile into a
//                  shared-memory ring (src, and pre in backward mode).  TMA
//                  needs 16-byte aligned row starts: for N_t % 4 == 2 (the CO2
//                  grid's N_t = 86) two unswizzled maps load the even and the
//                  odd z rows (row pairs are aligned; the odd map starts two
//                  floats early), 36-float lines read with 8-byte loads; for
//                  odd N_t two warps write the swizzled tiles with 4-byte
//                  cp.async instead, zero-filling outside the grid
//   twiddle warp   builds the stage-Y operand of each y chunk (hi / lo planes,
//                  K = 8 y re | im) from an fp64 phase table into a 2-slot
//                  ring, so no N_y-sized table is resident
//   converters     warps 0-3, thread = tile row (y, z): 8 conflict-free
//                  LDS.128 of its 32 t, act / grad * act' fused, TF32 hi/lo
//                  split, tcgen05.st into A_T (TMEM lane = row, column = t)
//   MMA T          D1[(y,z)][kt re|im]   = A_T . [C | -S]_t            N=32
//   transposers    warps 4-7: D1 -> registers -> per-warp 16x16 shared
//                  transpose -> A_Z[(y,kt)][(re|im, z)] (same TMEM quarter)
//   MMA Z          D2[(y,kt)][kz re|im] += A_Z . [[C,S];[-S,C]]_z      N=32
//                  (accumulated over the z blocks of a y chunk)
//   transposers    D2 -> shared stash -> A_Y[(kz,kt)][(re|im, y)] (2 tiles)
//   MMA Y          D3[(kz,kt)][ky re|im] += A_Y . [[C,S];[-S,C]]_y     N=32
//                  (accumulated over the y chunks of the slab)
//   transposers    D3 -> XK exchange buffer (coalesced float2 stores)
//
// Each hand-off is an mbarrier full/empty pair; A_T, D1, A_Z, D2 are double
// buffered; two issuing threads (stage T; stages Z + Y) keep the tensor pipe
// fed (a single tcgen05.mma issue costs ~50 cycles, measured by
// tests/test_gpu_tc_probe.py).  TMEM: 512 columns, one CTA per SM, persistent
// over slabs.
//
// Envelope: fp32, r_y, r_z, r_t <= 16, inputs aligned to their cp.async piece
// (8 bytes for even N_t, 4 otherwise; 16 for the TMA path), and the resident
// t / z twiddle tables plus a 2-stage ring within shared memory (N_z <= 128 at
// N_t <= 96 in backward mode).
#include <cuda.h>
#include <string.h>

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace dfno {

namespace {

// warp roles
constexpr int kConvW = 8;                 // converters: two sets of 4 (tile parity), one warp per TMEM quarter
constexpr int kTepiW0 = 8;                // warps 8-15: D1 -> A_Z, two sets of 4 (group parity)
constexpr int kZepiW0 = 16;               // warps 16-19: D2 -> A_Y, D3 -> output
constexpr int kTmaW = 20;                 // TMA producer
constexpr int kIssT0 = 21, kIssT1 = 22;   // stage-T issuers (group parity when one t block per group)
constexpr int kIssZ = 23, kIssY = 24;     // stage-Z / stage-Y issuers
constexpr int kTwW = 25;                  // stage-Y twiddle builder
constexpr int kWarps = 26;
constexpr int kThreads2 = kWarps * 32;
constexpr int kTileBytes = 128 * 32 * 4;            // 128 rows x 32 t fp32
// N_t % 4 == 2 (the CO2 grid's 86): even and odd z rows come from two TMA maps
// (no swizzle) with 36-float rows; an odd row's data starts 8 bytes in
constexpr int kPairRow = 36 * 4;
constexpr int kPairHalf = 64 * kPairRow;            // one parity: 8 y x 8 z pairs
constexpr int kPairTile = 2 * kPairHalf;
constexpr int kScratchWarp = 2 * 16 * 17 * 4;       // [yy][kt][z (+1)], one part (re / im) at a time
constexpr int kStashBytes = 2 * 16 * 16 * 9 * 4;    // [part][kz][kt][y (+1)]
constexpr int kAYPlane = 16 * 512;                  // 128 rows x K 16, SBO 512 (one hi or lo plane of one tile)
constexpr int kAYBytes = 4 * kAYPlane;              // 2 tiles x (hi, lo)
constexpr int kBYPlane = 4 * 512;                   // 32 rows x K 16 (8 y re | im), SBO 512
constexpr int kBYSlot = 2 * kBYPlane;               // hi, lo

// TMEM column map (512): A_T 2x64 | D1 2x32 | A_Z 2x64 | D2 2x64 (hi.hi | hi.lo+lo.hi) | D3 2 tiles x 32
constexpr uint32_t cAT = 0, cD1 = 128, cAZ = 192, cD2 = 320, cD3 = 448;

struct Lay {
  int nyc, nzb, ntb;            // y chunks (8), z blocks (16), t blocks (32)
  int kt_tot, kz_tot;           // K extents of the resident twiddle operands
  int sbo_t, sbo_z;
  int off_ring, off_bt, off_bz, off_by, off_ph, off_scr, off_stash, off_ay, total, tile;
  int stages, srcs;             // ring depth, tiles per stage (1 or 2)
};

__host__ __device__ inline Lay make_lay(int ny, int nz, int nt, int srcs, int smem_cap, int tile = kTileBytes) {
  Lay L;
  L.nyc = (ny + 7) / 8;
  L.nzb = (nz + 15) / 16;
  L.ntb = (nt + 31) / 32;
  L.kt_tot = L.ntb * 32;
  L.kz_tot = L.nzb * 32;
  L.sbo_t = (L.kt_tot / 4) * 128;
  L.sbo_z = (L.kz_tot / 4) * 128;
  L.srcs = srcs;
  int o = 0;
  L.off_bt = o; o += 2 * 4 * L.sbo_t;   // hi, lo planes of 32 rows
  L.off_bz = o; o += 2 * 4 * L.sbo_z;
  L.off_by = o; o += 2 * kBYSlot;       // 2-slot ring of per-chunk Y operands
  L.off_ph = o; o += ((16 * ny + 127) / 128) * 128;  // e^{2 pi i j / N_y} as (cos hi, cos lo, sin hi, sin lo)
  L.off_scr = o; o += 8 * kScratchWarp;
  L.off_stash = o; o += kStashBytes;
  o = (o + 1023) & ~1023;
  L.off_ay = o; o += kAYBytes;
  L.off_ring = o;
  const int stage = srcs * tile;
  int s = (smem_cap - o) / stage;
  // up to 4 stages; an odd depth makes a stage alternate between the two
  // converter sets, whose waits then check the stage's previous phase first
  s = s >= 4 ? 4 : (s >= 2 ? s : 0);
  L.stages = s;
  L.tile = tile;
  L.total = o + s * stage;
  return L;
}

__device__ __forceinline__ int kmaj32(int r, int k, int sbo) {
  return (r >> 3) * sbo + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ void put_split(unsigned char* b, int plane, int off, double v) {
  const float hi = tc::round_tf32((float)v);
  const float lo = tc::round_tf32((float)(v - (double)hi));
  *reinterpret_cast<float*>(b + off) = hi;
  *reinterpret_cast<float*>(b + plane + off) = lo;
}

__device__ __forceinline__ void cs(int k, int n, int N, int m, int r, double& c, double& s) {
  c = s = 0.0;
  if (k < r && n < N) {
    const long long idx = ((long long)mode_freq(k, N, m) * n) % N;
    sincospi(2.0 * (double)idx / N, &s, &c);
  }
}

// source conversion of an element pair: act(v), g * act'(pre) or raw
template <int MODE, int ACT>
__device__ __forceinline__ float2 conv2(float2 v, float2 p) {
  if constexpr (MODE == DFNO_SRC_ACT) return act_apply2<ACT>(v);
  if constexpr (MODE == DFNO_SRC_GRAD) return f2mul(v, act_deriv2<ACT>(p));
  return v;
}

// (y chunk, z block) of group G, walked incrementally
struct GroupIdx {
  int yc = 0, zb = 0, slab_g = 0;
  __device__ void next(const Lay& L) {
    if (++zb < L.nzb) return;
    zb = 0;
    if (++yc < L.nyc) return;
    yc = 0;
    ++slab_g;
  }
};

}  // namespace

template <int MODE, int ACT>
__global__ void __launch_bounds__(kThreads2, 1)
    k_yzt_fwd_tc2(const dfno_geom g, const __grid_constant__ CUtensorMap tm_src,
                  const __grid_constant__ CUtensorMap tm_pre, const __grid_constant__ CUtensorMap tm_src_odd,
                  const __grid_constant__ CUtensorMap tm_pre_odd, const float* __restrict__ srcp,
                  const float* __restrict__ prep, int use_ca, int zpair, float scale, float2* __restrict__ out,
                  int smem_cap) {
  constexpr bool GRAD = (MODE == DFNO_SRC_GRAD);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  // full: one barrier per (converter set, stage), so each set sees exactly
  // one phase per tile of its own even when an odd ring depth makes a stage
  // alternate between the sets
  __shared__ uint64_t full[2][4], empty[4], at_full[2], at_empty[2], d1_full[2], d1_empty[2];
  __shared__ uint64_t az_full[2], az_empty[2], d2_full[2], d2_empty[2], ay_full, ay_empty, d3_full, d3_empty;
  __shared__ uint64_t by_full[2], by_empty[2];
  __shared__ uint32_t tmem_base;

  const int Ny = g.ny, Nz = g.nz, Nt = g.nt;
  const int XL = x_local(g);
  const Lay L = make_lay(Ny, Nz, Nt, GRAD ? 2 : 1, smem_cap, zpair ? kPairTile : kTileBytes);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* bt = smem + L.off_bt;
  unsigned char* bz = smem + L.off_bz;
  unsigned char* by = smem + L.off_by;
  unsigned char* ay = smem + L.off_ay;
  float4* ph = reinterpret_cast<float4*>(smem + L.off_ph);

  // ---- twiddle operands (hi / lo planes, K-major, 32 rows each) -----------
  {
    const int pl = 4 * L.sbo_t;  // t: rows 0-15 cos(kt), 16-31 -sin(kt); K = t
    for (int e = tid; e < 32 * L.kt_tot; e += blockDim.x) {
      const int n = e / L.kt_tot, t = e % L.kt_tot;
      double c, s;
      cs(n & 15, t, Nt, g.mt, g.rt, c, s);
      put_split(bt, pl, kmaj32(n, t, L.sbo_t), n < 16 ? c : -s);
    }
    // z / y: realified complex e^{-i}: K = (block, part, index); rows 0-15 out
    // re (C on re, S on im), rows 16-31 out im (-S on re, C on im).  The lo
    // plane sits 32 rows below the hi plane, so one N = 64 descriptor covers
    // [hi | lo] (stage Z stacks them in a single MMA).
    const int plz = 4 * L.sbo_z;
    for (int e = tid; e < 32 * L.kz_tot; e += blockDim.x) {
      const int n = e / L.kz_tot, k = e % L.kz_tot;
      const int z = (k / 32) * 16 + (k & 15), part = (k >> 4) & 1;
      double c, s;
      cs(n & 15, z, Nz, g.mz, g.rz, c, s);
      put_split(bz, plz, kmaj32(n, k, L.sbo_z), (n < 16) ? (part ? s : c) : (part ? c : -s));
    }
    for (int j = tid; j < Ny; j += blockDim.x) {
      double c, s;
      sincospi(2.0 * (double)j / Ny, &s, &c);
      const float ch = tc::round_tf32((float)c), sh = tc::round_tf32((float)s);
      ph[j] = make_float4(ch, tc::round_tf32((float)(c - (double)ch)), sh, tc::round_tf32((float)(s - (double)sh)));
    }
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    for (int s = 0; s < 4; ++s) {
      tc::mbar_init(&full[0][s], use_ca ? 64 : 1);  // cp.async: one arrival per producer lane (2 warps)
      tc::mbar_init(&full[1][s], use_ca ? 64 : 1);
      tc::mbar_init(&empty[s], 128);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&by_full[b], 32);
      tc::mbar_init(&by_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&at_full[b], 128);
      tc::mbar_init(&at_empty[b], 1);
      tc::mbar_init(&d1_full[b], 1);
      tc::mbar_init(&d1_empty[b], 128);  // T-epilogue set b
      tc::mbar_init(&az_full[b], 128);
      tc::mbar_init(&az_empty[b], 1);
      tc::mbar_init(&d2_full[b], 1);
      tc::mbar_init(&d2_empty[b], 128);
    }
    tc::mbar_init(&ay_full, 128);
    tc::mbar_init(&ay_empty, 1);
    tc::mbar_init(&d3_full, 1);
    tc::mbar_init(&d3_empty, 128);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
#ifdef DFNO_WAIT_PROF
  const long long t_start = clock64();
#endif

  const int slabs = g.batch * g.c * XL;
  const int my_slabs = (slabs - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int groups_per_slab = L.nyc * L.nzb;
  const int n_groups = my_slabs * groups_per_slab;
  const int n_tiles = n_groups * L.ntb;
  const int n_chunks = my_slabs * L.nyc;
  const int S = L.stages;
  const bool two_t = (L.ntb == 1);
  const uint32_t quarter_off = (uint32_t)(32 * (warp & 3)) << 16;

  // cp.async producer (N_t % 4 != 0: no legal TMA row stride), run by two warps
  // that split each tile's rows: row r = (y_l, z_l) of 32 t, 16-byte chunk c at
  // c ^ (r & 7) (the TMA SWIZZLE_128B order the converters read), zero fill
  // outside the grid.  `at_chunk(c)` runs when half 1 reaches y chunk c.
  auto cp_async_producer = [&](int half, auto&& at_chunk) {
    GroupIdx gi;
    int tb = 0, chunk = 0;
    const bool even = (Nt & 1) == 0;
    const long long slab_elems = (long long)Ny * Nz * Nt;
    for (int j = 0; j < n_tiles; ++j) {
      if (tb == 0 && gi.zb == 0) at_chunk(chunk++);
      const int s = j % S, n = j / S;
      const long long slab = (long long)blockIdx.x + (long long)gi.slab_g * gridDim.x;
      tc::mbar_wait_lazy(&empty[s], (n & 1) ^ 1, 64);
      unsigned char* dst = smem + L.off_ring + s * L.srcs * L.tile;
#pragma unroll 1
      for (int si = 0; si < L.srcs; ++si) {
        const float* base = (si == 0 ? srcp : prep) + slab * slab_elems;
        const uint32_t d0 = tc::smem_u32(dst + si * kTileBytes);
        if (even) {
          const int jj = lane & 15, rs = lane >> 4, t = tb * 32 + 2 * jj;
          const bool tok = t < Nt;
#pragma unroll 1
          for (int yl = 4 * half; yl < 4 * half + 4; ++yl) {
            const int y = gi.yc * 8 + yl;
            const bool ok_y = tok && y < Ny;
            const float* rowp = base + ((long long)y * Nz + gi.zb * 16) * Nt + t;
#pragma unroll
            for (int zz = 0; zz < 8; ++zz) {
              const int zl = 2 * zz + rs, r = yl * 16 + zl;
              const bool ok = ok_y && gi.zb * 16 + zl < Nz;
              tc::cp_async8(d0 + r * 128 + ((((jj >> 1) ^ (zl & 7))) << 4) + (jj & 1) * 8,
                            ok ? rowp + zl * Nt : base, ok ? 8u : 0u);
            }
          }
        } else {
          const int t = tb * 32 + lane;
          const bool tok = t < Nt;
#pragma unroll 1
          for (int yl = 4 * half; yl < 4 * half + 4; ++yl) {
            const int y = gi.yc * 8 + yl;
            const bool ok_y = tok && y < Ny;
            const float* rowp = base + ((long long)y * Nz + gi.zb * 16) * Nt + t;
#pragma unroll 4
            for (int zl = 0; zl < 16; ++zl) {
              const int r = yl * 16 + zl;
              const bool ok = ok_y && gi.zb * 16 + zl < Nz;
              tc::cp_async4(d0 + r * 128 + (((lane >> 2) ^ (zl & 7)) << 4) + (lane & 3) * 4,
                            ok ? rowp + zl * Nt : base, ok ? 4u : 0u);
            }
          }
        }
      }
      tc::cp_async_mbar_arrive(&full[j & 1][s]);
      if (++tb == L.ntb) {
        tb = 0;
        gi.next(L);
      }
    }
  };
  auto no_chunk = [](int) {};

  if (warp < kConvW) {
    // ======================= converters =======================
    // two sets of 4 warps alternate tiles (measured faster than one set with a
    // deeper ring in both modes)
    constexpr int kSets = 2;
    const int set = warp >> 2, r = 32 * (warp & 3) + lane;  // tile row (y_l, z_l) = TMEM lane
    const int sw = r & 7;
    for (int i = set; set < kSets && i < n_tiles; i += kSets) {
      const int s = i % S, n = i / S;
      // this set's uses of stage s: every fill (even depth) or every other (odd)
      tc::mbar_wait_lazy(&full[set][s], ((S & 1) ? (n >> 1) : n) & 1, 32);
      const unsigned char* ring = smem + L.off_ring + s * L.srcs * L.tile;
      const unsigned char* rowp = ring + r * 128;
      const int b = i & 1;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float h[16], l[16];
        if (zpair) {
          // row (y, z): parity half of the tile, (y, z / 2) line of 36 floats,
          // odd rows 8 bytes in; eight-byte loads (conflict-free: lanes
          // alternate parity, z pairs step the bank by 4)
          const int zl = r & 15;
          const unsigned char* prow = ring + (zl & 1) * kPairHalf + ((r >> 4) * 8 + (zl >> 1)) * kPairRow + (zl & 1) * 8;
#pragma unroll
          for (int c2 = 0; c2 < 8; ++c2) {
            const float2 q = *reinterpret_cast<const float2*>(prow + (16 * half + 2 * c2) * 4);
            float2 pp = make_float2(0.f, 0.f);
            if constexpr (GRAD) pp = *reinterpret_cast<const float2*>(prow + L.tile + (16 * half + 2 * c2) * 4);
            tc::split_hl2(conv2<MODE, ACT>(q, pp), h[2 * c2], h[2 * c2 + 1], l[2 * c2], l[2 * c2 + 1]);
          }
        } else {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int c = 4 * half + c4;
            const float4 q = *reinterpret_cast<const float4*>(rowp + ((c ^ sw) << 4));
            float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
            if constexpr (GRAD) p = *reinterpret_cast<const float4*>(rowp + kTileBytes + ((c ^ sw) << 4));
            const float2 a = conv2<MODE, ACT>(make_float2(q.x, q.y), make_float2(p.x, p.y));
            const float2 bq = conv2<MODE, ACT>(make_float2(q.z, q.w), make_float2(p.z, p.w));
            tc::split_hl2(a, h[4 * c4], h[4 * c4 + 1], l[4 * c4], l[4 * c4 + 1]);
            tc::split_hl2(bq, h[4 * c4 + 2], h[4 * c4 + 3], l[4 * c4 + 2], l[4 * c4 + 3]);
          }
        }
        if (half == 0) tc::mbar_wait(&at_empty[b], ((i >> 1) & 1) ^ 1);
        tc::tmem_st16(tmem + cAT + 64 * b + 16 * half + quarter_off, h);
        tc::tmem_st16(tmem + cAT + 64 * b + 32 + 16 * half + quarter_off, l);
      }
      tc::mbar_arrive(&empty[s]);
      tc::tmem_st_wait();
      tc::fence_before();
      tc::mbar_arrive(&at_full[b]);
    }
  } else if (warp < kZepiW0) {
    // ======================= T epilogue: D1 -> A_Z =======================
    const int set = (warp - kTepiW0) >> 2;
    float* scr = reinterpret_cast<float*>(smem + L.off_scr + (warp - kTepiW0) * kScratchWarp);  // [part][yy][kt][17]
    const int yy = lane >> 4, lo16 = lane & 15;
    for (int G = set; G < n_groups; G += 2) {
      const int b = G & 1;
      tc::mbar_wait(&d1_full[b], (G >> 1) & 1);
      tc::fence_after();
      uint32_t u[32];
      tc::tmem_ld32_nowait(tmem + cD1 + 32 * b + quarter_off, u);
      tc::tmem_ld_wait();
      tc::fence_before();
      tc::mbar_arrive(&d1_empty[b]);
      tc::mbar_wait(&az_empty[b], ((G >> 1) & 1) ^ 1);
      tc::fence_after();
#pragma unroll
      for (int part = 0; part < 2; ++part) {  // A_Z cols: hi re | hi im | lo re | lo im
#pragma unroll
        for (int kt = 0; kt < 16; ++kt) scr[(yy * 16 + kt) * 17 + lo16] = __uint_as_float(u[16 * part + kt]);
        __syncwarp();
        float h[16], l[16];
#pragma unroll
        for (int z = 0; z < 16; z += 2)
          tc::split_hl2(make_float2(scr[(yy * 16 + lo16) * 17 + z], scr[(yy * 16 + lo16) * 17 + z + 1]), h[z],
                        h[z + 1], l[z], l[z + 1]);
        tc::tmem_st16(tmem + cAZ + 64 * b + 16 * part + quarter_off, h);
        tc::tmem_st16(tmem + cAZ + 64 * b + 32 + 16 * part + quarter_off, l);
        __syncwarp();
      }
      tc::tmem_st_wait();
      tc::fence_before();
      tc::mbar_arrive(&az_full[b]);
    }
  } else if (warp < kTmaW) {
    // ======================= Z epilogue: D2 -> A_Y (smem), D3 -> XK =======================
    const int q = warp - kZepiW0;
    float* stash = reinterpret_cast<float*>(smem + L.off_stash);  // [part][kz][kt][9]
    const int yy = lane >> 4, lo16 = lane & 15;
    const int row = 32 * q + lane;  // A_Y / D3 row (kz_l, kt)
    int slab_i = 0;
    for (int c = 0; c < n_chunks; ++c) {
      const int yc = c % L.nyc, cb = c & 1;
      tc::mbar_wait_lazy(&d2_full[cb], (c >> 1) & 1);
      tc::fence_after();
      uint32_t u0[32];
      {
        uint32_t u1[32];
        tc::tmem_ld32_nowait(tmem + cD2 + 64 * cb + quarter_off, u0);
        tc::tmem_ld32_nowait(tmem + cD2 + 64 * cb + 32 + quarter_off, u1);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) u0[j] = __float_as_uint(__uint_as_float(u0[j]) + __uint_as_float(u1[j]));
      }
      tc::fence_before();
      tc::mbar_arrive(&d2_empty[cb]);
      {
        const int yl = 2 * q + yy, kt = lo16;  // D2 row (y_l, kt): hi.hi + (hi.lo + lo.hi)
#pragma unroll
        for (int kz = 0; kz < 16; ++kz) {
          stash[((0 * 16 + kz) * 16 + kt) * 9 + yl] = __uint_as_float(u0[kz]);
          stash[((1 * 16 + kz) * 16 + kt) * 9 + yl] = __uint_as_float(u0[16 + kz]);
        }
      }
      tc::named_sync(1, 128);
      tc::mbar_wait_lazy(&ay_empty, (c & 1) ^ 1);
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        // A_Y tile hh row (kz_l, kt), K = (re y0..7, im y0..7), hi / lo planes,
        // K-major (LBO 128, SBO 512)
        const int kz = 8 * hh + 2 * q + yy, kt = lo16;
        float ah[16], al[16];
#pragma unroll
        for (int y = 0; y < 8; ++y) {
          tc::split_rn(stash[((0 * 16 + kz) * 16 + kt) * 9 + y], ah[y], al[y]);
          tc::split_rn(stash[((1 * 16 + kz) * 16 + kt) * 9 + y], ah[8 + y], al[8 + y]);
        }
        unsigned char* th = ay + (2 * hh) * kAYPlane + (row >> 3) * 512 + (row & 7) * 16;
        unsigned char* tl = th + kAYPlane;
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          *reinterpret_cast<float4*>(th + k4 * 128) = make_float4(ah[4 * k4], ah[4 * k4 + 1], ah[4 * k4 + 2], ah[4 * k4 + 3]);
          *reinterpret_cast<float4*>(tl + k4 * 128) = make_float4(al[4 * k4], al[4 * k4 + 1], al[4 * k4 + 2], al[4 * k4 + 3]);
        }
      }
      tc::named_sync(1, 128);  // stash consumed before the next chunk overwrites it
      tc::fence_proxy_async();
      tc::mbar_arrive(&ay_full);
      if (yc != L.nyc - 1) continue;
      // ---- slab end: D3 -> XK exchange layout
      const int slab = (int)blockIdx.x + slab_i * (int)gridDim.x;
      const int xl = slab % XL, ch = (slab / XL) % g.c, bb = slab / (XL * g.c);
      tc::mbar_wait_lazy(&d3_full, slab_i & 1);
      tc::fence_after();
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        tc::tmem_ld32_nowait(tmem + cD3 + 32 * hh + quarter_off, u0);
        tc::tmem_ld_wait();
        const int kz = 8 * hh + 2 * q + yy, kt = lo16;
        if (kz < g.rz && kt < g.rt) {
#pragma unroll
          for (int ky = 0; ky < 16; ++ky)
            if (ky < g.ry)
              out[xk_row(g, bb, ch, xl, ky) + kz * g.rt + kt] =
                  make_float2(scale * __uint_as_float(u0[ky]), scale * __uint_as_float(u0[16 + ky]));
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&d3_empty);
      ++slab_i;
    }
  } else if (warp == kTmaW) {
    // ======================= producer =======================
    if (!use_ca) {
      if (lane == 0) {
        tc::tma_prefetch_desc(&tm_src);
        if (GRAD) tc::tma_prefetch_desc(&tm_pre);
        if (zpair) {
          tc::tma_prefetch_desc(&tm_src_odd);
          if (GRAD) tc::tma_prefetch_desc(&tm_pre_odd);
        }
        GroupIdx gi;
        int tb = 0;
        for (int j = 0; j < n_tiles; ++j) {
          const int s = j % S, n = j / S;
          const int slab = (int)blockIdx.x + gi.slab_g * (int)gridDim.x;
          tc::mbar_wait_lazy(&empty[s], (n & 1) ^ 1, 64);
          tc::mbar_expect_tx(&full[j & 1][s], L.srcs * L.tile);
          unsigned char* dst = smem + L.off_ring + s * L.srcs * L.tile;
          if (zpair) {  // even z rows, odd z rows (the odd map starts 2 floats early)
            tc::tma_load_4d(dst, &tm_src, tb * 32, gi.zb * 8, gi.yc * 8, slab, &full[j & 1][s]);
            tc::tma_load_4d(dst + kPairHalf, &tm_src_odd, tb * 32, gi.zb * 8, gi.yc * 8, slab, &full[j & 1][s]);
            if (GRAD) {
              tc::tma_load_4d(dst + L.tile, &tm_pre, tb * 32, gi.zb * 8, gi.yc * 8, slab, &full[j & 1][s]);
              tc::tma_load_4d(dst + L.tile + kPairHalf, &tm_pre_odd, tb * 32, gi.zb * 8, gi.yc * 8, slab, &full[j & 1][s]);
            }
          } else {
            tc::tma_load_4d(dst, &tm_src, tb * 32, gi.zb * 16, gi.yc * 8, slab, &full[j & 1][s]);
            if (GRAD) tc::tma_load_4d(dst + kTileBytes, &tm_pre, tb * 32, gi.zb * 16, gi.yc * 8, slab, &full[j & 1][s]);
          }
          if (++tb == L.ntb) {
            tb = 0;
            gi.next(L);
          }
        }
      }
    } else {
      cp_async_producer(0, no_chunk);
    }
  } else if (warp == kTwW) {
    // ======================= stage-Y twiddles (+ half the cp.async rows) =======================
    // rows n: 0-15 out re (C on re, S on im), 16-31 out im (-S on re, C on im);
    // K = (re y0..7, im y0..7) of the chunk; e^{-i}: value from the phase table
    const int ky = lane & 15, y0 = 4 * (lane >> 4);
    const bool ky_ok = ky < g.ry;
    const int f = mode_freq(ky, Ny, g.my);
    auto build = [&](int c) {
      const int yc = c % L.nyc, b = c & 1;
      tc::mbar_wait_lazy(&by_empty[b], ((c >> 1) & 1) ^ 1, 64);
      float* hi = reinterpret_cast<float*>(by + b * kBYSlot);
      float* lo = hi + kBYPlane / 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int yl = y0 + j, y = yc * 8 + yl;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ky_ok && y < Ny) v = ph[(f * y) % Ny];
        // (row, K): (ky, y re) C | (ky, y im) S | (16 + ky, y re) -S | (16 + ky, y im) C
        const int o00 = kmaj32(ky, yl, 512) / 4, o01 = kmaj32(ky, 8 + yl, 512) / 4;
        const int o10 = kmaj32(16 + ky, yl, 512) / 4, o11 = kmaj32(16 + ky, 8 + yl, 512) / 4;
        hi[o00] = v.x; lo[o00] = v.y;
        hi[o01] = v.z; lo[o01] = v.w;
        hi[o10] = -v.z; lo[o10] = -v.w;
        hi[o11] = v.x; lo[o11] = v.y;
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&by_full[b]);
    };
    if (use_ca) {
      cp_async_producer(1, build);
    } else {
      for (int c = 0; c < n_chunks; ++c) build(c);
    }
  } else if (warp == kIssT0 || warp == kIssT1) {
    // ======================= stage T issuers =======================
    const int k = warp - kIssT0;
    if (lane == 0 && (two_t || k == 0)) {
      const uint32_t id = tc::idesc_tf32(128, 32);
      const uint32_t sbt = tc::smem_u32(bt), plt = 4 * L.sbo_t;
      for (int G = two_t ? k : 0; G < n_groups; G += two_t ? 2 : 1) {
        const int b = G & 1;
        tc::mbar_wait(&d1_empty[b], ((G >> 1) & 1) ^ 1);
        for (int tb = 0; tb < L.ntb; ++tb) {
          const int i = G * L.ntb + tb, ab = i & 1;
          tc::mbar_wait(&at_full[ab], (i >> 1) & 1);
          tc::fence_after();
          const uint32_t a = tmem + cAT + 64 * ab, d = tmem + cD1 + 32 * b;
          // lo products first, hi.hi last: the accumulator's adds are not
          // round-to-nearest, so only the hi.hi sums should meet a
          // full-magnitude accumulator
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint32_t kb = (uint32_t)(tb * 4 + s) * 256;
            const uint64_t bh = tc::desc(sbt + kb, 128, L.sbo_t), bl = tc::desc(sbt + plt + kb, 128, L.sbo_t);
            tc::mma_tf32_ts(d, a + 32 + 8 * s, bh, id, (tb | s) ? 1u : 0u);
            tc::mma_tf32_ts(d, a + 8 * s, bl, id, 1u);
          }
#pragma unroll
          for (int s = 0; s < 4; ++s)
            tc::mma_tf32_ts(d, a + 8 * s, tc::desc(sbt + (uint32_t)(tb * 4 + s) * 256, 128, L.sbo_t), id, 1u);
          tc::commit(&at_empty[ab]);
        }
        tc::commit(&d1_full[b]);
      }
    }
  } else if (warp == kIssZ) {
    // ======================= stage Z issuer (hi/lo twiddles stacked, N = 64) ==========
    if (lane == 0) {
      const uint32_t id64 = tc::idesc_tf32(128, 64), id32 = tc::idesc_tf32(128, 32);
      const uint32_t sbz = tc::smem_u32(bz);
      GroupIdx gi;
      int chunk = 0;
      for (int G = 0; G < n_groups; ++G) {
        const int b = G & 1, cb = chunk & 1;
        tc::mbar_wait(&az_full[b], (G >> 1) & 1);
        if (gi.zb == 0) tc::mbar_wait(&d2_empty[cb], ((chunk >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t a = tmem + cAZ + 64 * b, d = tmem + cD2 + 64 * cb;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint64_t bb = tc::desc(sbz + (uint32_t)(gi.zb * 4 + s) * 256, 128, L.sbo_z);
          tc::mma_tf32_ts(d, a + 8 * s, bb, id64, (gi.zb | s) ? 1u : 0u);  // hi.[hi | lo]
          tc::mma_tf32_ts(d + 32, a + 32 + 8 * s, bb, id32, 1u);          // lo.hi, with hi.lo
        }
        tc::commit(&az_empty[b]);
        if (gi.zb == L.nzb - 1) {
          tc::commit(&d2_full[cb]);
          ++chunk;
        }
        gi.next(L);
      }
    }
  } else if (warp == kIssY) {
    // ======================= stage Y issuer (A_Y in shared memory) =======================
    if (lane == 0) {
      const uint32_t id = tc::idesc_tf32(128, 32);
      const uint32_t say = tc::smem_u32(ay);
      int slab_i = 0;
      for (int c = 0; c < n_chunks; ++c) {
        const int yc = c % L.nyc, bb = c & 1;
        const uint32_t sby = tc::smem_u32(by + bb * kBYSlot);
        tc::mbar_wait_lazy(&ay_full, c & 1, 64);
        tc::mbar_wait_lazy(&by_full[bb], (c >> 1) & 1, 32);
        if (yc == 0) tc::mbar_wait_lazy(&d3_empty, (slab_i & 1) ^ 1, 64);
        tc::fence_after();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t d = tmem + cD3 + 32 * hh;
          const uint32_t a_hi = say + (2 * hh) * kAYPlane, a_lo = a_hi + kAYPlane;
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const uint32_t kb = (uint32_t)s * 256;
            const uint64_t bh = tc::desc(sby + kb, 128, 512), bl = tc::desc(sby + kBYPlane + kb, 128, 512);
            const uint64_t ah = tc::desc(a_hi + s * 256, 128, 512), al = tc::desc(a_lo + s * 256, 128, 512);
            tc::mma_tf32(d, ah, bh, id, (yc | s) ? 1u : 0u);
            tc::mma_tf32(d, al, bh, id, 1u);
            tc::mma_tf32(d, ah, bl, id, 1u);
          }
        }
        tc::commit(&ay_empty);
        tc::commit(&by_empty[bb]);
        if (yc == L.nyc - 1) {
          tc::commit(&d3_full);
          ++slab_i;
        }
      }
    }
  }
#ifdef DFNO_WAIT_PROF
  tc::prof_life(t_start);
#endif
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// ===========================================================================
// host side
// ===========================================================================
namespace {

int sm_count2() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int smem_optin() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (n <= 0) n = 227 * 1024;
    n -= 2048 + 1024;  // static shared memory of the kernel, alignment slack
  }
  return n;
}

template <int MODE, int ACT>
int launch2(const dfno_geom& g, const void* src, const void* pre, double scale, void* out, cudaStream_t st) {
  const int cap = smem_optin();
  const int slabs = g.batch * g.c * x_local(g);
  constexpr bool GRADM = MODE == DFNO_SRC_GRAD;
  CUtensorMap ms, mp, ms2, mp2;
  memset(&ms2, 0, sizeof(ms2));
  memset(&mp2, 0, sizeof(mp2));
  const bool al16 = !((uintptr_t)src & 15) && !(pre && ((uintptr_t)pre & 15));
  // 1) N_t % 4 == 0: one 128B-swizzled map per source; 2) N_t % 4 == 2, N_z
  // even: even / odd z-row maps (make_slab_pair_maps); 3) otherwise cp.async
  bool tma = g.nt % 4 == 0 && al16 &&
             make_slab_map(&ms, src, g.ny, g.nz, g.nt, slabs, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (tma && GRADM) tma = make_slab_map(&mp, pre, g.ny, g.nz, g.nt, slabs, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  bool pair = !tma && al16 && make_slab_pair_maps(&ms, &ms2, src, g.ny, g.nz, g.nt, slabs);
  if (pair && GRADM) pair = make_slab_pair_maps(&mp, &mp2, pre, g.ny, g.nz, g.nt, slabs);
  const Lay L = make_lay(g.ny, g.nz, g.nt, GRADM ? 2 : 1, cap, pair ? kPairTile : kTileBytes);
  if (L.stages < 2) return DFNO_ERR_UNSUPPORTED;
  if (!tma && !pair) {
    const uintptr_t piece = (g.nt % 2 == 0) ? 7 : 3;
    if (((uintptr_t)src & piece) || (pre && ((uintptr_t)pre & piece))) return DFNO_ERR_UNSUPPORTED;
    memset(&ms, 0, sizeof(ms));
  }
  if (!GRADM || (!tma && !pair)) {
    mp = ms;
    mp2 = ms2;
  }
  auto kern = k_yzt_fwd_tc2<MODE, ACT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total + 1024) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int grid = sm_count2() < slabs ? sm_count2() : slabs;
  kern<<<grid, kThreads2, L.total + 1024, st>>>(g, ms, mp, ms2, mp2, (const float*)src, (const float*)pre,
                                                (tma || pair) ? 0 : 1, pair ? 1 : 0, (float)scale, (float2*)out, cap);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

template <int MODE>
int launch2_act(const dfno_geom& g, const void* src, const void* pre, double scale, void* out, cudaStream_t st) {
  switch (g.act) {
    case DFNO_ACT_GELU: return launch2<MODE, DFNO_ACT_GELU>(g, src, pre, scale, out, st);
    case DFNO_ACT_RELU: return launch2<MODE, DFNO_ACT_RELU>(g, src, pre, scale, out, st);
    default: return launch2<MODE, DFNO_ACT_IDENTITY>(g, src, pre, scale, out, st);
  }
}

}  // namespace

#ifdef DFNO_WAIT_PROF
// diagnostics build only: copy out (and clear) the per-(CTA, warp) wait /
// lifetime cycle counters of the last yzt forward launches
extern "C" int dfno_debug_wait_prof_fwd(unsigned long long* host) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, tc::g_wait_prof, sizeof(tc::g_wait_prof));
  static unsigned long long zero[tc::kProfCtas][tc::kProfWarps][2];
  cudaMemcpyToSymbol(tc::g_wait_prof, zero, sizeof(zero));
  return DFNO_OK;
}
#endif

int yzt_fwd_tc2(const dfno_geom& g, const void* src, const void* pre, int mode, double scale, void* out,
                cudaStream_t st) {
  if (g.dtype != DFNO_F32 || g.ry > 16 || g.rz > 16 || g.rt > 16) return DFNO_ERR_UNSUPPORTED;
  switch (mode) {
    case DFNO_SRC_ACT: return launch2_act<DFNO_SRC_ACT>(g, src, pre, scale, out, st);
    case DFNO_SRC_GRAD: return launch2_act<DFNO_SRC_GRAD>(g, src, pre, scale, out, st);
    default: return launch2<DFNO_SRC_RAW, DFNO_ACT_IDENTITY>(g, src, pre, scale, out, st);
  }
}

}  // namespace dfno
