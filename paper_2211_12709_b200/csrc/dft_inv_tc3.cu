// Truncated inverse (ky, kz, kt) -> (y, z, t) DFT with real output on the
// tcgen05 tensor cores (kind::tf32, 3xTF32), stage order Y' -> T' -> Z'.
//
// Replaces pad_modes + ifft_dims(yzt) + .real (reference d/fno.py:338-343,
// scale 1/N_yzt) and its backward use (d/fno.py:459-464, scale 1), like
// dft_inv_tc.cu, whose Y' -> Z' -> T' order ends on a real N = N_t = 32 stage
// with 32 output tiles per slab and a per-tile (kt <-> z) transpose.  Here the
// last stage contracts kz with the real z output as the MMA N (= 64): half the
// output tiles, twice the N per MMA, and the accumulator rows (y, t) are
// already the output's contiguous dimension, so the output epilogue stores
// straight from TMEM with coalesced 128-byte rows -- no transposes.
//
// Per slab (b, c, x):
//   loader  warp 20: V (16 contiguous (kz, kt) blocks per slab) -> shared, bulk
//           copies one slab ahead
//   front   warps 0-3: V -> A_Y (shared), rows (kz, kt) [2 tiles], K = (ky re | ky im)
//   MMA Y'  D_Y[(kz,kt)][y re 16 | y im 16] = A_Y . [[C,-S];[S,C]]_y  (SS, N=32,
//           16 y per pass)
//   front   D_Y -> stash1 -> A_T[(y 8, kz)][(kt re | kt im)] (TMEM) per 8-y chunk
//   MMA T'  D_T[(y,kz)][t re 32 | t im 32] = A_T . [[C,-S];[S,C]]_t  (TS, N=64)
//   T epi   warps 4-7: D_T -> stash2 -> A_Z[(y 4, t)][(kz re | kz im)] (TMEM),
//           two Z' tiles per T' tile
//   MMA Z'  D_Z[(y,t)][z] = Re(A_Z . e^{+i kz z}) = A_Z . [C ; -S]_z  (TS, N=64;
//           two issuers by tile parity)
//   O epi   warps 8-15 (two sets by tile parity): D_Z -> global, one 128-byte
//           t row per (warp, z) (the output scale is folded into B_Z)
// All hand-offs are mbarrier full / empty pairs; TMEM 512 columns, one CTA per
// SM, persistent over slabs.
//
// Envelope: fp32, r_y, r_z, r_t <= 16, N_z <= 64, N_t <= 32 (the caller falls
// back to dft_inv_tc.cu otherwise).
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"

namespace dfno {

namespace {

constexpr int wTepi3 = 4;    // warps 4-7
constexpr int wOepi3 = 8;    // warps 8-15, set = (warp - 8) / 4
constexpr int wIssY3 = 16, wIssT3 = 17, wIssZ3 = 18;  // Z': 18, 19
constexpr int wLoad3 = 20;
constexpr int kWarps3 = 21;
constexpr int kThreads3 = kWarps3 * 32;
constexpr int kAYPlane3 = 16 * 1024;          // 128 rows x K 32 fp32
constexpr int kS1 = 20;                       // stash1 kt pitch (floats)
constexpr int kS2 = 65;                       // stash2 row pitch (floats)

// TMEM columns: D_Y 2 x 32 | A_T 64 | D_T 2 x 64 | A_Z 2 x 64 | D_Z 2 x 64
constexpr uint32_t jDY = 0, jAT = 64, jDT = 128, jAZ = 256, jDZ = 384;

struct Lay3 {
  int npass, nyc;
  int off_ay, off_by, off_bt, off_bz, off_s1, off_s2, off_v, total;
  int by_plane;
};

__host__ __device__ inline Lay3 make_lay3(int ny) {
  Lay3 L;
  L.npass = (ny + 15) / 16;
  L.nyc = (ny + 7) / 8;
  L.by_plane = L.npass * 32 / 8 * 1024;  // rows (pass, re|im, y 16) x K 32
  int o = 0;
  L.off_ay = o; o += 4 * kAYPlane3;      // tile 0 hi, tile 0 lo, tile 1 hi, tile 1 lo
  L.off_by = o; o += 2 * L.by_plane;
  L.off_bt = o; o += 2 * 8 * 1024;       // rows t re 32 | t im 32
  L.off_bz = o; o += 2 * 8 * 1024;       // rows z 64
  L.off_s1 = o; o += 2 * 8 * 16 * kS1 * 4;
  L.off_s2 = o; o += ((8 * 16 * kS2 * 4 + 1023) / 1024) * 1024;
  L.off_v = o; o += 16 * 256 * 8;        // a slab's modes [ky][kz][kt] complex (r_z r_t per ky)
  L.total = o;
  return L;
}

__device__ __forceinline__ int kmaj3(int r, int k) { return (r >> 3) * 1024 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4; }

__device__ __forceinline__ void put_split3(unsigned char* b, int plane, int off, double v) {
  const float hi = tc::round_tf32((float)v);
  const float lo = tc::round_tf32((float)(v - (double)hi));
  *reinterpret_cast<float*>(b + off) = hi;
  *reinterpret_cast<float*>(b + plane + off) = lo;
}

__device__ __forceinline__ void csi3(int k, int n, int N, int m, int r, double& c, double& s) {
  c = s = 0.0;
  if (k < r && n < N) {
    const long long idx = ((long long)mode_freq(k, N, m) * n) % N;
    sincospi(2.0 * (double)idx / N, &s, &c);
  }
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&u)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
               : "r"(taddr));
}

}  // namespace

template <bool FAST>  // FAST: N_z == 64 and N_t == 32 (compile-time store offsets)
__global__ void __launch_bounds__(kThreads3, 1)
    k_yzt_inv_tc3(const dfno_geom g, const float2* __restrict__ in, float* __restrict__ out, float scale,
                  unsigned long long* __restrict__ prof) {
  long long wt[4] = {0, 0, 0, 0};
  const long long t_start = clock64();
#define DFNO_W(slot, call)                \
  do {                                    \
    const long long t0_ = clock64();      \
    call;                                 \
    if (prof) wt[slot] += clock64() - t0_; \
  } while (0)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t v_full, v_empty, ay_full, ay_empty, dy_full, dy_empty, at_full, at_empty;
  __shared__ uint64_t dt_full[2], dt_empty[2], az_full[2], az_empty[2], dz_full[2], dz_empty[2];
  __shared__ uint32_t tmem_base;

  const int Ny = g.ny, Nz = g.nz, Nt = g.nt;
  const int XL = x_local(g);
  const Lay3 L = make_lay3(Ny);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* ay = smem + L.off_ay;
  unsigned char* by = smem + L.off_by;
  unsigned char* bt = smem + L.off_bt;
  unsigned char* bz = smem + L.off_bz;

  // ---- twiddles (hi / lo planes, K-major) -----------------------------------
  // B_Y rows (pass, re|im, y 16), K = (ky re | ky im): e^{+i ky y}
  for (int e = tid; e < L.npass * 32 * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    const int y = (n / 32) * 16 + (n & 15), out_im = (n >> 4) & 1, in_im = k >> 4;
    double c, s;
    csi3(k & 15, y, Ny, g.my, g.ry, c, s);
    put_split3(by, L.by_plane, kmaj3(n, k), out_im ? (in_im ? c : s) : (in_im ? -s : c));
  }
  // B_T rows (t re 32 | t im 32), K = (kt re | kt im)
  for (int e = tid; e < 64 * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    const int t = n & 31, out_im = n >> 5, in_im = k >> 4;
    double c, s;
    csi3(k & 15, t, Nt, g.mt, g.rt, c, s);
    put_split3(bt, 8 * 1024, kmaj3(n, k), out_im ? (in_im ? c : s) : (in_im ? -s : c));
  }
  // B_Z rows z 64, K = (kz re | kz im): Re(A e^{+i kz z}) = Are C - Aim S; the
  // output scale is folded in (exact for the power-of-two 1 / N_yzt)
  for (int e = tid; e < 64 * 32; e += blockDim.x) {
    const int z = e / 32, k = e % 32, in_im = k >> 4;
    double c, s;
    csi3(k & 15, z, Nz, g.mz, g.rz, c, s);
    put_split3(bz, 8 * 1024, kmaj3(z, k), (double)scale * (in_im ? -s : c));
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&v_full, 1);
    tc::mbar_init(&v_empty, 128);
    tc::mbar_init(&ay_full, 128);
    tc::mbar_init(&ay_empty, 1);
    tc::mbar_init(&dy_full, 1);
    tc::mbar_init(&dy_empty, 128);
    tc::mbar_init(&at_full, 128);
    tc::mbar_init(&at_empty, 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&dt_full[b], 1);
      tc::mbar_init(&dt_empty[b], 128);
      tc::mbar_init(&az_full[b], 128);
      tc::mbar_init(&az_empty[b], 1);
      tc::mbar_init(&dz_full[b], 1);
      tc::mbar_init(&dz_empty[b], 128);
    }
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t qoff = (uint32_t)(32 * (warp & 3)) << 16;

  const int slabs = g.batch * g.c * XL;
  const int my_slabs = (slabs - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int n_chunks = my_slabs * L.nyc;  // T' tiles (8 y)
  const int n_ztiles = 2 * n_chunks;      // Z' tiles (4 y)

  if (warp < wTepi3) {
    // ======================= front: V -> A_Y ; D_Y -> A_T =======================
    const int q = warp, row = tid;
    float* s1 = reinterpret_cast<float*>(smem + L.off_s1);  // [part][y 8][kz 16][kt (kS1)]
    int pass_i = 0, chunk = 0;
    const float2* vs = reinterpret_cast<const float2*>(smem + L.off_v);
    const int rzt = g.rz * g.rt;
    for (int si = 0; si < my_slabs; ++si) {
      DFNO_W(0, tc::mbar_wait_lazy(&ay_empty, (si & 1) ^ 1, 64));
      DFNO_W(0, tc::mbar_wait(&v_full, si & 1));
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        float re[16], im[16];
        const int kz = 8 * hh + (row >> 4), kt = row & 15;
        const bool ok = kz < g.rz && kt < g.rt;
        const float2* vp = vs + kz * g.rt + kt;
#pragma unroll
        for (int ky = 0; ky < 16; ++ky) {
          const float2 v = (ok && ky < g.ry) ? vp[ky * rzt] : make_float2(0.f, 0.f);
          re[ky] = v.x;
          im[ky] = v.y;
        }
        unsigned char* ph = ay + (2 * hh) * kAYPlane3 + (row >> 3) * 1024 + (row & 7) * 16;
        unsigned char* pl = ph + kAYPlane3;
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          float h4[4], l4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = 4 * k4 + j;
            tc::split_rn(k < 16 ? re[k] : im[k - 16], h4[j], l4[j]);
          }
          *reinterpret_cast<float4*>(ph + k4 * 128) = make_float4(h4[0], h4[1], h4[2], h4[3]);
          *reinterpret_cast<float4*>(pl + k4 * 128) = make_float4(l4[0], l4[1], l4[2], l4[3]);
        }
      }
      tc::mbar_arrive(&v_empty);
      tc::fence_proxy_async();
      tc::mbar_arrive(&ay_full);
      for (int p = 0; p < L.npass; ++p, ++pass_i) {
        DFNO_W(1, tc::mbar_wait(&dy_full, pass_i & 1));
        tc::fence_after();
        const int nchunk = min(2, L.nyc - 2 * p);
        for (int j = 0; j < nchunk; ++j, ++chunk) {
          // D_Y tile hh rows (kz_l, kt), cols y re 8j.. | y im 16+8j..  -> s1[part][y][kz][kt]
          uint32_t u[4][8];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            tmem_ld8(tmem + jDY + 32 * hh + 8 * j + qoff, u[2 * hh]);
            tmem_ld8(tmem + jDY + 32 * hh + 16 + 8 * j + qoff, u[2 * hh + 1]);
          }
          tc::tmem_ld_wait();
          if (j == nchunk - 1) {
            tc::fence_before();
            tc::mbar_arrive(&dy_empty);
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int kz = 8 * hh + (row >> 4), kt = row & 15;
#pragma unroll
            for (int y = 0; y < 8; ++y) {
              s1[((0 * 8 + y) * 16 + kz) * kS1 + kt] = __uint_as_float(u[2 * hh][y]);
              s1[((1 * 8 + y) * 16 + kz) * kS1 + kt] = __uint_as_float(u[2 * hh + 1][y]);
            }
          }
          DFNO_W(3, tc::named_sync(1, 128));
          DFNO_W(2, tc::mbar_wait(&at_empty, (chunk & 1) ^ 1));
          tc::fence_after();
          {
            const int yl = 2 * q + (lane >> 4), kz = lane & 15;  // A_T row (y_l, kz)
#pragma unroll
            for (int part = 0; part < 2; ++part) {
              const float* src = s1 + ((part * 8 + yl) * 16 + kz) * kS1;
              float h[16], l[16];
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const float4 v = *reinterpret_cast<const float4*>(src + 4 * c4);
                tc::split_hl(v.x, h[4 * c4], l[4 * c4]);
                tc::split_hl(v.y, h[4 * c4 + 1], l[4 * c4 + 1]);
                tc::split_hl(v.z, h[4 * c4 + 2], l[4 * c4 + 2]);
                tc::split_hl(v.w, h[4 * c4 + 3], l[4 * c4 + 3]);
              }
              tc::tmem_st16(tmem + jAT + 16 * part + qoff, h);
              tc::tmem_st16(tmem + jAT + 32 + 16 * part + qoff, l);
            }
          }
          tc::tmem_st_wait();
          tc::fence_before();
          tc::mbar_arrive(&at_full);
          DFNO_W(3, tc::named_sync(1, 128));  // s1 consumed
        }
      }
    }
  } else if (warp < wOepi3) {
    // ======================= T epilogue: D_T -> A_Z (two Z' tiles) =======================
    const int q = warp - wTepi3;
    float* s2 = reinterpret_cast<float*>(smem + L.off_s2);  // [y 8][kz 16][c 64 (t re | t im)], pitch kS2
    const int yl = 2 * q + (lane >> 4), kz = lane & 15;      // D_T row
    for (int i = 0; i < n_chunks; ++i) {
      const int b = i & 1;
      DFNO_W(0, tc::mbar_wait(&dt_full[b], (i >> 1) & 1));
      tc::fence_after();
      uint32_t u[64];
      {
        uint32_t (&u0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&u[0]);
        uint32_t (&u1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&u[32]);
        tc::tmem_ld32_nowait(tmem + jDT + 64 * b + qoff, u0);
        tc::tmem_ld32_nowait(tmem + jDT + 64 * b + 32 + qoff, u1);
      }
      tc::tmem_ld_wait();
      tc::fence_before();
      tc::mbar_arrive(&dt_empty[b]);
      float* dst = s2 + (yl * 16 + kz) * kS2;
#pragma unroll
      for (int c = 0; c < 64; ++c) dst[c] = __uint_as_float(u[c]);
      DFNO_W(3, tc::named_sync(2, 128));
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int zi = 2 * i + h, ab = zi & 1;
        DFNO_W(1, tc::mbar_wait(&az_empty[ab], ((zi >> 1) & 1) ^ 1));
        tc::fence_after();
        const float* src = s2 + ((4 * h + q) * 16) * kS2 + lane;  // A_Z row (y_l = 4h + q, t = lane)
        float hr[32], lr[32];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          tc::split_hl(src[k * kS2], hr[k], lr[k]);             // kz re
          tc::split_hl(src[k * kS2 + 32], hr[16 + k], lr[16 + k]);  // kz im
        }
        tc::tmem_st32(tmem + jAZ + 64 * ab + qoff, hr);
        tc::tmem_st32(tmem + jAZ + 64 * ab + 32 + qoff, lr);
        tc::tmem_st_wait();
        tc::fence_before();
        tc::mbar_arrive(&az_full[ab]);
      }
      DFNO_W(3, tc::named_sync(2, 128));  // s2 consumed
    }
  } else if (warp < wIssY3) {
    // ======================= O epilogue: D_Z -> global =======================
    const int k = (warp - wOepi3) >> 2, yq = warp & 3, t = lane;
    const long long plane = (long long)Nz * Nt;
    for (int zi = k; zi < n_ztiles; zi += 2) {
      DFNO_W(0, tc::mbar_wait(&dz_full[k], (zi >> 1) & 1));
      tc::fence_after();
      uint32_t u[64];
      {
        uint32_t (&u0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&u[0]);
        uint32_t (&u1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&u[32]);
        tc::tmem_ld32_nowait(tmem + jDZ + 64 * k + qoff, u0);
        tc::tmem_ld32_nowait(tmem + jDZ + 64 * k + 32 + qoff, u1);
      }
      tc::tmem_ld_wait();
      tc::fence_before();
      tc::mbar_arrive(&dz_empty[k]);
      const int si = zi / (2 * L.nyc), yt = zi % (2 * L.nyc);
      const int slab = (int)blockIdx.x + si * (int)gridDim.x;
      const int y = 4 * yt + yq;
      float* o = out + ((long long)slab * Ny + y) * plane + t;
      if (FAST) {
        if (y < Ny) {
#pragma unroll
          for (int z = 0; z < 64; ++z) __stcs(o + z * 32, __uint_as_float(u[z]));
        }
      } else if (y < Ny && t < Nt) {
#pragma unroll
        for (int z = 0; z < 64; ++z)
          if (z < Nz) __stcs(o + (long long)z * Nt, __uint_as_float(u[z]));
      }
    }
  } else if (warp == wIssY3) {
    // ======================= MMA Y' (SS, N = 32) =======================
    if (lane == 0) {
      const uint32_t id = tc::idesc_tf32(128, 32);
      const uint32_t say = tc::smem_u32(ay), sby = tc::smem_u32(by);
      int pass_i = 0;
      for (int si = 0; si < my_slabs; ++si) {
        DFNO_W(0, tc::mbar_wait_lazy(&ay_full, si & 1, 64));
        for (int p = 0; p < L.npass; ++p, ++pass_i) {
          DFNO_W(1, tc::mbar_wait(&dy_empty, (pass_i & 1) ^ 1));
          tc::fence_after();
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t d = tmem + jDY + 32 * hh;
            const uint32_t ah0 = say + (2 * hh) * kAYPlane3, al0 = ah0 + kAYPlane3;
            // the small lo products first, the hi.hi products last: the
            // accumulator's non-round-to-nearest adds then bias only the
            // last four sums at full magnitude
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const uint32_t kb = (uint32_t)s * 256;
              const uint64_t ah = tc::desc(ah0 + kb, 128, 1024), al = tc::desc(al0 + kb, 128, 1024);
              const uint64_t bh = tc::desc(sby + (uint32_t)p * 4096 + kb, 128, 1024);
              const uint64_t bl = tc::desc(sby + L.by_plane + (uint32_t)p * 4096 + kb, 128, 1024);
              tc::mma_tf32(d, al, bh, id, s ? 1u : 0u);
              tc::mma_tf32(d, ah, bl, id, 1u);
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const uint32_t kb = (uint32_t)s * 256;
              tc::mma_tf32(d, tc::desc(ah0 + kb, 128, 1024), tc::desc(sby + (uint32_t)p * 4096 + kb, 128, 1024), id,
                           1u);
            }
          }
          tc::commit(&dy_full);
        }
        tc::commit(&ay_empty);
      }
    }
  } else if (warp == wIssT3) {
    // ======================= MMA T' (TS, N = 64) =======================
    if (lane == 0) {
      const uint32_t id = tc::idesc_tf32(128, 64);
      const uint32_t sbt = tc::smem_u32(bt);
      for (int i = 0; i < n_chunks; ++i) {
        const int b = i & 1;
        DFNO_W(0, tc::mbar_wait(&at_full, i & 1));
        DFNO_W(1, tc::mbar_wait(&dt_empty[b], ((i >> 1) & 1) ^ 1));
        tc::fence_after();
        const uint32_t a = tmem + jAT, d = tmem + jDT + 64 * b;
#pragma unroll
        for (int s = 0; s < 4; ++s) {  // lo products first, hi.hi last (see the Y' issuer)
          const uint32_t kb = (uint32_t)s * 256;
          const uint64_t bh = tc::desc(sbt + kb, 128, 1024), bl = tc::desc(sbt + 8 * 1024 + kb, 128, 1024);
          tc::mma_tf32_ts(d, a + 32 + 8 * s, bh, id, s ? 1u : 0u);
          tc::mma_tf32_ts(d, a + 8 * s, bl, id, 1u);
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) tc::mma_tf32_ts(d, a + 8 * s, tc::desc(sbt + (uint32_t)s * 256, 128, 1024), id, 1u);
        tc::commit(&dt_full[b]);
        tc::commit(&at_empty);
      }
    }
  } else if (warp == wLoad3) {
    // ======================= loader: V -> shared =======================
    if (lane == 0) {
      const uint32_t blk = (uint32_t)(g.rz * g.rt) * 8;
      unsigned char* vdst = smem + L.off_v;
      for (int si = 0; si < my_slabs; ++si) {
        const int slab = (int)blockIdx.x + si * (int)gridDim.x;
        const int xl = slab % XL, ch = (slab / XL) % g.c, bb = slab / (XL * g.c);
        tc::mbar_wait_lazy(&v_empty, (si & 1) ^ 1, 64);
        tc::mbar_expect_tx(&v_full, blk * g.ry);
        for (int ky = 0; ky < g.ry; ++ky) tc::bulk_load(vdst + ky * blk, in + xk_row(g, bb, ch, xl, ky), blk, &v_full);
      }
    }
  } else {
    // ======================= MMA Z' (TS, N = 64), tile parity =======================
    const int k = warp - wIssZ3;
    if (lane == 0) {
      const uint32_t id = tc::idesc_tf32(128, 64);
      const uint32_t sbz = tc::smem_u32(bz);
      for (int zi = k; zi < n_ztiles; zi += 2) {
        const int ph = (zi >> 1) & 1;
        DFNO_W(0, tc::mbar_wait(&az_full[k], ph));
        DFNO_W(1, tc::mbar_wait(&dz_empty[k], ph ^ 1));
        tc::fence_after();
        const uint32_t a = tmem + jAZ + 64 * k, d = tmem + jDZ + 64 * k;
#pragma unroll
        for (int s = 0; s < 4; ++s) {  // lo products first, hi.hi last (see the Y' issuer)
          const uint32_t kb = (uint32_t)s * 256;
          const uint64_t bh = tc::desc(sbz + kb, 128, 1024), bl = tc::desc(sbz + 8 * 1024 + kb, 128, 1024);
          tc::mma_tf32_ts(d, a + 32 + 8 * s, bh, id, s ? 1u : 0u);
          tc::mma_tf32_ts(d, a + 8 * s, bl, id, 1u);
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) tc::mma_tf32_ts(d, a + 8 * s, tc::desc(sbz + (uint32_t)s * 256, 128, 1024), id, 1u);
        tc::commit(&dz_full[k]);
        tc::commit(&az_empty[k]);
      }
    }
  }
  if (prof && lane == 0) {
    const long long tot = clock64() - t_start;
    for (int i = 0; i < 4; ++i) atomicAdd(prof + warp * 5 + i, (unsigned long long)wt[i]);
    atomicAdd(prof + warp * 5 + 4, (unsigned long long)tot);
  }
#undef DFNO_W
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// ===========================================================================
// host side
// ===========================================================================
namespace {

int sm_count_3() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int smem_cap_3() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (n <= 0) n = 227 * 1024;
    n -= 2048 + 1024;
  }
  return n;
}

}  // namespace

int yzt_inv_tc3(const dfno_geom& g, const void* in, double scale, void* out, cudaStream_t st) {
  if (g.dtype != DFNO_F32 || g.ry > 16 || g.rz > 16 || g.rt > 16) return DFNO_ERR_UNSUPPORTED;
  if (g.nz > 64 || g.nt > 32) return DFNO_ERR_UNSUPPORTED;
  if ((g.rz * g.rt) % 2 != 0 || ((uintptr_t)in & 15)) return DFNO_ERR_UNSUPPORTED;  // 16-byte bulk copies
  const Lay3 L = make_lay3(g.ny);
  if (L.total > smem_cap_3()) return DFNO_ERR_UNSUPPORTED;
  const bool fast = g.nz == 64 && g.nt == 32;
  auto kern = fast ? k_yzt_inv_tc3<true> : k_yzt_inv_tc3<false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total + 1024) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int slabs = g.batch * g.c * x_local(g);
  const int grid = sm_count_3() < slabs ? sm_count_3() : slabs;
  static unsigned long long* prof = nullptr;
  static const bool want_prof = getenv("DFNO_WAIT_PROFILE") && getenv("DFNO_WAIT_PROFILE")[0] == '1';
  if (want_prof && !prof) cudaMalloc(&prof, kWarps3 * 5 * sizeof(unsigned long long));
  if (prof) cudaMemsetAsync(prof, 0, kWarps3 * 5 * sizeof(unsigned long long), st);
  kern<<<grid, kThreads3, L.total + 1024, st>>>(g, (const float2*)in, (float*)out, (float)scale, prof);
  DFNO_CUDA_CHECK_LAUNCH();
  if (prof) {  // debug: per-warp wait cycles averaged over CTAs
    unsigned long long h[kWarps3 * 5];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "yzt_inv_tc3: per-CTA avg cycles  [w0 w1 w2 w3 | total]\n");
    for (int w = 0; w < kWarps3; ++w)
      fprintf(stderr, "  warp %2d: %9.0f %9.0f %9.0f %9.0f | %9.0f\n", w, h[w * 5] / (double)grid,
              h[w * 5 + 1] / (double)grid, h[w * 5 + 2] / (double)grid, h[w * 5 + 3] / (double)grid,
              h[w * 5 + 4] / (double)grid);
  }
  return DFNO_OK;
}

}  // namespace dfno
