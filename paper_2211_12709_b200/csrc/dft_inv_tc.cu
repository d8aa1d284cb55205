// Truncated inverse (ky, kz, kt) -> (y, z, t) DFT with real output, on the
// tcgen05 tensor cores (kind::tf32, 3xTF32 for fp32 accuracy), data operands
// in TENSOR MEMORY where they are re-laid out between stages.
//
// Replaces pad_modes + ifft_dims(yzt) + .real (reference d/fno.py:338-343,
// scale 1/N_yzt) and its backward use (d/fno.py:459-464, scale 1).  Input is
// the peer-major XK exchange buffer (include/dfno.h); output the real
// (b, c, x, y, z, t) slab, streamed out with TMA tensor stores.
//
// Per slab (b, c, x):
//   front      warps 0-3: V (16^3 complex modes) -> A_Y in shared memory,
//              rows (kz, kt) [2 tiles], K = (ky re | ky im), hi / lo planes
//   MMA Y'     D_Y[(kz,kt)][y re | y im]  = A_Y . [[C,-S];[S,C]]_y   (SS, N=64,
//              32 y per pass)
//   front      D_Y -> shared stash -> A_Z[(y,kt)][(kz re | kz im)] per 8-y chunk
//   MMA Z'     D_Z[(y,kt)][z re | z im]  = A_Z . [[C,-S];[S,C]]_z   (TS, N=32,
//              per 16-z block; two issuers, z-block parity)
//   T epilogue warps 4-11 (two sets): D_Z -> per-warp 16x16 transpose ->
//              A_T[(y,z)][(kt re | kt im)]
//   MMA T'     D_T[(y,z)][t] = Re(A_T . e^{+i kt t}) = A_T . [C ; -S]_t (TS,
//              N=32; two issuers)
//   O epilogue warps 12-19 (two sets): D_T * scale -> swizzled staging ->
//              TMA tensor store of the 8 y x 16 z x 32 t tile
// All hand-offs are mbarrier full / empty pairs; TMEM: 512 columns, one CTA
// per SM, persistent over slabs.
//
// Envelope: fp32, r_y, r_z, r_t <= 16, Nt % 4 == 0, 16-byte aligned output,
// shared memory permitting (the caller falls back to dft_yzt_tc.cu).
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace dfno {

namespace {

// warps 0-3: front
constexpr int wTepi = 4;                    // warps 4-11, set = (warp - 4) / 4
constexpr int wOepi = 12;                   // warps 12-19, set = (warp - 12) / 4
constexpr int wIssY = 20, wIssZ = 21, wIssT = 23;  // Z': 21, 22; T': 23, 24
constexpr int kWarpsI = 25;
constexpr int kThreadsI = kWarpsI * 32;
constexpr int kTile = 128 * 32 * 4;         // 8 y x 16 z x 32 t fp32
constexpr int kAYPlane = 16 * 1024;         // 128 rows x K 32 (SBO 1024): one hi or lo plane of one tile
constexpr int kScrW = 2 * 336 * 4;          // per T-epilogue warp: [yy (stride 336)][z (20)][kt], one part at a time
constexpr int kStash = 2 * 8 * 16 * 20 * 4; // [part][y][kt][kz (20)]

// TMEM columns: D_Y 2 tiles x 64 | A_Z 2 x 64 | D_Z 2 x 32 | A_T 2 x 64 | D_T 2 x 32
constexpr uint32_t iDY = 0, iAZ = 128, iDZ = 256, iAT = 320, iDT = 448;

struct LayI {
  int npass, nyc, nzb, ntb;      // y passes (32), y chunks (8), z blocks (16), t blocks (32)
  int off_ay, off_by, off_bz, off_bt, off_stash, off_scr, off_out, total;
  int by_plane, bz_plane, bt_plane;
};

__host__ __device__ inline LayI make_layi(int ny, int nz, int nt) {
  LayI L;
  L.npass = (ny + 31) / 32;
  L.nyc = (ny + 7) / 8;
  L.nzb = (nz + 15) / 16;
  L.ntb = (nt + 31) / 32;
  L.by_plane = L.npass * 64 / 8 * 1024;   // rows (pass, re|im, y) x K 32
  L.bz_plane = L.nzb * 32 / 8 * 1024;     // rows (block, re|im, z)
  L.bt_plane = L.ntb * 32 / 8 * 1024;     // rows t
  int o = 0;
  L.off_ay = o; o += 4 * kAYPlane;        // tile 0 hi, tile 0 lo, tile 1 hi, tile 1 lo
  L.off_out = o; o += 2 * kTile;          // TMA store staging, one per O-epilogue set (1024-aligned)
  L.off_by = o; o += 2 * L.by_plane;
  L.off_bz = o; o += 2 * L.bz_plane;
  L.off_bt = o; o += 2 * L.bt_plane;
  L.off_stash = o; o += kStash;
  L.off_scr = o; o += 8 * kScrW;
  L.total = o;
  return L;
}

__device__ __forceinline__ int kmaj(int r, int k, int sbo) {
  return (r >> 3) * sbo + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ void put_split(unsigned char* b, int plane, int off, double v) {
  const float hi = tc::round_tf32((float)v);
  const float lo = tc::round_tf32((float)(v - (double)hi));
  *reinterpret_cast<float*>(b + off) = hi;
  *reinterpret_cast<float*>(b + plane + off) = lo;
}

__device__ __forceinline__ void csi(int k, int n, int N, int m, int r, double& c, double& s) {
  c = s = 0.0;
  if (k < r && n < N) {
    const long long idx = ((long long)mode_freq(k, N, m) * n) % N;
    sincospi(2.0 * (double)idx / N, &s, &c);
  }
}

__device__ __forceinline__ void tma_store_4d(const void* tmap, const void* ssrc, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(tmap),
               "r"(tc::smem_u32(ssrc)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace

__global__ void __launch_bounds__(kThreadsI, 1)
    k_yzt_inv_tc2(const dfno_geom g, const float2* __restrict__ in, const __grid_constant__ CUtensorMap tm_out,
                  float scale, unsigned long long* __restrict__ prof) {
  // optional wait profile (debug, DFNO_WAIT_PROFILE=1): per warp, cycles in wait slots 0..3 and total
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
  __shared__ uint64_t ay_full, ay_empty, dy_full, dy_empty, az_full[2], az_empty[2];
  __shared__ uint64_t dz_full[2], dz_empty[2], at_full[2], at_empty[2], dt_full[2], dt_empty[2];
  __shared__ uint32_t tmem_base;

  const int Ny = g.ny, Nz = g.nz, Nt = g.nt;
  const int XL = x_local(g);
  const LayI L = make_layi(Ny, Nz, Nt);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* ay = smem + L.off_ay;
  unsigned char* by = smem + L.off_by;
  unsigned char* bz = smem + L.off_bz;
  unsigned char* bt = smem + L.off_bt;

  // ---- twiddles, e^{+i}: K = (re | im) of the input modes --------------------
  for (int e = tid; e < L.npass * 64 * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    const int y = (n / 64) * 32 + (n & 31), out_im = (n >> 5) & 1, in_im = k >> 4;
    double c, s;
    csi(k & 15, y, Ny, g.my, g.ry, c, s);
    const double v = out_im ? (in_im ? c : s) : (in_im ? -s : c);
    put_split(by, L.by_plane, kmaj(n, k, 1024), v);
  }
  for (int e = tid; e < L.nzb * 32 * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    const int z = (n / 32) * 16 + (n & 15), out_im = (n >> 4) & 1, in_im = k >> 4;
    double c, s;
    csi(k & 15, z, Nz, g.mz, g.rz, c, s);
    const double v = out_im ? (in_im ? c : s) : (in_im ? -s : c);
    put_split(bz, L.bz_plane, kmaj(n, k, 1024), v);
  }
  for (int e = tid; e < L.ntb * 32 * 32; e += blockDim.x) {
    const int t = e / 32, k = e % 32, in_im = k >> 4;  // Re(V e^{+i}) = Vre C - Vim S
    double c, s;
    csi(k & 15, t, Nt, g.mt, g.rt, c, s);
    put_split(bt, L.bt_plane, kmaj(t, k, 1024), in_im ? -s : c);
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&ay_full, 128);
    tc::mbar_init(&ay_empty, 1);
    tc::mbar_init(&dy_full, 1);
    tc::mbar_init(&dy_empty, 128);
    const int nz_iss = L.nzb >= 2 ? 2 : 1;
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&az_full[b], 128);
      tc::mbar_init(&az_empty[b], nz_iss);
      tc::mbar_init(&dz_full[b], 1);
      tc::mbar_init(&dz_empty[b], 128);
      tc::mbar_init(&at_full[b], 128);
      tc::mbar_init(&at_empty[b], 1);
      tc::mbar_init(&dt_full[b], 1);
      tc::mbar_init(&dt_empty[b], 128);
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
  const int n_chunks = my_slabs * L.nyc;

  if (warp < wTepi) {
    // ======================= front: V -> A_Y ; D_Y -> A_Z =======================
    const int q = warp, row = tid;  // A_Y / D_Y row (kz_l, kt) within a tile; TMEM lane
    float* stash = reinterpret_cast<float*>(smem + L.off_stash);  // [part][y_l][kt][20]
    const int yy = lane >> 4, lo16 = lane & 15;
    int pass_i = 0, chunk = 0;
    for (int si = 0; si < my_slabs; ++si) {
      const int slab = (int)blockIdx.x + si * (int)gridDim.x;
      const int xl = slab % XL, ch = (slab / XL) % g.c, bb = slab / (XL * g.c);
      DFNO_W(0, tc::mbar_wait_lazy(&ay_empty, (si & 1) ^ 1, 64));
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        const int kz = 8 * hh + (row >> 4), kt = row & 15;
        float re[16], im[16];
#pragma unroll
        for (int ky = 0; ky < 16; ++ky) {
          float2 v = make_float2(0.f, 0.f);
          if (ky < g.ry && kz < g.rz && kt < g.rt) v = __ldg(in + xk_row(g, bb, ch, xl, ky) + kz * g.rt + kt);
          re[ky] = v.x;
          im[ky] = v.y;
        }
        unsigned char* ph = ay + (2 * hh) * kAYPlane + (row >> 3) * 1024 + (row & 7) * 16;
        unsigned char* pl = ph + kAYPlane;
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
      tc::fence_proxy_async();
      tc::mbar_arrive(&ay_full);
      for (int p = 0; p < L.npass; ++p, ++pass_i) {
        DFNO_W(1, tc::mbar_wait(&dy_full, pass_i & 1));
        tc::fence_after();
        const int nchunk = min(4, L.nyc - 4 * p);
        for (int j = 0; j < nchunk; ++j, ++chunk) {
          // D_Y rows (kz_l, kt) of tile hh, cols re y 8j.. | im y 32+8j..  -> stash[part][y][kt][kz]
          uint32_t u[4][8];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(u[2 * hh][0]), "=r"(u[2 * hh][1]), "=r"(u[2 * hh][2]), "=r"(u[2 * hh][3]),
                  "=r"(u[2 * hh][4]), "=r"(u[2 * hh][5]), "=r"(u[2 * hh][6]), "=r"(u[2 * hh][7])
                : "r"(tmem + iDY + 64 * hh + 8 * j + qoff));
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(u[2 * hh + 1][0]), "=r"(u[2 * hh + 1][1]), "=r"(u[2 * hh + 1][2]), "=r"(u[2 * hh + 1][3]),
                  "=r"(u[2 * hh + 1][4]), "=r"(u[2 * hh + 1][5]), "=r"(u[2 * hh + 1][6]), "=r"(u[2 * hh + 1][7])
                : "r"(tmem + iDY + 64 * hh + 32 + 8 * j + qoff));
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
              stash[((0 * 8 + y) * 16 + kt) * 20 + kz] = __uint_as_float(u[2 * hh][y]);
              stash[((1 * 8 + y) * 16 + kt) * 20 + kz] = __uint_as_float(u[2 * hh + 1][y]);
            }
          }
          DFNO_W(3, tc::named_sync(1, 128));
          const int b = chunk & 1;
          DFNO_W(2, tc::mbar_wait(&az_empty[b], ((chunk >> 1) & 1) ^ 1));
          tc::fence_after();
          {
            const int yl = 2 * q + yy, kt = lo16;  // A_Z row (y_l, kt)
#pragma unroll
            for (int part = 0; part < 2; ++part) {
              const float* src = stash + ((part * 8 + yl) * 16 + kt) * 20;
              float h[16], l[16];
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const float4 v = *reinterpret_cast<const float4*>(src + 4 * c4);
                tc::split_hl(v.x, h[4 * c4], l[4 * c4]);
                tc::split_hl(v.y, h[4 * c4 + 1], l[4 * c4 + 1]);
                tc::split_hl(v.z, h[4 * c4 + 2], l[4 * c4 + 2]);
                tc::split_hl(v.w, h[4 * c4 + 3], l[4 * c4 + 3]);
              }
              tc::tmem_st16(tmem + iAZ + 64 * b + 16 * part + qoff, h);
              tc::tmem_st16(tmem + iAZ + 64 * b + 32 + 16 * part + qoff, l);
            }
          }
          tc::tmem_st_wait();
          tc::fence_before();
          tc::mbar_arrive(&az_full[b]);
          DFNO_W(3, tc::named_sync(1, 128));  // stash consumed
        }
      }
    }
  } else if (warp < wOepi) {
    // ======================= T epilogue: D_Z -> A_T =======================
    const int k = (warp - wTepi) >> 2;
    float* scr = reinterpret_cast<float*>(smem + L.off_scr + (warp - wTepi) * kScrW);
    const int yy = lane >> 4, lo16 = lane & 15;
    int n = 0;
    for (int c = 0; c < n_chunks; ++c) {
      for (int zb = k; zb < L.nzb; zb += 2, ++n) {
        DFNO_W(0, tc::mbar_wait(&dz_full[k], n & 1));
        tc::fence_after();
        uint32_t u[32];
        tc::tmem_ld32_nowait(tmem + iDZ + 32 * k + qoff, u);  // row (y_l, kt): z re 0..15 | z im
        tc::tmem_ld_wait();
        tc::fence_before();
        tc::mbar_arrive(&dz_empty[k]);
        DFNO_W(1, tc::mbar_wait(&at_empty[k], (n & 1) ^ 1));
        tc::fence_after();
#pragma unroll
        for (int part = 0; part < 2; ++part) {  // A_T row (y_l, z_l): kt re | kt im ; hi 0..31, lo 32..63
#pragma unroll
          for (int z = 0; z < 16; ++z) scr[yy * 336 + z * 20 + lo16] = __uint_as_float(u[16 * part + z]);
          __syncwarp();
          const float* src = scr + yy * 336 + lo16 * 20;
          float h[16], l[16];
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 v = *reinterpret_cast<const float4*>(src + 4 * c4);
            tc::split_hl(v.x, h[4 * c4], l[4 * c4]);
            tc::split_hl(v.y, h[4 * c4 + 1], l[4 * c4 + 1]);
            tc::split_hl(v.z, h[4 * c4 + 2], l[4 * c4 + 2]);
            tc::split_hl(v.w, h[4 * c4 + 3], l[4 * c4 + 3]);
          }
          tc::tmem_st16(tmem + iAT + 64 * k + 16 * part + qoff, h);
          tc::tmem_st16(tmem + iAT + 64 * k + 32 + 16 * part + qoff, l);
          __syncwarp();
        }
        tc::tmem_st_wait();
        tc::fence_before();
        tc::mbar_arrive(&at_full[k]);
      }
    }
  } else if (warp < wIssY) {
    // ======================= O epilogue: D_T -> TMA store =======================
    const int k = (warp - wOepi) >> 2, r = 32 * (warp & 3) + lane;  // output row (y_l, z_l)
    unsigned char* stg = smem + L.off_out + k * kTile;
    const bool leader = (warp & 3) == 0 && lane == 0;
    int n = 0;
    for (int c = 0; c < n_chunks; ++c) {
      const int si = c / L.nyc, yc = c % L.nyc;
      const int slab = (int)blockIdx.x + si * (int)gridDim.x;
      for (int zb = k; zb < L.nzb; zb += 2) {
        for (int tb = 0; tb < L.ntb; ++tb, ++n) {
          DFNO_W(0, tc::mbar_wait(&dt_full[k], n & 1));
          tc::fence_after();
          uint32_t u[32];
          tc::tmem_ld32_nowait(tmem + iDT + 32 * k + qoff, u);
          tc::tmem_ld_wait();
          tc::fence_before();
          tc::mbar_arrive(&dt_empty[k]);
          DFNO_W(1, if (leader) bulk_wait_read0(); tc::named_sync(2 + k, 128));  // previous store has read the staging buffer
          unsigned char* rowp = stg + r * 128;
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4)
            *reinterpret_cast<float4*>(rowp + ((c4 ^ (r & 7)) << 4)) =
                make_float4(scale * __uint_as_float(u[4 * c4]), scale * __uint_as_float(u[4 * c4 + 1]),
                            scale * __uint_as_float(u[4 * c4 + 2]), scale * __uint_as_float(u[4 * c4 + 3]));
          tc::fence_proxy_async();
          DFNO_W(2, tc::named_sync(2 + k, 128));
          if (leader) {
            tma_store_4d(&tm_out, stg, tb * 32, zb * 16, yc * 8, slab);
            bulk_commit();
          }
        }
      }
    }
    if (leader) bulk_wait0();
  } else if (warp == wIssY) {
    // ======================= MMA Y' (SS) =======================
    if (lane == 0) {
      const uint32_t id = tc::idesc_tf32(128, 64);
      const uint32_t say = tc::smem_u32(ay), sby = tc::smem_u32(by);
      int pass_i = 0;
      for (int si = 0; si < my_slabs; ++si) {
        DFNO_W(0, tc::mbar_wait_lazy(&ay_full, si & 1, 64));
        for (int p = 0; p < L.npass; ++p, ++pass_i) {
          DFNO_W(1, tc::mbar_wait(&dy_empty, (pass_i & 1) ^ 1));
          tc::fence_after();
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t d = tmem + iDY + 64 * hh;
            const uint32_t ah0 = say + (2 * hh) * kAYPlane, al0 = ah0 + kAYPlane;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const uint32_t kb = (uint32_t)s * 256;
              const uint64_t ah = tc::desc(ah0 + kb, 128, 1024), al = tc::desc(al0 + kb, 128, 1024);
              const uint64_t bh = tc::desc(sby + (uint32_t)p * 8192 + kb, 128, 1024);
              const uint64_t bl = tc::desc(sby + L.by_plane + (uint32_t)p * 8192 + kb, 128, 1024);
              tc::mma_tf32(d, ah, bh, id, s ? 1u : 0u);
              tc::mma_tf32(d, al, bh, id, 1u);
              tc::mma_tf32(d, ah, bl, id, 1u);
            }
          }
          tc::commit(&dy_full);
        }
        tc::commit(&ay_empty);
      }
    }
  } else if (warp < wIssT) {
    // ======================= MMA Z' (TS), z-block parity =======================
    const int k = warp - wIssZ;
    if (lane == 0 && k < L.nzb) {
      const uint32_t id = tc::idesc_tf32(128, 32);
      const uint32_t sbz = tc::smem_u32(bz);
      int n = 0;
      for (int c = 0; c < n_chunks; ++c) {
        const int ab = c & 1;
        DFNO_W(0, tc::mbar_wait(&az_full[ab], (c >> 1) & 1));
        for (int zb = k; zb < L.nzb; zb += 2, ++n) {
          DFNO_W(1, tc::mbar_wait(&dz_empty[k], (n & 1) ^ 1));
          tc::fence_after();
          const uint32_t a = tmem + iAZ + 64 * ab, d = tmem + iDZ + 32 * k;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint32_t kb = (uint32_t)zb * 4096 + s * 256;
            const uint64_t bh = tc::desc(sbz + kb, 128, 1024), bl = tc::desc(sbz + L.bz_plane + kb, 128, 1024);
            tc::mma_tf32_ts(d, a + 8 * s, bh, id, s ? 1u : 0u);
            tc::mma_tf32_ts(d, a + 32 + 8 * s, bh, id, 1u);
            tc::mma_tf32_ts(d, a + 8 * s, bl, id, 1u);
          }
          tc::commit(&dz_full[k]);
        }
        tc::commit(&az_empty[ab]);
      }
    }
  } else {
    // ======================= MMA T' (TS), z-block parity =======================
    const int k = warp - wIssT;
    if (lane == 0 && k < L.nzb) {
      const uint32_t id = tc::idesc_tf32(128, 32);
      const uint32_t sbt = tc::smem_u32(bt);
      int n = 0, m = 0;
      for (int c = 0; c < n_chunks; ++c) {
        for (int zb = k; zb < L.nzb; zb += 2, ++n) {
          DFNO_W(0, tc::mbar_wait(&at_full[k], n & 1));
          for (int tb = 0; tb < L.ntb; ++tb, ++m) {
            DFNO_W(1, tc::mbar_wait(&dt_empty[k], (m & 1) ^ 1));
            tc::fence_after();
            const uint32_t a = tmem + iAT + 64 * k, d = tmem + iDT + 32 * k;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const uint32_t kb = (uint32_t)tb * 4096 + s * 256;
              const uint64_t bh = tc::desc(sbt + kb, 128, 1024), bl = tc::desc(sbt + L.bt_plane + kb, 128, 1024);
              tc::mma_tf32_ts(d, a + 8 * s, bh, id, s ? 1u : 0u);
              tc::mma_tf32_ts(d, a + 32 + 8 * s, bh, id, 1u);
              tc::mma_tf32_ts(d, a + 8 * s, bl, id, 1u);
            }
            tc::commit(&dt_full[k]);
          }
          tc::commit(&at_empty[k]);
        }
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

int sm_count_i() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int smem_cap_i() {
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

int yzt_inv_tc2(const dfno_geom& g, const void* in, double scale, void* out, cudaStream_t st) {
  if (g.dtype != DFNO_F32 || g.ry > 16 || g.rz > 16 || g.rt > 16) return DFNO_ERR_UNSUPPORTED;
  if (g.nt % 4 != 0 || ((uintptr_t)out & 15)) return DFNO_ERR_UNSUPPORTED;
  const LayI L = make_layi(g.ny, g.nz, g.nt);
  if (L.total > smem_cap_i()) return DFNO_ERR_UNSUPPORTED;
  const int slabs = g.batch * g.c * x_local(g);
  CUtensorMap mo;
  if (!make_slab_map(&mo, out, g.ny, g.nz, g.nt, slabs, CU_TENSOR_MAP_L2_PROMOTION_NONE)) return DFNO_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(k_yzt_inv_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total + 1024) !=
      cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int grid = sm_count_i() < slabs ? sm_count_i() : slabs;
  static unsigned long long* prof = nullptr;
  static const bool want_prof = getenv("DFNO_WAIT_PROFILE") && getenv("DFNO_WAIT_PROFILE")[0] == '1';
  if (want_prof && !prof) cudaMalloc(&prof, kWarpsI * 5 * sizeof(unsigned long long));
  if (prof) cudaMemsetAsync(prof, 0, kWarpsI * 5 * sizeof(unsigned long long), st);
  k_yzt_inv_tc2<<<grid, kThreadsI, L.total + 1024, st>>>(g, (const float2*)in, mo, (float)scale, prof);
  DFNO_CUDA_CHECK_LAUNCH();
  if (prof) {  // debug: per-warp wait cycles averaged over CTAs
    unsigned long long h[kWarpsI * 5];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "yzt_inv_tc2: per-CTA avg cycles  [w0 w1 w2 w3 | total]\n");
    for (int w = 0; w < kWarpsI; ++w)
      fprintf(stderr, "  warp %2d: %9.0f %9.0f %9.0f %9.0f | %9.0f\n", w, h[w * 5] / (double)grid,
              h[w * 5 + 1] / (double)grid, h[w * 5 + 2] / (double)grid, h[w * 5 + 3] / (double)grid,
              h[w * 5 + 4] / (double)grid);
  }
  return DFNO_OK;
}

}  // namespace dfno
