// Truncated inverse (ky, kz, kt) -> (y, z, t) DFT with real output on the
// tcgen05 tensor cores (kind::tf32, 3xTF32), stage order Y' -> T' -> Z'.
//
// Replaces pad_modes + ifft_dims(yzt) + .real (reference d/fno.py:338-343,
// scale 1/N_yzt) and its backward use (d/fno.py:459-464, scale 1).  The last
// stage contracts kz with the real z output as the MMA N (= 64 per z block),
// so the accumulator rows (y, t) are already the output's contiguous
// dimension and the output epilogue stores straight from TMEM with coalesced
// 128-byte t rows -- no transposes, no alignment rule on the output grid.
//
// Per slab (b, c, x):
//   loader   warp 20: V (16 contiguous (kz, kt) blocks per slab) -> shared, bulk
//            copies one slab ahead
//   twiddle  warp 21: the Y' operand of each 16-y pass (hi / lo planes) from a
//            phase table: all passes built once when shared memory holds them
//            (N_y <= 64), else into a two-slot ring (one slot when short)
//   front    warps 0-3: V -> A_Y (shared), rows (kz, kt) [2 tiles], K = (ky re | ky im)
//   MMA Y'   D_Y[(kz,kt)][y re 16 | y im 16] = A_Y . [[C,-S];[S,C]]_y  (SS, N=32,
//            16 y per pass)
//   front    D_Y -> stash1 -> A_T[(y 8, kz)][(kt re | kt im)] (TMEM) per 8-y chunk
//   MMA T'   per 32-t block tb: D_T[(y,kz)][t re 32 | t im 32] = A_T . [[C,-S];[S,C]]_t
//            (TS, N=64)
//   T epi    warps 4-7 and 22-25 (set h = Z' tile h): D_T -> stash2 ->
//            A_Z[(y 4, t)][(kz re | kz im)] (TMEM), two Z' tiles per (chunk,
//            t block); tile h takes y_l = 2q + h in lane quarter q, rows warp q
//            of set h already holds in D_T, so each warp transposes through its
//            own stash rows (no CTA barrier)
//   MMA Z'   per 64-z block: D_Z[(y,t)][z] = Re(A_Z . e^{+i kz z}) = A_Z . [C ; -S]_z
//            (TS, N=64; two issuers by tile parity)
//   O epi    warps 8-15 (two sets by tile parity): D_Z -> global, one 128-byte
//            t row per (warp, z) (the output scale is folded into B_Z)
// All hand-offs are mbarrier full / empty pairs; TMEM 512 columns, one CTA per
// SM, persistent over slabs.  Every accumulation issues its small lo products
// before the hi.hi products: the accumulator's adds are not round-to-nearest,
// so only the hi.hi sums should meet a full-magnitude accumulator (DESIGN.md
// section 3).
//
// Envelope: fp32, r_y, r_z, r_t <= 16, r_z r_t even, 16-byte aligned input,
// and the resident t / z twiddles (16 KB per 32-t / 64-z block) within shared
// memory (e.g. the CO2 grid's N_t = 86 with N_z = 64, or N_z = 128 with N_t = 32).
#include "common.cuh"
#include "tc.cuh"

namespace dfno {

namespace {

constexpr int wTepi3 = 4;    // warps 4-7
constexpr int wOepi3 = 8;    // warps 8-15, set = (warp - 8) / 4
constexpr int wIssY3 = 16, wIssT3 = 17, wIssZ3 = 18;  // Z': 18, 19
constexpr int wLoad3 = 20, wTw3 = 21;
constexpr int wTepi3b = 22;  // warps 22-25: the second T-epilogue set (Z' tiles h = 1)
constexpr int kWarps3 = 26;
constexpr int kThreads3 = kWarps3 * 32;
constexpr int kAYPlane3 = 16 * 1024;          // 128 rows x K 32 fp32
constexpr int kBYPlane3 = 4 * 1024;           // one pass: 32 rows (re | im, y 16) x K 32
constexpr int kBlk3 = 16 * 1024;              // one t or z block of twiddles: 64 rows x K 32, hi + lo
constexpr int kS1 = 20;                       // stash1 kt pitch (floats)
constexpr int kS2 = 68;                       // stash2 row pitch (floats): 16-byte rows, conflict-free STS.128

// TMEM columns: D_Y 2 x 32 | A_T 64 | D_T 2 x 64 | A_Z 2 x 64 | D_Z 2 x 64
constexpr uint32_t jDY = 0, jAT = 64, jDT = 128, jAZ = 256, jDZ = 384;

struct Lay3 {
  int npass, nyc, ntb, nzo, nby;
  int off_ay, off_by, off_bt, off_bz, off_ph, off_s1, off_s2, off_v, total;
};

__host__ __device__ inline Lay3 make_lay3(int ny, int nz, int nt, int nby) {
  Lay3 L;
  L.nby = nby;
  L.npass = (ny + 15) / 16;
  L.nyc = (ny + 7) / 8;
  L.ntb = (nt + 31) / 32;
  L.nzo = (nz + 63) / 64;
  int o = 0;
  L.off_ay = o; o += 4 * kAYPlane3;      // tile 0 hi, tile 0 lo, tile 1 hi, tile 1 lo
  L.off_by = o; o += nby * 2 * kBYPlane3;  // nby passes, hi | lo each
  L.off_bt = o; o += L.ntb * kBlk3;      // per t block: rows t re 32 | t im 32, hi | lo
  L.off_bz = o; o += L.nzo * kBlk3;      // per z block: rows z 64, hi | lo
  L.off_ph = o; o += ((16 * ny + 1023) / 1024) * 1024;  // e^{2 pi i j / N_y}: cos hi, cos lo, sin hi, sin lo
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

// NT > 0: N_t known at compile time (32 for the 3-D Navier-Stokes grids, 86
// for the CO2 grid), so the output epilogue's z-strided stores use immediate
// offsets; ZFULL: N_z % 64 == 0 (no partial z block).  NT = 0: generic.
template <int NT, bool ZFULL>
__global__ void __launch_bounds__(kThreads3, 1)
    k_yzt_inv_tc3(const dfno_geom g, const float2* __restrict__ in, float* __restrict__ out, float scale, int nby) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t v_full, v_empty, ay_full, ay_empty, dy_full, dy_empty, at_full, at_empty, by_full[2], by_empty[2];
  __shared__ uint64_t dt_full[2], dt_empty[2], az_full[2], az_empty[2], dz_full[2], dz_empty[2];
  __shared__ uint32_t tmem_base;

  const int Ny = g.ny, Nz = g.nz, Nt = NT > 0 ? NT : g.nt;
  constexpr bool FAST = NT == 32;
  const int XL = x_local(g);
  const Lay3 L = make_lay3(Ny, Nz, Nt, nby);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* ay = smem + L.off_ay;
  unsigned char* by = smem + L.off_by;
  unsigned char* bt = smem + L.off_bt;
  unsigned char* bz = smem + L.off_bz;
  float4* ph = reinterpret_cast<float4*>(smem + L.off_ph);

  // ---- resident twiddles (hi / lo planes, K-major) and the y phase table ----
  // B_T block tb: rows (t re 32 | t im 32), K = (kt re | kt im), t = 32 tb + row
  for (int e = tid; e < L.ntb * 64 * 32; e += blockDim.x) {
    const int tb = e / 2048, n = (e / 32) & 63, k = e % 32;
    const int t = 32 * tb + (n & 31), out_im = n >> 5, in_im = k >> 4;
    double c, s;
    csi3(k & 15, t, Nt, g.mt, g.rt, c, s);
    put_split3(bt + tb * kBlk3, 8 * 1024, kmaj3(n, k), out_im ? (in_im ? c : s) : (in_im ? -s : c));
  }
  // B_Z block zo: rows z 64, K = (kz re | kz im): Re(A e^{+i kz z}) = Are C - Aim S;
  // the output scale is folded in (exact for the power-of-two 1 / N_yzt)
  for (int e = tid; e < L.nzo * 64 * 32; e += blockDim.x) {
    const int zo = e / 2048, n = (e / 32) & 63, k = e % 32, in_im = k >> 4;
    double c, s;
    csi3(k & 15, 64 * zo + n, Nz, g.mz, g.rz, c, s);
    put_split3(bz + zo * kBlk3, 8 * 1024, kmaj3(n, k), (double)scale * (in_im ? -s : c));
  }
  for (int j = tid; j < Ny; j += blockDim.x) {
    double c, s;
    sincospi(2.0 * (double)j / Ny, &s, &c);
    const float ch = tc::round_tf32((float)c), sh = tc::round_tf32((float)s);
    ph[j] = make_float4(ch, tc::round_tf32((float)(c - (double)ch)), sh, tc::round_tf32((float)(s - (double)sh)));
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
      tc::mbar_init(&by_full[b], 32);
      tc::mbar_init(&by_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&dt_full[b], 1);
      tc::mbar_init(&dt_empty[b], 256);  // both T-epilogue sets read every D_T
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
#ifdef DFNO_WAIT_PROF
  const long long t_start = clock64();
#endif
  const uint32_t qoff = (uint32_t)(32 * (warp & 3)) << 16;

  const int slabs = g.batch * g.c * XL;
  const int my_slabs = (slabs - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int n_chunks = my_slabs * L.nyc;  // A_T tiles (8 y)
  const int n_units = n_chunks * L.ntb;   // T' tiles (8 y, 32 t)
  const int n_ztiles = 2 * n_units;       // Z' tiles (4 y, 32 t)

  if (warp < wTepi3) {
    // ======================= front: V -> A_Y ; D_Y -> A_T =======================
    const int q = warp, row = tid;
    float* s1 = reinterpret_cast<float*>(smem + L.off_s1);  // [part][y 8][kz 16][kt (kS1)]
    int pass_i = 0, chunk = 0;
    const float2* vs = reinterpret_cast<const float2*>(smem + L.off_v);
    const int rzt = g.rz * g.rt;
    for (int si = 0; si < my_slabs; ++si) {
      tc::mbar_wait_lazy(&ay_empty, (si & 1) ^ 1, 64);
      tc::mbar_wait(&v_full, si & 1);
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
        unsigned char* phi = ay + (2 * hh) * kAYPlane3 + (row >> 3) * 1024 + (row & 7) * 16;
        unsigned char* plo = phi + kAYPlane3;
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          float h4[4], l4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = 4 * k4 + j;
            tc::split_rn(k < 16 ? re[k] : im[k - 16], h4[j], l4[j]);
          }
          *reinterpret_cast<float4*>(phi + k4 * 128) = make_float4(h4[0], h4[1], h4[2], h4[3]);
          *reinterpret_cast<float4*>(plo + k4 * 128) = make_float4(l4[0], l4[1], l4[2], l4[3]);
        }
      }
      tc::mbar_arrive(&v_empty);
      tc::fence_proxy_async();
      tc::mbar_arrive(&ay_full);
      for (int p = 0; p < L.npass; ++p, ++pass_i) {
        tc::mbar_wait(&dy_full, pass_i & 1);
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
          tc::named_sync(1, 128);
          tc::mbar_wait(&at_empty, (chunk & 1) ^ 1);
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
          tc::named_sync(1, 128);  // s1 consumed
        }
      }
    }
  } else if (warp < wOepi3 || warp >= wTepi3b) {
    // ======================= T epilogue: D_T -> A_Z, set h builds Z' tile h =======================
    // Set h (warps 4-7: h = 0, warps 22-25: h = 1) owns A_Z buffer h: its warp
    // in lane quarter q takes the D_T rows y_l = 2q + h (lanes 16h..16h+15 of
    // the quarter), transposes them through its own stash rows and writes A_Z
    // row (y_l = 2q + h, t = lane).  One producer and one consumer (Z' issuer h)
    // per A_Z buffer; both sets read every D_T.
    const int h = warp >= wTepi3b ? 1 : 0, q = warp & 3;
    float* s2 = reinterpret_cast<float*>(smem + L.off_s2) + (4 * h + q) * 16 * kS2;  // [kz 16][c 64], pitch kS2
    const int kz = lane & 15;
    const bool mine = (lane >> 4) == h;
    for (int i = 0; i < n_units; ++i) {
      const int b = i & 1;
      tc::mbar_wait(&dt_full[b], (i >> 1) & 1);
      tc::fence_after();
      float* dst = s2 + kz * kS2;
#pragma unroll
      for (int part = 0; part < 2; ++part) {  // t re | t im
        uint32_t u[32];
        tc::tmem_ld32_nowait(tmem + jDT + 64 * b + 32 * part + qoff, u);
        tc::tmem_ld_wait();
        if (part == 1) {
          tc::fence_before();
          tc::mbar_arrive(&dt_empty[b]);
        }
        if (mine) {
#pragma unroll
          for (int c = 0; c < 32; c += 4)
            *reinterpret_cast<float4*>(dst + 32 * part + c) = make_float4(
                __uint_as_float(u[c]), __uint_as_float(u[c + 1]), __uint_as_float(u[c + 2]), __uint_as_float(u[c + 3]));
        }
      }
      __syncwarp();
      tc::mbar_wait(&az_empty[h], (i & 1) ^ 1);
      tc::fence_after();
      const float* src = s2 + lane;  // A_Z row (y_l = 2q + h, t = lane)
      float hr[32], lr[32];
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        tc::split_hl2(make_float2(src[k * kS2], src[(k + 1) * kS2]), hr[k], hr[k + 1], lr[k], lr[k + 1]);  // kz re
        tc::split_hl2(make_float2(src[k * kS2 + 32], src[(k + 1) * kS2 + 32]), hr[16 + k], hr[17 + k], lr[16 + k],
                      lr[17 + k]);  // kz im
      }
      tc::tmem_st32(tmem + jAZ + 64 * h + qoff, hr);
      tc::tmem_st32(tmem + jAZ + 64 * h + 32 + qoff, lr);
      tc::tmem_st_wait();
      tc::fence_before();
      tc::mbar_arrive(&az_full[h]);
      __syncwarp();  // stash rows consumed
    }
  } else if (warp < wIssY3) {
    // ======================= O epilogue: D_Z -> global =======================
    const int k = (warp - wOepi3) >> 2, yq = warp & 3;
    const long long plane = (long long)Nz * Nt;
    int v = 0;  // D_Z[k] fill count
    for (int zi = k; zi < n_ztiles; zi += 2) {
      const int u = zi >> 1, h = zi & 1;
      const int i = u / L.ntb, tb = u - i * L.ntb;
      const int si = i / L.nyc, yc = i - si * L.nyc;
      const int slab = (int)blockIdx.x + si * (int)gridDim.x;
      const int y = 8 * yc + 2 * yq + h, t = 32 * tb + lane;  // Z' tile h holds y_l = 2q + h in lane quarter q
      float* o = out + ((long long)slab * Ny + y) * plane + t;
      for (int zo = 0; zo < L.nzo; ++zo, ++v) {
        tc::mbar_wait(&dz_full[k], v & 1);
        tc::fence_after();
#pragma unroll
        for (int half = 0; half < 2; ++half) {  // z 0-31, z 32-63 of the block (32 live registers)
          uint32_t w[32];
          tc::tmem_ld32_nowait(tmem + jDZ + 64 * k + 32 * half + qoff, w);
          tc::tmem_ld_wait();
          if (half == 1) {
            tc::fence_before();
            tc::mbar_arrive(&dz_empty[k]);
          }
          if (FAST && Nz == 64) {
            if (y < Ny) {
#pragma unroll
              for (int z = 0; z < 32; ++z) __stcs(o + (32 * half + z) * 32, __uint_as_float(w[z]));
            }
          } else if (NT > 0 && ZFULL) {
            if (y < Ny && t < Nt) {
              float* oz = o + (long long)(64 * zo + 32 * half) * Nt;
#pragma unroll
              for (int z = 0; z < 32; ++z) __stcs(oz + z * Nt, __uint_as_float(w[z]));
            }
          } else if (y < Ny && t < Nt) {
            float* oz = o + (long long)(64 * zo + 32 * half) * Nt;
            const int zn = min(64, Nz - 64 * zo) - 32 * half;
#pragma unroll
            for (int z = 0; z < 32; ++z) {
              if (z < zn) __stcs(oz, __uint_as_float(w[z]));
              oz += Nt;
            }
          }
        }
      }
    }
  } else if (warp == wIssY3) {
    // ======================= MMA Y' (SS, N = 32) =======================
    if (lane == 0) {
      const uint32_t id = tc::idesc_tf32(128, 32);
      const uint32_t say = tc::smem_u32(ay);
      const bool resident = L.nby >= L.npass;  // every pass's operand built once, before the first slab
      int pass_i = 0;
      for (int si = 0; si < my_slabs; ++si) {
        tc::mbar_wait_lazy(&ay_full, si & 1, 64);
        for (int p = 0; p < L.npass; ++p, ++pass_i) {
          const int bs = resident ? p : pass_i % L.nby;
          const uint32_t sby = tc::smem_u32(by + bs * 2 * kBYPlane3);
          tc::mbar_wait(&dy_empty, (pass_i & 1) ^ 1);
          if (!resident) tc::mbar_wait(&by_full[bs], (pass_i / L.nby) & 1);
          else if (pass_i == 0) tc::mbar_wait(&by_full[0], 0);
          tc::fence_after();
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t d = tmem + jDY + 32 * hh;
            const uint32_t ah0 = say + (2 * hh) * kAYPlane3, al0 = ah0 + kAYPlane3;
#pragma unroll
            for (int s = 0; s < 4; ++s) {  // lo products first
              const uint32_t kb = (uint32_t)s * 256;
              tc::mma_tf32(d, tc::desc(al0 + kb, 128, 1024), tc::desc(sby + kb, 128, 1024), id, s ? 1u : 0u);
              tc::mma_tf32(d, tc::desc(ah0 + kb, 128, 1024), tc::desc(sby + kBYPlane3 + kb, 128, 1024), id, 1u);
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) {  // hi.hi last
              const uint32_t kb = (uint32_t)s * 256;
              tc::mma_tf32(d, tc::desc(ah0 + kb, 128, 1024), tc::desc(sby + kb, 128, 1024), id, 1u);
            }
          }
          if (!resident) tc::commit(&by_empty[bs]);
          tc::commit(&dy_full);
        }
        tc::commit(&ay_empty);
      }
    }
  } else if (warp == wIssT3) {
    // ======================= MMA T' (TS, N = 64), one unit per 32-t block =======================
    if (lane == 0) {
      const uint32_t id = tc::idesc_tf32(128, 64);
      const uint32_t sbt0 = tc::smem_u32(bt);
      int u = 0;
      for (int i = 0; i < n_chunks; ++i) {
        tc::mbar_wait(&at_full, i & 1);
        tc::fence_after();
        const uint32_t a = tmem + jAT;
        for (int tb = 0; tb < L.ntb; ++tb, ++u) {
          const int b = u & 1;
          tc::mbar_wait(&dt_empty[b], ((u >> 1) & 1) ^ 1);
          tc::fence_after();
          const uint32_t d = tmem + jDT + 64 * b, sbt = sbt0 + tb * kBlk3;
#pragma unroll
          for (int s = 0; s < 4; ++s) {  // lo products first
            const uint32_t kb = (uint32_t)s * 256;
            tc::mma_tf32_ts(d, a + 32 + 8 * s, tc::desc(sbt + kb, 128, 1024), id, s ? 1u : 0u);
            tc::mma_tf32_ts(d, a + 8 * s, tc::desc(sbt + 8 * 1024 + kb, 128, 1024), id, 1u);
          }
#pragma unroll
          for (int s = 0; s < 4; ++s) tc::mma_tf32_ts(d, a + 8 * s, tc::desc(sbt + (uint32_t)s * 256, 128, 1024), id, 1u);
          tc::commit(&dt_full[b]);
        }
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
  } else if (warp == wTw3) {
    // ======================= Y' twiddles, one 16-y pass at a time =======================
    // rows n = (out re | out im, y 16), K = (ky re | ky im): e^{+i ky y}
    // value: out re: C on re, -S on im; out im: S on re, C on im
    const int ky = lane & 15, y8 = 8 * (lane >> 4);
    const bool ky_ok = ky < g.ry;
    const int f = mode_freq(ky, Ny, g.my);
    auto build = [&](int p, int bs) {
      float* hi = reinterpret_cast<float*>(by + bs * 2 * kBYPlane3);
      float* lo = hi + kBYPlane3 / 4;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int yl = y8 + j, y = 16 * p + yl;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ky_ok && y < Ny) v = ph[(f * y) % Ny];
        const int o_rr = kmaj3(yl, ky) / 4, o_ri = kmaj3(yl, 16 + ky) / 4;
        const int o_ir = kmaj3(16 + yl, ky) / 4, o_ii = kmaj3(16 + yl, 16 + ky) / 4;
        hi[o_rr] = v.x; lo[o_rr] = v.y;
        hi[o_ri] = -v.z; lo[o_ri] = -v.w;
        hi[o_ir] = v.z; lo[o_ir] = v.w;
        hi[o_ii] = v.x; lo[o_ii] = v.y;
      }
    };
    if (L.nby >= L.npass) {  // resident (N_y <= 64 leaves room): the passes are the same for every slab
      for (int p = 0; p < L.npass; ++p) build(p, p);
      tc::fence_proxy_async();
      tc::mbar_arrive(&by_full[0]);
    } else {
      int pass_i = 0;
      for (int si = 0; si < my_slabs; ++si) {
        for (int p = 0; p < L.npass; ++p, ++pass_i) {
          const int bs = pass_i % L.nby;
          tc::mbar_wait_lazy(&by_empty[bs], ((pass_i / L.nby) & 1) ^ 1, 64);
          build(p, bs);
          tc::fence_proxy_async();
          tc::mbar_arrive(&by_full[bs]);
        }
      }
    }
  } else {
    // ======================= MMA Z' (TS, N = 64 per z block), tile parity =======================
    const int k = warp - wIssZ3;
    if (lane == 0) {
      const uint32_t id = tc::idesc_tf32(128, 64);
      const uint32_t sbz0 = tc::smem_u32(bz);
      int v = 0;  // D_Z[k] fill count
      for (int zi = k; zi < n_ztiles; zi += 2) {
        tc::mbar_wait(&az_full[k], (zi >> 1) & 1);
        tc::fence_after();
        const uint32_t a = tmem + jAZ + 64 * k, d = tmem + jDZ + 64 * k;
        for (int zo = 0; zo < L.nzo; ++zo, ++v) {
          tc::mbar_wait(&dz_empty[k], (v & 1) ^ 1);
          tc::fence_after();
          const uint32_t sbz = sbz0 + zo * kBlk3;
#pragma unroll
          for (int s = 0; s < 4; ++s) {  // lo products first
            const uint32_t kb = (uint32_t)s * 256;
            tc::mma_tf32_ts(d, a + 32 + 8 * s, tc::desc(sbz + kb, 128, 1024), id, s ? 1u : 0u);
            tc::mma_tf32_ts(d, a + 8 * s, tc::desc(sbz + 8 * 1024 + kb, 128, 1024), id, 1u);
          }
#pragma unroll
          for (int s = 0; s < 4; ++s) tc::mma_tf32_ts(d, a + 8 * s, tc::desc(sbz + (uint32_t)s * 256, 128, 1024), id, 1u);
          tc::commit(&dz_full[k]);
        }
        tc::commit(&az_empty[k]);
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
    n -= 1024 + 512;  // alignment slack, static shared memory (barriers)
  }
  return n;
}

}  // namespace

#ifdef DFNO_WAIT_PROF
extern "C" int dfno_debug_wait_prof_inv(unsigned long long* host) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, tc::g_wait_prof, sizeof(tc::g_wait_prof));
  static unsigned long long zero[tc::kProfCtas][tc::kProfWarps][2];
  cudaMemcpyToSymbol(tc::g_wait_prof, zero, sizeof(zero));
  return DFNO_OK;
}
#endif

int yzt_inv_tc3(const dfno_geom& g, const void* in, double scale, void* out, cudaStream_t st) {
  if (g.dtype != DFNO_F32 || g.ry > 16 || g.rz > 16 || g.rt > 16) return DFNO_ERR_UNSUPPORTED;
  if ((g.rz * g.rt) % 2 != 0 || ((uintptr_t)in & 15)) return DFNO_ERR_UNSUPPORTED;  // 16-byte bulk copies
  Lay3 L = make_lay3(g.ny, g.nz, g.nt, (g.ny + 15) / 16);  // every Y' pass resident
  if (L.total > smem_cap_3()) L = make_lay3(g.ny, g.nz, g.nt, 2);
  if (L.total > smem_cap_3()) L = make_lay3(g.ny, g.nz, g.nt, 1);
  if (L.total > smem_cap_3()) return DFNO_ERR_UNSUPPORTED;
  const bool zfull = g.nz % 64 == 0;
  auto kern = (g.nt == 32 && zfull)        ? k_yzt_inv_tc3<32, true>
              : (g.nt == 86 && zfull)      ? k_yzt_inv_tc3<86, true>
                                           : k_yzt_inv_tc3<0, false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total + 1024) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int slabs = g.batch * g.c * x_local(g);
  const int grid = sm_count_3() < slabs ? sm_count_3() : slabs;
  kern<<<grid, kThreads3, L.total + 1024, st>>>(g, (const float2*)in, (float*)out, (float)scale, L.nby);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

}  // namespace dfno
