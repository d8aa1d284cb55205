// Point-wise channel mix (encoder / decoder) forward and backward.
//
// Forward replaces _mix_layer_forward (reference d/fno.py:286-289):
// einsum_channel_mix (d/tensor.py:210-228) + activation (d/fno.py:41-46).
// Backward replaces the mixer part of fno_backward (d/fno.py:484-486,
// d/fno.py:497-499): g*act'(pre), _mix_weight_grad (d/fno.py:405-406) and
// _mix_input_grad (d/fno.py:409-412).
//
// Both are HBM-streaming kernels: each thread owns VEC consecutive points of
// one batch entry, reads every input channel once with vector loads, keeps the
// (cin x CO) weight tile in shared memory (broadcast reads) and the CO output
// accumulators in registers.  The weight gradient is a (cin x cout) reduction
// over all points: per-CTA register-tiled 4x4 partial sums, reduced across
// point groups with warp shuffles + shared memory, written as one partial per
// CTA and summed in a fixed order by k_reduce_partials8 (deterministic).
#include "common.cuh"

namespace dfno {

template <typename R, int VEC>
struct Vec;
template <>
struct Vec<float, 4> {
  using T = float4;
};
template <>
struct Vec<float, 2> {
  using T = float2;
};
template <>
struct Vec<double, 2> {
  using T = double2;
};
template <typename R>
struct Vec<R, 1> {
  using T = R;
};

template <typename R, int VEC>
__device__ __forceinline__ void ldv(const R* p, R (&v)[VEC]) {
  if constexpr (VEC == 1) {
    v[0] = __ldg(p);
  } else {
    typename Vec<R, VEC>::T t = __ldg(reinterpret_cast<const typename Vec<R, VEC>::T*>(p));
    const R* tr = reinterpret_cast<const R*>(&t);
#pragma unroll
    for (int k = 0; k < VEC; ++k) v[k] = tr[k];
  }
}

template <typename R, int VEC>
__device__ __forceinline__ void stv(R* p, const R (&v)[VEC]) {
  if constexpr (VEC == 1) {
    p[0] = v[0];
  } else {
    typename Vec<R, VEC>::T t;
    R* tr = reinterpret_cast<R*>(&t);
#pragma unroll
    for (int k = 0; k < VEC; ++k) tr[k] = v[k];
    *reinterpret_cast<typename Vec<R, VEC>::T*>(p) = t;
  }
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <typename R, int CO, int VEC>
__global__ void __launch_bounds__(256) k_mix_fwd(long long npts, int nb, int cin, int cout, int o0,
                                                 const R* __restrict__ src, int src_act, int act,
                                                 const R* __restrict__ w, R* __restrict__ pre,
                                                 R* __restrict__ post) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* ws = reinterpret_cast<R*>(smem_raw);  // [cin][CO]
  for (int k = threadIdx.x; k < cin * CO; k += blockDim.x) {
    const int i = k / CO, o = k % CO;
    ws[k] = (o0 + o < cout) ? w[(long long)i * cout + o0 + o] : (R)0;
  }
  __syncthreads();
  const long long nvec = npts / VEC;
  const long long total = (long long)nb * nvec;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long bb = q / nvec;
    const long long p = (q - bb * nvec) * VEC;
    R acc[CO][VEC];
#pragma unroll
    for (int o = 0; o < CO; ++o)
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[o][k] = (R)0;
    const R* s = src + bb * cin * npts + p;
    for (int i = 0; i < cin; ++i) {
      R v[VEC];
      ldv<R, VEC>(s + (long long)i * npts, v);
      if (src_act) {
#pragma unroll
        for (int k = 0; k < VEC; ++k) v[k] = act_apply<R>(act, v[k]);
      }
      const R* wr = ws + i * CO;
#pragma unroll
      for (int o = 0; o < CO; ++o) {
        const R wv = wr[o];
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[o][k] = fma(v[k], wv, acc[o][k]);
      }
    }
    R* pr = pre + bb * cout * npts + p;
    R* po = post ? post + bb * cout * npts + p : nullptr;
#pragma unroll
    for (int o = 0; o < CO; ++o) {
      if (o0 + o < cout) {
        stv<R, VEC>(pr + (long long)(o0 + o) * npts, acc[o]);
        if (po) {
          R a[VEC];
#pragma unroll
          for (int k = 0; k < VEC; ++k) a[k] = act_apply<R>(act, acc[o][k]);
          stv<R, VEC>(po + (long long)(o0 + o) * npts, a);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------
constexpr int kMixBwdThreads = 256;

// CM = padded max(cin, cout) (multiple of 4); V consecutive points per thread
// (vector loads / stores along the contiguous point index); a tile is
// kMixBwdThreads * V points of one batch entry.
//   phase 1  gp[o][v] = gout * act'(pre)            (registers + smem Gs[o][p])
//   phase 2  a[i][v]  = f(src); gin[i] = sum_o gp[o] w[i][o]   (smem As[i][p])
//   phase 3  gW partial (4x4 register tiles per thread, point groups)
//
// Channel blocks (widths above 32): the launch covers input channels
// [i0, i0 + cin) and output channels [o0, o0 + cout) of a (cin_tot, cout_tot)
// mixer; the input gradient of the block is written (first output block) or
// added (gin_add), and the weight-gradient partial lands at its block of the
// CTA's (cin_tot x cout_tot) partial.
template <typename R, int CM, int V>
__global__ void __launch_bounds__(kMixBwdThreads) k_mix_bwd(
    long long npts, int nb, int cin, int cout, const R* __restrict__ gout, const R* __restrict__ pre,
    const R* __restrict__ src, int src_act, int act, const R* __restrict__ w, R* __restrict__ gin,
    R* __restrict__ partials, int cin_tot, int cout_tot, int i0, int o0, int gin_add) {
  constexpr int TP = kMixBwdThreads * V;      // points per tile
  constexpr int NB4 = CM / 4;
  constexpr int NPAIR = NB4 * NB4;
  constexpr int NGRP = (kMixBwdThreads / NPAIR) > 0 ? (kMixBwdThreads / NPAIR) : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* ws = reinterpret_cast<R*>(smem_raw);     // [CM][CM] (i, o), zero padded
  R* As = ws + CM * CM;                       // [CM][TP]
  R* Gs = As + CM * TP;                       // [CM][TP]
  R* red = Gs + CM * TP;                      // [NGRP][NPAIR*16]

  for (int k = threadIdx.x; k < CM * CM; k += blockDim.x) {
    const int i = k / CM, o = k % CM;
    ws[k] = (i < cin && o < cout) ? w[(long long)(i0 + i) * cout_tot + o0 + o] : (R)0;
  }
  const int tid = threadIdx.x;
  const int pair = tid % NPAIR, grp = tid / NPAIR;
  const bool reducer = tid < NPAIR * NGRP;
  const int ib = pair / NB4, ob = pair % NB4;
  R acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = (R)0;

  const long long tiles_per_b = (npts + TP - 1) / TP;
  const long long ntiles = tiles_per_b * nb;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long bb = tile / tiles_per_b;
    const long long p0 = (tile - bb * tiles_per_b) * TP;
    const long long p = p0 + (long long)tid * V;
    const bool full = (p + V <= npts);
    __syncthreads();  // previous tile's As / Gs consumed
    // ---- phase 1: gp = gout * act'(pre)
    R gp[CM][V];
    const R* go = gout + (bb * cout_tot + o0) * npts + p;
    const R* pr = pre + (bb * cout_tot + o0) * npts + p;
#pragma unroll
    for (int o = 0; o < CM; ++o) {
      R gv[V], pv[V];
      if (o < cout && full) {
        ldv<R, V>(go + (long long)o * npts, gv);
        ldv<R, V>(pr + (long long)o * npts, pv);
      } else {
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const bool ok = (o < cout) && (p + k < npts);
          gv[k] = ok ? go[(long long)o * npts + k] : (R)0;
          pv[k] = ok ? pr[(long long)o * npts + k] : (R)0;
        }
      }
#pragma unroll
      for (int k = 0; k < V; ++k) gp[o][k] = gv[k] * act_deriv<R>(act, pv[k]);
      stv<R, V>(Gs + o * TP + tid * V, gp[o]);
    }
    // ---- phase 2: a = f(src) -> As ; gin = sum_o gp w
    const R* sp = src + (bb * cin_tot + i0) * npts + p;
    R* gi = gin ? gin + (bb * cin_tot + i0) * npts + p : nullptr;
    for (int i = 0; i < CM; ++i) {
      if (i >= cin) {
        R z[V];
#pragma unroll
        for (int k = 0; k < V; ++k) z[k] = (R)0;
        stv<R, V>(As + i * TP + tid * V, z);
        continue;
      }
      R av[V];
      if (full) {
        ldv<R, V>(sp + (long long)i * npts, av);
      } else {
#pragma unroll
        for (int k = 0; k < V; ++k) av[k] = (p + k < npts) ? sp[(long long)i * npts + k] : (R)0;
      }
      if (src_act) {
#pragma unroll
        for (int k = 0; k < V; ++k) av[k] = act_apply<R>(act, av[k]);
      }
      stv<R, V>(As + i * TP + tid * V, av);
      if (gi) {
        R s[V];
#pragma unroll
        for (int k = 0; k < V; ++k) s[k] = (R)0;
        const R* wr = ws + i * CM;
#pragma unroll
        for (int o = 0; o < CM; ++o) {
          const R wv = wr[o];
#pragma unroll
          for (int k = 0; k < V; ++k) s[k] = fma(gp[o][k], wv, s[k]);
        }
        if (full) {
          if (gin_add) {
            R prev[V];
            ldv<R, V>(gi + (long long)i * npts, prev);
#pragma unroll
            for (int k = 0; k < V; ++k) s[k] += prev[k];
          }
          stv<R, V>(gi + (long long)i * npts, s);
        } else {
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (p + k < npts) gi[(long long)i * npts + k] = gin_add ? gi[(long long)i * npts + k] + s[k] : s[k];
        }
      }
    }
    __syncthreads();
    // ---- phase 3: weight-gradient partial sums
    if (reducer) {
      const R* ar = As + ib * 4 * TP;
      const R* gr = Gs + ob * 4 * TP;
      for (int t = grp; t < TP; t += NGRP) {
        R a4[4], g4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a4[k] = ar[k * TP + t];
          g4[k] = gr[k * TP + t];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(a4[a], g4[b], acc[a][b]);
      }
    }
  }
  // Cross-group reduction in fixed order.
  __syncthreads();
  if (reducer) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) red[grp * NPAIR * 16 + pair * 16 + a * 4 + b] = acc[a][b];
  }
  __syncthreads();
  R* outp = partials + (long long)blockIdx.x * cin_tot * cout_tot;
  for (int e = tid; e < NPAIR * 16; e += blockDim.x) {
    R s = (R)0;
    for (int gI = 0; gI < NGRP; ++gI) s += red[gI * NPAIR * 16 + e];
    const int pr2 = e / 16, ab = e % 16;
    const int i = (pr2 / NB4) * 4 + ab / 4;
    const int o = (pr2 % NB4) * 4 + ab % 4;
    if (i < cin && o < cout) outp[(long long)(i0 + i) * cout_tot + o0 + o] = s;
  }
}

// Fixed-shape tree over the partials (deterministic, independent of
// scheduling): 32 consecutive elements per warp (coalesced), eight warps take
// every eighth partial, then the eight group sums are added pairwise.
template <typename R>
__global__ void __launch_bounds__(256) k_reduce_partials8(int nparts, long long n, const R* __restrict__ partials,
                                                          R* __restrict__ out) {
  __shared__ R grp_sum[8][32];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const long long e = (long long)blockIdx.x * 32 + lane;
  R s = (R)0;
  if (e < n)
    for (int k = grp; k < nparts; k += 8) s += partials[(long long)k * n + e];
  grp_sum[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && e < n) {
    const R a = (grp_sum[0][lane] + grp_sum[1][lane]) + (grp_sum[2][lane] + grp_sum[3][lane]);
    const R b = (grp_sum[4][lane] + grp_sum[5][lane]) + (grp_sum[6][lane] + grp_sum[7][lane]);
    out[e] = a + b;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename R, int CO, int VEC>
static int launch_mix_fwd(long long npts, int nb, int cin, int cout, int o0, const void* src, int src_act,
                          int act, const void* w, void* pre, void* post, cudaStream_t st) {
  const size_t smem = (size_t)cin * CO * sizeof(R);
  auto kern = k_mix_fwd<R, CO, VEC>;
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return DFNO_ERR_UNSUPPORTED;
  }
  const long long work = (long long)nb * (npts / VEC);
  long long blocks = (work + 255) / 256;
  const long long cap = (long long)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, 256, smem, st>>>(npts, nb, cin, cout, o0, (const R*)src, src_act, act, (const R*)w,
                                            (R*)pre, (R*)post);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

template <typename R, int CO>
static int mix_fwd_vec(long long npts, int nb, int cin, int cout, int o0, const void* src, int src_act, int act,
                       const void* w, void* pre, void* post, cudaStream_t st) {
  constexpr int V = sizeof(R) == 4 ? 4 : 2;
  const bool aligned = (npts % V == 0) && ((uintptr_t)src % (V * sizeof(R)) == 0) &&
                       ((uintptr_t)pre % (V * sizeof(R)) == 0) &&
                       (post == nullptr || (uintptr_t)post % (V * sizeof(R)) == 0);
  if (aligned) return launch_mix_fwd<R, CO, V>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
  return launch_mix_fwd<R, CO, 1>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
}

template <typename R>
static int mix_fwd_dispatch(long long npts, int nb, int cin, int cout, const void* src, int src_act, int act,
                            const void* w, void* pre, void* post, cudaStream_t st) {
  for (int o0 = 0; o0 < cout; o0 += 32) {
    const int rem = cout - o0;
    int rc;
    if (rem <= 1) rc = mix_fwd_vec<R, 1>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    else if (rem <= 2) rc = mix_fwd_vec<R, 2>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    else if (rem <= 4) rc = mix_fwd_vec<R, 4>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    else if (rem <= 8) rc = mix_fwd_vec<R, 8>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    else if (rem <= 12) rc = mix_fwd_vec<R, 12>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    else if (rem <= 16) rc = mix_fwd_vec<R, 16>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    else if (rem <= 20) rc = mix_fwd_vec<R, 20>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    else if (rem <= 24) rc = mix_fwd_vec<R, 24>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    else rc = mix_fwd_vec<R, 32>(npts, nb, cin, cout, o0, src, src_act, act, w, pre, post, st);
    if (rc != DFNO_OK) return rc;
  }
  return DFNO_OK;
}

static int mix_bwd_cm(int cin, int cout) {
  const int m = cin > cout ? cin : cout;
  if (m <= 4) return 4;
  if (m <= 8) return 8;
  if (m <= 12) return 12;
  if (m <= 16) return 16;
  if (m <= 20) return 20;
  if (m <= 24) return 24;
  if (m <= 32) return 32;
  return 64;  // channel blocks of 32 (mix_bwd_dispatch)
}

template <typename R>
static constexpr int mix_bwd_v() {
  return sizeof(R) == 4 ? 2 : 1;
}

// CTA count (= number of weight-gradient partials): independent of the
// vector width so dfno_mix_bwd_partials can size the buffer up front.
static int mix_bwd_blocks(long long npts, int nb) {
  const long long tiles = ((npts + kMixBwdThreads - 1) / kMixBwdThreads) * nb;
  long long blocks = (long long)num_sms() * 2;
  if (blocks > tiles) blocks = tiles;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

struct MixBlock {
  int cin_tot, cout_tot, i0, o0, gin_add;
};

template <typename R, int CM, int V>
static int launch_mix_bwd_v(long long npts, int nb, int cin, int cout, const void* gout, const void* pre,
                            const void* src, int src_act, int act, const void* w, void* gin, void* partials,
                            cudaStream_t st, MixBlock blk) {
  constexpr int NB4 = CM / 4;
  constexpr int NPAIR = NB4 * NB4;
  constexpr int NGRP = (kMixBwdThreads / NPAIR) > 0 ? (kMixBwdThreads / NPAIR) : 1;
  constexpr int TP = kMixBwdThreads * V;
  const size_t smem = sizeof(R) * ((size_t)CM * CM + 2 * (size_t)TP * CM + (size_t)NGRP * NPAIR * 16);
  auto kern = k_mix_bwd<R, CM, V>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  const int blocks = mix_bwd_blocks(npts, nb);
  kern<<<blocks, kMixBwdThreads, smem, st>>>(npts, nb, cin, cout, (const R*)gout, (const R*)pre, (const R*)src,
                                             src_act, act, (const R*)w, (R*)gin, (R*)partials, blk.cin_tot,
                                             blk.cout_tot, blk.i0, blk.o0, blk.gin_add);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

template <typename R, int CM>
static int launch_mix_bwd(long long npts, int nb, int cin, int cout, const void* gout, const void* pre,
                          const void* src, int src_act, int act, const void* w, void* gin, void* partials,
                          cudaStream_t st, MixBlock blk = MixBlock{-1, -1, 0, 0, 0}) {
  if (blk.cin_tot < 0) blk = MixBlock{cin, cout, 0, 0, 0};
  constexpr int V = mix_bwd_v<R>();
  // vector path needs every row V-aligned
  const bool aligned = (npts % V == 0) && ((uintptr_t)gout % (V * sizeof(R)) == 0) &&
                       ((uintptr_t)pre % (V * sizeof(R)) == 0) && ((uintptr_t)src % (V * sizeof(R)) == 0) &&
                       (gin == nullptr || (uintptr_t)gin % (V * sizeof(R)) == 0);
  if (aligned)
    return launch_mix_bwd_v<R, CM, V>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st, blk);
  return launch_mix_bwd_v<R, CM, 1>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st, blk);
}

template <typename R>
static int mix_bwd_dispatch(long long npts, int nb, int cin, int cout, const void* gout, const void* pre,
                            const void* src, int src_act, int act, const void* w, void* gin, void* partials,
                            cudaStream_t st) {
  switch (mix_bwd_cm(cin, cout)) {
    case 4: return launch_mix_bwd<R, 4>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st);
    case 8: return launch_mix_bwd<R, 8>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st);
    case 12: return launch_mix_bwd<R, 12>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st);
    case 16: return launch_mix_bwd<R, 16>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st);
    case 20: return launch_mix_bwd<R, 20>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st);
    case 24: return launch_mix_bwd<R, 24>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st);
    case 32: return launch_mix_bwd<R, 32>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, st);
    default: break;
  }
  // wider mixers: 32 x 32 channel blocks; the input gradient of an input block
  // is written by its first output block and accumulated by the rest (stream
  // order), each block pair fills its part of the per-CTA weight partials
  for (int i0 = 0; i0 < cin; i0 += 32)
    for (int o0 = 0; o0 < cout; o0 += 32) {
      const int ni = cin - i0 < 32 ? cin - i0 : 32, no = cout - o0 < 32 ? cout - o0 : 32;
      const int rc = launch_mix_bwd<R, 32>(npts, nb, ni, no, gout, pre, src, src_act, act, w, gin, partials, st,
                                           MixBlock{cin, cout, i0, o0, o0 > 0 ? 1 : 0});
      if (rc != DFNO_OK) return rc;
    }
  return DFNO_OK;
}

int mix_bwd_tc(long long npts, int nb, int cin, int cout, const void* gout, const void* pre, const void* src,
               int src_act, int act, const void* w, void* gin, void* partials, int blocks, cudaStream_t st);
int mix_fwd_tc(long long npts, int nb, int cin, int cout, const void* src, int src_act, int act, const void* w,
               void* pre, void* post, cudaStream_t st);

}  // namespace dfno

using namespace dfno;

extern "C" int dfno_mix_fwd(const dfno_geom* g, int64_t npts, int cin, int cout, const void* src, int src_act,
                            const void* w, void* pre, void* post, void* stream) {
  if (!g || !src || !w || !pre) return DFNO_ERR_NULL;
  if (npts < 0 || cin < 1 || cout < 1) return DFNO_ERR_DIMENSION;
  if (npts == 0 || g->batch == 0) return DFNO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->dtype == DFNO_F32) {
    const int rc = mix_fwd_tc(npts, g->batch, cin, cout, src, src_act, g->act, w, pre, post, st);
    if (rc != DFNO_ERR_UNSUPPORTED) return rc;
    return mix_fwd_dispatch<float>(npts, g->batch, cin, cout, src, src_act, g->act, w, pre, post, st);
  }
  if (g->dtype == DFNO_F64)
    return mix_fwd_dispatch<double>(npts, g->batch, cin, cout, src, src_act, g->act, w, pre, post, st);
  return DFNO_ERR_DTYPE;
}

extern "C" int dfno_mix_bwd_partials(const dfno_geom* g, int64_t npts, int cin, int cout, int64_t* partial_elems,
                                     int* num_partials) {
  if (!g || !partial_elems || !num_partials) return DFNO_ERR_NULL;
  if (mix_bwd_cm(cin, cout) < 0) return DFNO_ERR_UNSUPPORTED;
  const int blocks = mix_bwd_blocks(npts, g->batch);
  *num_partials = blocks;
  *partial_elems = (int64_t)blocks * cin * cout;
  return DFNO_OK;
}

extern "C" int dfno_mix_bwd(const dfno_geom* g, int64_t npts, int cin, int cout, const void* gout, const void* pre,
                            const void* src, int src_act, const void* w, void* gin, void* partials, void* stream) {
  if (!g || !gout || !pre || !src || !w || !partials) return DFNO_ERR_NULL;
  if (npts < 1 || cin < 1 || cout < 1) return DFNO_ERR_DIMENSION;
  if (src_act < 0 || src_act > 2) return DFNO_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  if (src_act == 2) {  // fused act'(src) on the input gradient: tcgen05 path only
    if (g->dtype != DFNO_F32 || !gin) return DFNO_ERR_UNSUPPORTED;
    return mix_bwd_tc(npts, g->batch, cin, cout, gout, pre, src, src_act, g->act, w, gin, partials,
                      mix_bwd_blocks(npts, g->batch), st);
  }
  if (g->dtype == DFNO_F32) {
    const int rc = mix_bwd_tc(npts, g->batch, cin, cout, gout, pre, src, src_act, g->act, w, gin, partials,
                              mix_bwd_blocks(npts, g->batch), st);
    if (rc != DFNO_ERR_UNSUPPORTED) return rc;
    return mix_bwd_dispatch<float>(npts, g->batch, cin, cout, gout, pre, src, src_act, g->act, w, gin, partials, st);
  }
  if (g->dtype == DFNO_F64)
    return mix_bwd_dispatch<double>(npts, g->batch, cin, cout, gout, pre, src, src_act, g->act, w, gin, partials,
                                    st);
  return DFNO_ERR_DTYPE;
}

extern "C" int dfno_reduce_partials(const dfno_geom* g, int num_partials, int64_t n, const void* partials, void* out,
                                    void* stream) {
  if (!g || !partials || !out) return DFNO_ERR_NULL;
  cudaStream_t st = (cudaStream_t)stream;
  const int blocks = (int)((n + 31) / 32);
  if (g->dtype == DFNO_F32)
    k_reduce_partials8<float><<<blocks, 256, 0, st>>>(num_partials, n, (const float*)partials, (float*)out);
  else if (g->dtype == DFNO_F64)
    k_reduce_partials8<double><<<blocks, 256, 0, st>>>(num_partials, n, (const double*)partials, (double*)out);
  else
    return DFNO_ERR_DTYPE;
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}
