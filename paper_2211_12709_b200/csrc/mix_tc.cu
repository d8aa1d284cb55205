// Channel-mix backward on the tcgen05 tensor cores (fp32 via 3xTF32).
//
// Replaces the mixer part of fno_backward (reference d/fno.py:484-486 and
// :497-499): gp = g * act'(pre) (d/fno.py:484, :497), _mix_input_grad
// (d/fno.py:409-412) and _mix_weight_grad (d/fno.py:405-406).  Both
// contractions are GEMMs over a 128-point tile held one point per thread:
//
//   GEMM1 (input grad)   D1[p][i]  = sum_o gp[p][o] W[i][o]
//        A = gp (128 points x K = o) in TMEM (tcgen05.st from the owning
//        thread), B = W (i x o) in shared memory, 3 products per K step
//        (hi*hi + lo*hi + hi*lo), D1 read back by the owning thread and
//        stored coalesced.
//   GEMM2 (weight grad)  D2[r][c] += sum_p A2[r][p] B2[c][p]
//        rows r: a_hi(i) at r = i, a_lo(i) at r = 32 + i; columns c: gp_hi(o)
//        at c = o, gp_lo(o) at c = 32 + o, so ONE M=64 N=64 K=8 MMA per 8
//        points yields all four hi/lo cross products.  D2 accumulates kMbFlush
//        tiles in TMEM, then warps 0-1 fold its quadrants into a per-CTA
//        accumulator (TMEM columns 192..223, round-to-nearest fp32 adds in
//        registers) and the next tile restarts D2: the
//        tensor core's fp32 accumulation is not round-to-nearest, and left to
//        run over a whole CTA's share of points (~3.5k MMAs at C2) its bias
//        cost 7.5e-5 relative on the weight gradient against a random upstream
//        gradient (tools/precision_probe.py).  The folded sums become this CTA's
//        partial (reduced in fixed order by k_reduce_partials8: deterministic,
//        d/training.py:77-82).  M = 64 reads only the 64 A2 rows
//        that exist (an M = 128 MMA would stream 2 KB more shared memory per
//        MMA; 743 -> 726 us at C2 in the sigma-on-source mode).
//
// Shared-memory operands are SWIZZLE_NONE K-major with a padded LBO of 144 B
// so the one-point-per-thread scalar stores are bank-conflict free.  The MMAs
// of tile i run while the CTA loads tile i + 1 (one mbarrier per CTA).
#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace dfno {

namespace {
constexpr int kMbThreads = 128;             // one thread per point of a 128-point tile
constexpr int kMbLbo = 144;                 // bytes between K-adjacent core matrices
constexpr int kMbSbo = 32 * kMbLbo;         // bytes between 8-row groups (K = 128 points)
constexpr int kMbOpBytes = 8 * kMbSbo;      // 64 rows x 128 points
constexpr uint32_t kMbTmemCols = 256;       // D1 0..31 | A1 hi 32..63 | A1 lo 64..95 | D2 128..191 | ACC 192..223
constexpr int kMbFlush = 16;                // tiles (2048 points) accumulated in D2 before the fold into ACC

__device__ __forceinline__ int mb_off(int r, int k) {
  return (r >> 3) * kMbSbo + (k >> 2) * kMbLbo + (r & 7) * 16 + (k & 3) * 4;
}
}  // namespace

// CM: channel bucket (>= cin, cout); EXACT: cin == cout == CM (no channel
// masks); ACT: activation code (compile time: no per-element branches).
template <int CM, bool EXACT, int ACT>
__global__ void __launch_bounds__(kMbThreads, 2) k_mix_bwd_tc(long long npts, int nb, int cin_rt, int cout_rt,
                                                              const float* __restrict__ gout,
                                                              const float* __restrict__ pre,
                                                              const float* __restrict__ src, int src_act,
                                                              const float* __restrict__ w, float* __restrict__ gin,
                                                              float* __restrict__ partials) {
  const int cin = EXACT ? CM : cin_rt, cout = EXACT ? CM : cout_rt;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar, bar2;  // GEMM1 (input grad, thread 0) / GEMM2 (weight grad, thread 32) commits
  __shared__ uint32_t tmem_base;
  unsigned char* a2 = smem;
  unsigned char* b2 = smem + kMbOpBytes;
  unsigned char* b1 = smem + 2 * kMbOpBytes;  // W hi plane, then lo plane
  const int KPo = (cout + 7) & ~7;             // GEMM1 K (o), multiple of 8
  const int NPi = (cin + 15) & ~15;            // GEMM1 N (i), multiple of 16
  const int sbo_b1 = (KPo / 4) * 128;
  const int b1_plane = (NPi / 8) * sbo_b1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool want_gin = gin != nullptr;

  for (int e = tid; e < NPi * KPo; e += kMbThreads) {
    const int i = e / KPo, o = e % KPo;
    const float v = (i < cin && o < cout) ? w[(long long)i * cout + o] : 0.f;
    float h, l;
    tc::split_rn(v, h, l);
    const int off = (i >> 3) * sbo_b1 + (o >> 2) * 128 + (i & 7) * 16 + (o & 3) * 4;
    *reinterpret_cast<float*>(b1 + off) = h;
    *reinterpret_cast<float*>(b1 + b1_plane + off) = l;
  }
  if (warp == 0) tc::tmem_alloc<kMbTmemCols>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&bar2, 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t d1 = tmem, a1h = tmem + 32, a1l = tmem + 64, d2 = tmem + 128, dacc = tmem + 192;
  const uint32_t lane_off = (uint32_t)(32 * warp) << 16;

  const long long tiles_per_b = (npts + kMbThreads - 1) / kMbThreads;
  const long long ntiles = tiles_per_b * nb;
  int it = 0;
  long long prev_out = -1;  // gin element offset of the previous tile's point (or -1)

  // src_act == 2: the input gradient leaves already multiplied by act'(src)
  // (the decoder's input is the last block's pre-activation, so the next
  // backward DFT needs no act' of its own); dprev holds act'(src) of the tile
  // being drained
  const bool gin_dact = src_act == 2;
  float dprev[CM], dcur[CM];
#pragma unroll
  for (int i = 0; i < CM; ++i) dprev[i] = dcur[i] = 1.f;
  auto drain_gin = [&]() {
    uint32_t r[32];
    tc::tmem_ld32_nowait(d1 + lane_off, r);
    tc::tmem_ld_wait();
    if (prev_out >= 0) {
#pragma unroll
      for (int i = 0; i < CM; ++i)
        if (EXACT || i < cin) {
          const float v = __uint_as_float(r[i]);
          __stcs(gin + prev_out + (long long)i * npts, gin_dact ? v * dprev[i] : v);
        }
    }
  };

  // fold D2 (rows 0..63: a_hi(i), a_lo(i); columns gp_hi(o) | gp_lo(o)) into
  // ACC[row][o] (TMEM).  GEMM2 is an M = 64 MMA: row r sits in TMEM lane
  // 32 (r / 16) + r % 16 (tools/probes/mma_m64_probe.cu), so every warp folds
  // the 16 rows in the first half of its lane quarter (row = 16 warp + lane)
  bool acc_live = false;
  auto fold_d2 = [&]() {
    {
      uint32_t r0[32], r1[32];
      float v[32];
      tc::tmem_ld32_nowait(d2 + lane_off, r0);
      tc::tmem_ld32_nowait(d2 + lane_off + 32, r1);
      tc::tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(r0[c]) + __uint_as_float(r1[c]);
      if (acc_live) {
        tc::tmem_ld32_nowait(dacc + lane_off, r0);
        tc::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] += __uint_as_float(r0[c]);
      }
      tc::tmem_st32(dacc + lane_off, v);
      tc::tmem_st_wait();
    }
    acc_live = true;
  };

  // register double buffer: tile i + 1 is loaded while tile i is converted
  float gv[CM], pv[CM], sv[CM];
  auto load = [&](long long tile) {
    const long long bb = tile / tiles_per_b;
    const long long p = (tile - bb * tiles_per_b) * kMbThreads + tid;
    const bool valid = tile < ntiles && p < npts;
    const float* g0 = gout + (bb * cout) * npts + p;
    const float* p0 = pre + (bb * cout) * npts + p;
    const float* s0 = src + (bb * cin) * npts + p;
#pragma unroll
    for (int o = 0; o < CM; ++o) {
      const bool ok = valid && (EXACT || o < cout);
      gv[o] = ok ? __ldcs(g0) : 0.f;
      pv[o] = ok ? __ldcs(p0) : 0.f;
      g0 += npts;
      p0 += npts;
    }
#pragma unroll
    for (int i = 0; i < CM; ++i) {
      sv[i] = (valid && (EXACT || i < cin)) ? __ldg(s0) : 0.f;
      s0 += npts;
    }
  };
  load(blockIdx.x);
#pragma unroll 1
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const long long bb = tile / tiles_per_b;
    const long long p = (tile - bb * tiles_per_b) * kMbThreads + tid;
    const bool valid = p < npts;
    float gp[CM], a[CM];
    // gp = g * act'(pre) ; a = act(src) or src  (zero for padding / invalid points)
    static_assert(CM % 2 == 0, "channel rows are converted in pairs");
#pragma unroll
    for (int o = 0; o < CM; o += 2) {
      const float2 v = f2mul(make_float2(gv[o], gv[o + 1]), act_deriv2<ACT>(make_float2(pv[o], pv[o + 1])));
      gp[o] = v.x;
      gp[o + 1] = v.y;
    }
    if (gin_dact) {
#pragma unroll
      for (int i = 0; i < CM; i += 2) {
        float2 av, dv;
        act_both2<ACT>(make_float2(sv[i], sv[i + 1]), av, dv);
        a[i] = av.x;
        a[i + 1] = av.y;
        dcur[i] = dv.x;
        dcur[i + 1] = dv.y;
      }
    } else if (src_act) {
#pragma unroll
      for (int i = 0; i < CM; i += 2) {
        const float2 av = act_apply2<ACT>(make_float2(sv[i], sv[i + 1]));
        a[i] = av.x;
        a[i + 1] = av.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CM; ++i) a[i] = sv[i];
    }
    load(tile + gridDim.x);
    if (it > 0) {  // MMAs of the previous tile done: its operands are free, D1 holds its input grad
      if (want_gin) tc::mbar_wait(&bar, (it - 1) & 1);
      tc::mbar_wait(&bar2, (it - 1) & 1);
      tc::fence_after();
      if (want_gin) drain_gin();
      if ((it - 1) % kMbFlush == kMbFlush - 1) fold_d2();  // D2 restarts at tile it
    }
#pragma unroll
    for (int i = 0; i < CM; ++i) dprev[i] = dcur[i];
    {
      // gp split once (round-to-nearest hi, exact remainder lo; the tensor
      // core's truncation of lo costs <= 2^-21 relative) and shared by the
      // GEMM1 A operand (TMEM) and the GEMM2 B operand (shared memory)
      float h[32], l[32];
#pragma unroll
      for (int o = 0; o < 32; o += 2) {
        if (o < CM) tc::split_hl2(make_float2(gp[o], gp[o + 1]), h[o], h[o + 1], l[o], l[o + 1]);
        else h[o] = l[o] = h[o + 1] = l[o + 1] = 0.f;
      }
      if (want_gin) {
        tc::tmem_st32(a1h + lane_off, h);
        tc::tmem_st32(a1l + lane_off, l);
      }
#pragma unroll
      for (int o = 0; o < CM; ++o) {
        if (EXACT || o < cout) {
          *reinterpret_cast<float*>(b2 + mb_off(o, tid)) = h[o];
          *reinterpret_cast<float*>(b2 + mb_off(32 + o, tid)) = l[o];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CM; ++i) {
      if (EXACT || i < cin) {
        float h, l;
        tc::split_hl(a[i], h, l);
        *reinterpret_cast<float*>(a2 + mb_off(i, tid)) = h;
        *reinterpret_cast<float*>(a2 + mb_off(32 + i, tid)) = l;
      }
    }
    if (want_gin) tc::tmem_st_wait();
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    if (tid == 0 && want_gin) {
      tc::fence_after();
      const uint32_t id1 = tc::idesc_tf32(128, NPi);
      const uint32_t sb1 = tc::smem_u32(b1);
      for (int s = 0; s < KPo / 8; ++s) {  // lo products first, hi.hi last
        const uint64_t bh = tc::desc(sb1 + s * 256, 128, sbo_b1);
        const uint64_t bl = tc::desc(sb1 + b1_plane + s * 256, 128, sbo_b1);
        tc::mma_tf32_ts(d1, a1l + 8 * s, bh, id1, s > 0 ? 1u : 0u);
        tc::mma_tf32_ts(d1, a1h + 8 * s, bl, id1, 1u);
      }
      for (int s = 0; s < KPo / 8; ++s) tc::mma_tf32_ts(d1, a1h + 8 * s, tc::desc(sb1 + s * 256, 128, sbo_b1), id1, 1u);
      tc::commit(&bar);
    }
    if (tid == 32) {  // second issuing warp: the weight-gradient GEMM overlaps GEMM1's issue
      tc::fence_after();
      const uint32_t id2 = tc::idesc_tf32(64, 64);  // only rows a_hi(i), a_lo(i) (0..63) of A2 exist
      const uint32_t sa2 = tc::smem_u32(a2), sb2 = tc::smem_u32(b2);
#pragma unroll 4
      for (int s = 0; s < kMbThreads / 8; ++s)
        tc::mma_tf32(d2, tc::desc(sa2 + s * 2 * kMbLbo, kMbLbo, kMbSbo), tc::desc(sb2 + s * 2 * kMbLbo, kMbLbo, kMbSbo),
                     id2, (it % kMbFlush != 0 || s > 0) ? 1u : 0u);
      tc::commit(&bar2);
    }
    prev_out = valid ? (bb * cin * npts + p) : -1;
  }
  if (it > 0) {
    if (want_gin) tc::mbar_wait(&bar, (it - 1) & 1);
    tc::mbar_wait(&bar2, (it - 1) & 1);
    tc::fence_after();
    if (want_gin) drain_gin();
    fold_d2();  // the last (possibly partial) chunk
  }
  // ---- weight-gradient partial: a_hi and a_lo rows of ACC -> shared -> partial
  __syncthreads();  // every thread is past its last operand write
  float* st = reinterpret_cast<float*>(smem);  // [64][33], aliases A2 (all MMAs done)
  if (it > 0) {
    uint32_t r0[32];
    tc::tmem_ld32_nowait(dacc + lane_off, r0);
    tc::tmem_ld_wait();
    const int row = 16 * warp + lane;  // M = 64 accumulator rows (see fold_d2)
    if (lane < 16) {
#pragma unroll
      for (int c = 0; c < 32; ++c) st[row * 33 + c] = __uint_as_float(r0[c]);
    }
  }
  __syncthreads();
  float* outp = partials + (long long)blockIdx.x * cin * cout;
  for (int e = tid; e < cin * cout; e += kMbThreads) {
    const int i = e / cout, o = e % cout;
    outp[e] = it > 0 ? st[i * 33 + o] + st[(32 + i) * 33 + o] : 0.f;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kMbTmemCols>(tmem);
}

template <int CM, bool EXACT, int ACT>
static int launch_mix_bwd_tc3(long long npts, int nb, int cin, int cout, const void* gout, const void* pre,
                              const void* src, int src_act, const void* w, void* gin, void* partials, int blocks,
                              cudaStream_t st) {
  const int smem = 2 * kMbOpBytes + 2 * 4 * 1024;
  auto kern = k_mix_bwd_tc<CM, EXACT, ACT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return DFNO_ERR_UNSUPPORTED;
  kern<<<blocks, kMbThreads, smem, st>>>(npts, nb, cin, cout, (const float*)gout, (const float*)pre,
                                         (const float*)src, src_act, (const float*)w, (float*)gin,
                                         (float*)partials);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

template <int CM, bool EXACT>
static int launch_mix_bwd_tc(long long npts, int nb, int cin, int cout, const void* gout, const void* pre,
                             const void* src, int src_act, int act, const void* w, void* gin, void* partials,
                             int blocks, cudaStream_t st) {
  switch (act) {
    case DFNO_ACT_GELU:
      return launch_mix_bwd_tc3<CM, EXACT, DFNO_ACT_GELU>(npts, nb, cin, cout, gout, pre, src, src_act, w, gin,
                                                          partials, blocks, st);
    case DFNO_ACT_RELU:
      return launch_mix_bwd_tc3<CM, EXACT, DFNO_ACT_RELU>(npts, nb, cin, cout, gout, pre, src, src_act, w, gin,
                                                          partials, blocks, st);
    default:
      return launch_mix_bwd_tc3<CM, EXACT, DFNO_ACT_IDENTITY>(npts, nb, cin, cout, gout, pre, src, src_act, w, gin,
                                                              partials, blocks, st);
  }
}

// fp32, cin and cout <= 32; returns DFNO_ERR_UNSUPPORTED otherwise.
int mix_bwd_tc(long long npts, int nb, int cin, int cout, const void* gout, const void* pre, const void* src,
               int src_act, int act, const void* w, void* gin, void* partials, int blocks, cudaStream_t st) {
  const int m = cin > cout ? cin : cout;
  if (m > 32 || blocks < 1) return DFNO_ERR_UNSUPPORTED;
#define DFNO_MB(CM, EX) \
  return launch_mix_bwd_tc<CM, EX>(npts, nb, cin, cout, gout, pre, src, src_act, act, w, gin, partials, blocks, st)
  if (cin == 20 && cout == 20) DFNO_MB(20, true);
  if (m <= 8) DFNO_MB(8, false);
  if (m <= 16) DFNO_MB(16, false);
  if (m <= 24) DFNO_MB(24, false);
  DFNO_MB(32, false);
#undef DFNO_MB
}

// ===========================================================================
// forward: pre[b][o][p] = sum_i f(src[b][i][p]) W[i][o]  (post = act(pre))
// reference _mix_layer_forward d/fno.py:286-289 -> einsum_channel_mix
// d/tensor.py:210-228, activation d/fno.py:41-46.  One thread per point of a
// 128-point tile: A = f(src) (128 points x K = i) in TMEM, B = W^T (o x i) in
// shared memory, D (points x o) read back by the owning thread.  Up to four
// CTAs per SM; the MMAs of tile t run while tile t + 1 is loaded.
// ===========================================================================
namespace {
constexpr uint32_t kMfTmemCols = 128;  // D 0..31 | A hi 32..63 | A lo 64..95
}

template <int CM, bool EXACT, int ACT>
__global__ void __launch_bounds__(kMbThreads, 4) k_mix_fwd_tc(long long npts, int nb, int cin_rt, int cout_rt,
                                                              const float* __restrict__ src, int src_act,
                                                              const float* __restrict__ w, float* __restrict__ pre,
                                                              float* __restrict__ post) {
  const int cin = EXACT ? CM : cin_rt, cout = EXACT ? CM : cout_rt;
  __shared__ __align__(1024) unsigned char b1[2 * 4096];  // W^T hi plane, lo plane (N = o <= 32, K = i <= 32)
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int KPi = (cin + 7) & ~7;    // K (i)
  const int NPo = (cout + 15) & ~15; // N (o)
  const int sbo = (KPi / 4) * 128;
  const int plane = (NPo / 8) * sbo;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < NPo * KPi; e += kMbThreads) {
    const int o = e / KPi, i = e % KPi;
    const float v = (i < cin && o < cout) ? w[(long long)i * cout + o] : 0.f;
    float h, l;
    tc::split_rn(v, h, l);
    const int off = (o >> 3) * sbo + (i >> 2) * 128 + (o & 7) * 16 + (i & 3) * 4;
    *reinterpret_cast<float*>(b1 + off) = h;
    *reinterpret_cast<float*>(b1 + plane + off) = l;
  }
  if (warp == 0) tc::tmem_alloc<kMfTmemCols>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t d = tmem, ah = tmem + 32, al = tmem + 64;
  const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
  const long long tiles_per_b = (npts + kMbThreads - 1) / kMbThreads;
  const long long ntiles = tiles_per_b * nb;

  float sv[CM];
  auto load = [&](long long tile) {
    const long long bb = tile / tiles_per_b;
    const long long p = (tile - bb * tiles_per_b) * kMbThreads + tid;
    const bool valid = tile < ntiles && p < npts;
    const float* s0 = src + (bb * cin) * npts + p;
#pragma unroll
    for (int i = 0; i < CM; ++i) {
      sv[i] = (valid && (EXACT || i < cin)) ? __ldcs(s0) : 0.f;
      s0 += npts;
    }
  };
  long long prev_out = -1;
  auto drain = [&]() {
    uint32_t r[32];
    tc::tmem_ld32_nowait(d + lane_off, r);
    tc::tmem_ld_wait();
    if (prev_out >= 0) {
#pragma unroll
      for (int o = 0; o < CM; ++o) {
        if (EXACT || o < cout) {
          const float v = __uint_as_float(r[o]);
          __stcs(pre + prev_out + (long long)o * npts, v);
          if (post) __stcs(post + prev_out + (long long)o * npts, act_apply<float>(ACT, v));
        }
      }
    }
  };
  int it = 0;
  load(blockIdx.x);
#pragma unroll 1
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const long long bb = tile / tiles_per_b;
    const long long p = (tile - bb * tiles_per_b) * kMbThreads + tid;
    float h[32], l[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i < CM) tc::split_hl(src_act ? act_apply<float>(ACT, sv[i]) : sv[i], h[i], l[i]);
      else h[i] = l[i] = 0.f;
    }
    load(tile + gridDim.x);
    if (it > 0) {
      tc::mbar_wait(&bar, (it - 1) & 1);
      tc::fence_after();
      drain();
    }
    tc::tmem_st32(ah + lane_off, h);
    tc::tmem_st32(al + lane_off, l);
    tc::tmem_st_wait();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      const uint32_t id = tc::idesc_tf32(128, NPo);
      const uint32_t sb = tc::smem_u32(b1);
      for (int s = 0; s < KPi / 8; ++s) {
        const uint64_t bh = tc::desc(sb + s * 256, 128, sbo), bl = tc::desc(sb + plane + s * 256, 128, sbo);
        tc::mma_tf32_ts(d, ah + 8 * s, bh, id, s > 0 ? 1u : 0u);
        tc::mma_tf32_ts(d, al + 8 * s, bh, id, 1u);
        tc::mma_tf32_ts(d, ah + 8 * s, bl, id, 1u);
      }
      tc::commit(&bar);
    }
    prev_out = (p < npts) ? (bb * cout * npts + p) : -1;
  }
  if (it > 0) {
    tc::mbar_wait(&bar, (it - 1) & 1);
    tc::fence_after();
    drain();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kMfTmemCols>(tmem);
}

// TMA-in / TMA-out variant of k_mix_fwd_tc.  Warp 4 streams (cin x 128-point)
// boxes of the input into a shared-memory ring; the four worker warps (thread
// = point) apply the source activation, split hi/lo and store A into TMEM,
// thread 0 issues the 3xTF32 MMAs into one of two TMEM accumulators, and the
// workers drain the OTHER accumulator (the previous tile) into a shared
// staging box that thread 0 writes back with a TMA tensor store one tile
// later.  One 128-thread barrier per tile; the MMA overlaps the drain and the
// next tile's loads, and no thread computes a global address.
constexpr int kMfMaxStages = 8;

template <int CM, bool EXACT, int ACT>
__global__ void __launch_bounds__(kMbThreads + 32, 4)
    k_mix_fwd_tma(long long npts, int nb, int cin_rt, int cout_rt, const __grid_constant__ CUtensorMap tm_src,
                  const __grid_constant__ CUtensorMap tm_pre, const __grid_constant__ CUtensorMap tm_post, int src_act,
                  const float* __restrict__ w, int has_post, int nstages, int nbuf) {
  const int cin = EXACT ? CM : cin_rt, cout = EXACT ? CM : cout_rt;
  // dynamic: ring[nstages][cin][128] | pre staging[2][cout][128] | post staging[2][cout][128]
  extern __shared__ __align__(1024) unsigned char dyn[];
  __shared__ __align__(1024) unsigned char b1[2 * 4096];
  __shared__ uint64_t bar, full[kMfMaxStages], empty[kMfMaxStages];
  __shared__ uint32_t tmem_base;
  const int KPi = (cin + 7) & ~7, NPo = (cout + 15) & ~15;
  const int sbo = (KPi / 4) * 128, plane = (NPo / 8) * sbo;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < NPo * KPi; e += blockDim.x) {
    const int o = e / KPi, i = e % KPi;
    const float v = (i < cin && o < cout) ? w[(long long)i * cout + o] : 0.f;
    float h, l;
    tc::split_rn(v, h, l);
    const int off = (o >> 3) * sbo + (i >> 2) * 128 + (o & 7) * 16 + (i & 3) * 4;
    *reinterpret_cast<float*>(b1 + off) = h;
    *reinterpret_cast<float*>(b1 + plane + off) = l;
  }
  if (warp == 0) tc::tmem_alloc<kMfTmemCols>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    for (int s = 0; s < nstages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], kMbThreads);
    }
    tc::mbar_fence_init();
    tc::tma_prefetch_desc(&tm_src);
    tc::tma_prefetch_desc(&tm_pre);
    if (has_post) tc::tma_prefetch_desc(&tm_post);
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // TMEM: D0 0..31 | A hi 32..63 | A lo 64..95 | D1 96..127
  const uint32_t tmem = tmem_base, ah = tmem + 32, al = tmem + 64;
  const long long tiles_per_b = (npts + kMbThreads - 1) / kMbThreads;
  const long long ntiles = tiles_per_b * nb;
  const int stage_bytes = cin * kMbThreads * 4, out_bytes = cout * kMbThreads * 4;
  unsigned char* ring = dyn;
  float* stage_pre = reinterpret_cast<float*>(dyn + nstages * stage_bytes);
  float* stage_post = reinterpret_cast<float*>(dyn + nstages * stage_bytes + nbuf * out_bytes);

  if (warp == 4) {
    // ---- TMA producer
    if ((tid & 31) == 0) {
      int j = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++j) {
        const int s = j % nstages, n = j / nstages;
        tc::mbar_wait_lazy(&empty[s], (n & 1) ^ 1, 64);
        const long long bb = tile / tiles_per_b;
        const int p0 = (int)((tile - bb * tiles_per_b) * kMbThreads);
        tc::mbar_expect_tx(&full[s], stage_bytes);
        tc::tma_load_2d(ring + s * stage_bytes, &tm_src, p0, (int)(bb * cin), &full[s]);
      }
    }
  } else {
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    auto dcol = [&](int k) { return tmem + ((k & 1) ? 96u : 0u); };
    // drain accumulator of tile k into staging buffer k&1
    auto drain = [&](int k) {
      uint32_t r[32];
      tc::tmem_ld32_nowait(dcol(k) + lane_off, r);
      tc::tmem_ld_wait();
      float* sp = stage_pre + (k & (nbuf - 1)) * (out_bytes / 4) + tid;
      float* sq = stage_post + (k & (nbuf - 1)) * (out_bytes / 4) + tid;
#pragma unroll
      for (int o = 0; o < CM; ++o) {
        if (EXACT || o < cout) {
          const float v = __uint_as_float(r[o]);
          sp[o * kMbThreads] = v;
          if (has_post) sq[o * kMbThreads] = act_apply<float>(ACT, v);
        }
      }
      tc::fence_proxy_async();
    };
    // TMA store of staged tile k (thread 0 only)
    auto store = [&](int k) {
      const long long tile = blockIdx.x + (long long)k * gridDim.x;
      const long long bb = tile / tiles_per_b;
      const int p0 = (int)((tile - bb * tiles_per_b) * kMbThreads), r0 = (int)(bb * cout);
      tc::tma_store_2d(&tm_pre, stage_pre + (k & (nbuf - 1)) * (out_bytes / 4), p0, r0);
      if (has_post) tc::tma_store_2d(&tm_post, stage_post + (k & (nbuf - 1)) * (out_bytes / 4), p0, r0);
      tc::bulk_commit();
    };
    int it = 0;
#pragma unroll 1
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int s = it % nstages, n = it / nstages;
      tc::mbar_wait(&full[s], n & 1);
      const float* row = reinterpret_cast<const float*>(ring + s * stage_bytes) + tid;
      float h[32], l[32];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        if (i < CM) {  // channel pairs (CM is even); act(0) = 0 keeps the padding zero
          float2 v = make_float2((EXACT || i < cin) ? row[i * kMbThreads] : 0.f,
                                 (EXACT || i + 1 < cin) ? row[(i + 1) * kMbThreads] : 0.f);
          if (src_act) v = act_apply2<ACT>(v);
          tc::split_hl2(v, h[i], h[i + 1], l[i], l[i + 1]);
        } else {
          h[i] = l[i] = h[i + 1] = l[i + 1] = 0.f;
        }
      }
      tc::mbar_arrive(&empty[s]);
      if (it > 0) {
        tc::mbar_wait(&bar, (it - 1) & 1);  // MMA it-1 done: A free, D(it-1) complete
        tc::fence_after();
      }
      tc::tmem_st32(ah + lane_off, h);
      tc::tmem_st32(al + lane_off, l);
      tc::tmem_st_wait();
      tc::fence_before();
      if (tid == 0) tc::bulk_wait_read0();  // store of tile it-3 has left staging buffer (it-1)&1
      tc::named_sync(1, kMbThreads);
      if (tid == 0) {
        tc::fence_after();
        const uint32_t id = tc::idesc_tf32(128, NPo);
        const uint32_t sb = tc::smem_u32(b1);
        const uint32_t d = dcol(it);
        // lo products first, hi.hi last: the accumulator's non-round-to-nearest
        // adds bias only the KPi / 8 full-magnitude sums
        for (int k = 0; k < KPi / 8; ++k) {
          const uint64_t bh = tc::desc(sb + k * 256, 128, sbo), bl = tc::desc(sb + plane + k * 256, 128, sbo);
          tc::mma_tf32_ts(d, al + 8 * k, bh, id, k > 0 ? 1u : 0u);
          tc::mma_tf32_ts(d, ah + 8 * k, bl, id, 1u);
        }
        for (int k = 0; k < KPi / 8; ++k) tc::mma_tf32_ts(d, ah + 8 * k, tc::desc(sb + k * 256, 128, sbo), id, 1u);
        tc::commit(&bar);
        if (nbuf == 2 && it >= 2) store(it - 2);  // staged by every worker before the barrier above
      }
      if (it > 0) {
        drain(it - 1);
        if (nbuf == 1) {  // single staging buffer: store it now; the next drain waits for its read
          tc::named_sync(1, kMbThreads);
          if (tid == 0) store(it - 1);
        }
      }
    }
    if (it > 0) {
      tc::mbar_wait(&bar, (it - 1) & 1);
      tc::fence_after();
      if (tid == 0) tc::bulk_wait_read0();
      tc::named_sync(1, kMbThreads);
      if (tid == 0 && nbuf == 2 && it >= 2) store(it - 2);
      drain(it - 1);
      tc::named_sync(1, kMbThreads);
      if (tid == 0) {
        store(it - 1);
        tc::bulk_wait0();
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kMfTmemCols>(tmem);
}

template <int CM, bool EXACT, int ACT>
static int launch_mix_fwd_tc3(long long npts, int nb, int cin, int cout, const void* src, int src_act, const void* w,
                              void* pre, void* post, cudaStream_t st) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long tiles = ((npts + kMbThreads - 1) / kMbThreads) * nb;
  CUtensorMap tm_src, tm_pre, tm_post;
  if (make_rows_map(&tm_src, src, npts, (long long)nb * cin, cin) &&
      make_rows_map(&tm_pre, pre, npts, (long long)nb * cout, cout) &&
      (!post || make_rows_map(&tm_post, post, npts, (long long)nb * cout, cout))) {
    if (!post) tm_post = tm_pre;
    // per-CTA dynamic shared memory: ring + double-buffered output staging;
    // up to 4 CTAs per SM (the TMEM limit at 128 columns each) while a ring
    // of >= 2 stages fits
    const int stage_bytes = cin * kMbThreads * 4, out_one = cout * kMbThreads * 4 * (post ? 2 : 1);
    const int static_bytes = 2 * 4096 + 256;
    int per_sm = 4, stages = 0, nbuf = 2;
    for (; per_sm >= 1; --per_sm) {  // double-buffered staging first, then single
      for (nbuf = 2; nbuf >= 1; --nbuf) {
        stages = ((227 * 1024) / per_sm - 1024 - static_bytes - nbuf * out_one) / stage_bytes;
        if (stages >= 2) break;
      }
      if (stages >= 2) break;
    }
    if (stages > 4) stages = 4;
    if (per_sm >= 1 && stages >= 2) {
      const int smem = stages * stage_bytes + nbuf * out_one;
      auto kt = k_mix_fwd_tma<CM, EXACT, ACT>;
      if (cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess) {
        const long long grid = tiles < (long long)per_sm * sms ? tiles : (long long)per_sm * sms;
        kt<<<(unsigned)grid, kMbThreads + 32, smem, st>>>(npts, nb, cin, cout, tm_src, tm_pre, tm_post, src_act,
                                                          (const float*)w, post ? 1 : 0, stages, nbuf);
        DFNO_CUDA_CHECK_LAUNCH();
        return DFNO_OK;
      }
    }
  }
  const long long blocks = tiles < 4LL * sms ? tiles : 4LL * sms;
  k_mix_fwd_tc<CM, EXACT, ACT><<<(unsigned)blocks, kMbThreads, 0, st>>>(npts, nb, cin, cout, (const float*)src, src_act,
                                                                        (const float*)w, (float*)pre, (float*)post);
  DFNO_CUDA_CHECK_LAUNCH();
  return DFNO_OK;
}

template <int CM, bool EXACT>
static int launch_mix_fwd_tc(long long npts, int nb, int cin, int cout, const void* src, int src_act, int act,
                             const void* w, void* pre, void* post, cudaStream_t st) {
  switch (act) {
    case DFNO_ACT_GELU:
      return launch_mix_fwd_tc3<CM, EXACT, DFNO_ACT_GELU>(npts, nb, cin, cout, src, src_act, w, pre, post, st);
    case DFNO_ACT_RELU:
      return launch_mix_fwd_tc3<CM, EXACT, DFNO_ACT_RELU>(npts, nb, cin, cout, src, src_act, w, pre, post, st);
    default:
      return launch_mix_fwd_tc3<CM, EXACT, DFNO_ACT_IDENTITY>(npts, nb, cin, cout, src, src_act, w, pre, post, st);
  }
}

// fp32, cin and cout <= 32; returns DFNO_ERR_UNSUPPORTED otherwise.
int mix_fwd_tc(long long npts, int nb, int cin, int cout, const void* src, int src_act, int act, const void* w,
               void* pre, void* post, cudaStream_t st) {
  const int m = cin > cout ? cin : cout;
  if (m > 32 || npts < 1) return DFNO_ERR_UNSUPPORTED;
#define DFNO_MF(CM, EX) return launch_mix_fwd_tc<CM, EX>(npts, nb, cin, cout, src, src_act, act, w, pre, post, st)
  if (cin == 20 && cout == 20) DFNO_MF(20, true);
  if (m <= 8) DFNO_MF(8, false);
  if (m <= 16) DFNO_MF(16, false);
  if (m <= 24) DFNO_MF(24, false);
  DFNO_MF(32, false);
#undef DFNO_MF
}

}  // namespace dfno
