// Hardware probe for the tcgen05 building blocks used by dft_yzt_tc.cu:
// one CTA stages A (M x K) and B (N x K) into SWIZZLE_NONE K-major layouts with
// caller-chosen LBO / SBO, issues K/8 kind::tf32 MMAs (descriptor start
// advanced by 2*LBO per K step), waits on tcgen05.commit, and reads D back
// with tcgen05.ld.32x32b.  Test-only (tests/test_gpu_tc_probe.py).
#include <cuda_runtime.h>
#include <stdint.h>
#include "tc.cuh"

using namespace dfno;

__global__ void probe(const float* A, const float* B, float* D, int M, int N, int K, int lbo_a, int sbo_a,
                      int lbo_b, int sbo_b, int neg_b, int accumulate_twice) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  float* sa = reinterpret_cast<float*>(smem);
  const int a_bytes = (M / 8) * sbo_a;
  float* sb = reinterpret_cast<float*>(smem + ((a_bytes + 1023) / 1024) * 1024);
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    int off = (r / 8) * sbo_a + (k / 4) * lbo_a + (r % 8) * 16 + (k % 4) * 4;
    sa[off / 4] = A[e];
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    int off = (r / 8) * sbo_b + (k / 4) * lbo_b + (r % 8) * 16 + (k % 4) * 4;
    sb[off / 4] = B[e];
  }
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&tbase);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t d = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_tf32(M, N, false, neg_b != 0);
    for (int rep = 0; rep < (accumulate_twice ? 2 : 1); ++rep)
      for (int s = 0; s < K / 8; ++s) {
        uint64_t da = tc::desc(tc::smem_u32(sa) + 2 * s * lbo_a, lbo_a, sbo_a);
        uint64_t db = tc::desc(tc::smem_u32(sb) + 2 * s * lbo_b, lbo_b, sbo_b);
        tc::mma_tf32(d, da, db, idesc, (rep | s) ? 1u : 0u);
      }
    tc::commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (w < 4 && 32 * w < M) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tc::tmem_ld16(d + ((uint32_t)(32 * w) << 16) + c0, v);
      for (int j = 0; j < 16; ++j) D[(32 * w + lane) * N + c0 + j] = v[j];
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tbase);
}

extern "C" int probe_run(const float* A, const float* B, float* D, int M, int N, int K, int lbo_a, int sbo_a,
                         int lbo_b, int sbo_b, int neg_b, int twice) {
  int smem = 64 * 1024 + 64 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(A, B, D, M, N, K, lbo_a, sbo_a, lbo_b, sbo_b, neg_b, twice);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}

// MN-major A (SWIZZLE_NONE): core matrix = 8 K rows x 4 M elements (128 B),
// element (r, k) at (r / 4) * sbo_a + (k / 8) * lbo_a + (k % 8) * 16 + (r % 4) * 4;
// one K group (8) per MMA, advanced by lbo_a.  B K-major as above.
__global__ void probe_mn(const float* A, const float* B, float* D, int M, int N, int K, int lbo_a, int sbo_a,
                         int lbo_b, int sbo_b, int sw) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  float* sa = reinterpret_cast<float*>(smem);
  float* sb = reinterpret_cast<float*>(smem + 64 * 1024);
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    // sw: element (r, k) of a SWIZZLE_128B MN-major atom stack: MN atoms of 32
    // (LBO apart), K groups of 8 rows (SBO apart), 16-byte chunk ^ (k % 8)
    // sw 3: SWIZZLE_128B_BASE32B (the 32-bit MN-major canonical form): MN atoms
    // of 32 (LBO apart) x K groups of 4 rows of 128 B (SBO apart), 32-byte chunk ^ (k % 4)
    int off = sw == 3 ? (r / 32) * lbo_a + (k / 4) * sbo_a + (k % 4) * 128 + ((((r % 32) / 8) ^ (k % 4)) * 32) + (r % 8) * 4
            : sw ? (r / 32) * lbo_a + (k / 8) * sbo_a + (k % 8) * 128 + ((((r % 32) / 4) ^ (k % 8)) * 16) + (r % 4) * 4
                 : (r / 4) * sbo_a + (k / 8) * lbo_a + (k % 8) * 16 + (r % 4) * 4;
    sa[off / 4] = A[e];
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    int off = (r / 8) * sbo_b + (k / 4) * lbo_b + (r % 8) * 16 + (k % 4) * 4;
    sb[off / 4] = B[e];
  }
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&tbase);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t d = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_tf32(M, N, false, false, sw != 2);  // sw 2: control, K-major bit
    for (int s = 0; s < K / 8; ++s) {
      uint64_t da = sw == 3 ? (tc::desc(tc::smem_u32(sa) + 2 * s * sbo_a, lbo_a, sbo_a) | ((uint64_t)1 << 61))
                    : sw ? (tc::desc(tc::smem_u32(sa) + s * sbo_a, lbo_a, sbo_a) | ((uint64_t)2 << 61))
                         : tc::desc(tc::smem_u32(sa) + s * lbo_a, lbo_a, sbo_a);
      uint64_t db = tc::desc(tc::smem_u32(sb) + 2 * s * lbo_b, lbo_b, sbo_b);
      tc::mma_tf32(d, da, db, idesc, s ? 1u : 0u);
    }
    tc::commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (w < 4 && 32 * w < M) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tc::tmem_ld16(d + ((uint32_t)(32 * w) << 16) + c0, v);
      for (int j = 0; j < 16; ++j) D[(32 * w + lane) * N + c0 + j] = v[j];
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tbase);
}

extern "C" int probe_run_mn(const float* A, const float* B, float* D, int M, int N, int K, int lbo_a, int sbo_a,
                            int lbo_b, int sbo_b, int sw) {
  int smem = 64 * 1024 + 64 * 1024;
  cudaFuncSetAttribute(probe_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_mn<<<1, 128, smem>>>(A, B, D, M, N, K, lbo_a, sbo_a, lbo_b, sbo_b, sw);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
