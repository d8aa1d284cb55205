// Where does a cta_group::1 kind::tf32 MMA with M = 64 put its accumulator
// rows in TMEM?  A[r][0] = r + 1, B[n][0] = 1000 (n + 1), all other K zero, so
// D[r][n] = 1000 (r + 1)(n + 1) names its own row and column.  Four warps read
// all 128 lanes x 64 columns; the host prints the (lane, column) -> (row, n)
// map.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -I include
// -I paper_2211_12709_b200/csrc tools/probes/mma_m64_probe.cu -o /tmp/m64
#include <cstdio>
#include <vector>

#include "tc.cuh"

using namespace dfno;

__global__ void probe(float* out, int M) {
  __shared__ __align__(1024) unsigned char sa[128 * 32];
  __shared__ __align__(1024) unsigned char sb[64 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  auto off = [](int r, int k) { return (r >> 3) * 256 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4; };
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    const int r = e / 8, k = e % 8;
    *reinterpret_cast<float*>(sa + off(r, k)) = (k == 0 && r < M) ? (float)(r + 1) : 0.f;
    if (r < 64) *reinterpret_cast<float*>(sb + off(r, k)) = k == 0 ? 1000.f * (r + 1) : 0.f;
  }
  if (warp == 0) tc::tmem_alloc<128>(&tbase);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  // clear the accumulator columns so stale TMEM cannot masquerade as output
  {
    float z[32];
    for (int j = 0; j < 32; ++j) z[j] = -1.f;
    tc::tmem_st32(tmem + ((uint32_t)(32 * warp) << 16), z);
    tc::tmem_st32(tmem + 32 + ((uint32_t)(32 * warp) << 16), z);
    tc::tmem_st_wait();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (tid == 0) {
    tc::mma_tf32(tmem, tc::desc(tc::smem_u32(sa), 128, 256), tc::desc(tc::smem_u32(sb), 128, 256),
                 tc::idesc_tf32(M, 64), 0u);
    tc::commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  uint32_t r0[32], r1[32];
  tc::tmem_ld32_nowait(tmem + ((uint32_t)(32 * warp) << 16), r0);
  tc::tmem_ld32_nowait(tmem + 32 + ((uint32_t)(32 * warp) << 16), r1);
  tc::tmem_ld_wait();
  for (int c = 0; c < 32; ++c) {
    out[tid * 64 + c] = __uint_as_float(r0[c]);
    out[tid * 64 + 32 + c] = __uint_as_float(r1[c]);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<128>(tmem);
}

int main() {
  for (int M : {128, 64}) {
    float* d;
    cudaMalloc(&d, 128 * 64 * 4);
    probe<<<1, 128>>>(d, M);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> h(128 * 64);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    printf("M = %d (%s)\n", M, cudaGetErrorString(e));
    for (int lane = 0; lane < 128; ++lane) {
      int first = -1, cnt = 0;
      for (int c = 0; c < 64; ++c)
        if (h[lane * 64 + c] > 0.f) {
          if (first < 0) first = c;
          ++cnt;
        }
      if (cnt) {
        const float v = h[lane * 64 + first];
        const int n = first;  // expect D[row][n] = 1000 (row + 1)(n + 1)
        printf("  lane %3d: %2d cols from col %2d, row = %.1f (col %d / n+1 = %.0f)\n", lane, cnt, first,
               v / (1000.f * (n + 1)) - 1.f, n, v / 1000.f / (h[lane * 64 + first] / (1000.f * (n + 1))));
      }
    }
    cudaFree(d);
  }
  return 0;
}
