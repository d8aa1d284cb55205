// Probe: 4-D TMA load with a grouped-row view (dims (G*nt, nz/G, ny, slabs)).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2211_12709_b200/csrc/tmap.cuh"
__global__ void k(const __grid_constant__ CUtensorMap tm, int c0, int c1, int bytes, float* out) {
  __shared__ __align__(1024) float buf[4096];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"((uint32_t)__cvta_generic_to_shared(buf)), "l"(&tm), "r"(c0), "r"(c1), "r"(0), "r"(0), "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = buf[i];
}
int main() {
  int cases[][4] = {{30, 20, 22, 4}, {118, 64, 86, 4}, {64, 64, 32, 4}};
  for (auto& cs : cases) {
    int ny = cs[0], nz = cs[1], nt = cs[2], slabs = cs[3];
    size_t n = (size_t)ny * nz * nt * slabs;
    float* d; cudaMalloc(&d, n * 4); float* o; cudaMalloc(&o, 4096 * 4);
    CUtensorMap m;
    bool ok = dfno::make_slab_map(&m, d, ny, nz, nt, slabs, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    int G = dfno::slab_group(nz, nt);
    for (int c0 : {0, nt, 64}) {
      k<<<1, 128>>>(m, c0, 0, 16384 / G, o);
      cudaError_t e = cudaDeviceSynchronize();
      printf("ny %d nz %d nt %d G %d encode %d c0 %d -> %s\n", ny, nz, nt, G, ok, c0, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  }
}
