// Tensor-map (TMA descriptor) encoding without a link-time dependency on
// libcuda: cuTensorMapEncodeTiled is resolved through the runtime's driver
// entry-point query, so libdfno.so still loads (and its host-only entry
// points work) on machines without a GPU driver.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

namespace dfno {

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 4-D fp32 map over (t, z, y, slab) of a (slabs, Ny, Nz, Nt) tensor, box
// (32, 16, 8, 1), 128-byte swizzle, out-of-bounds elements zero-filled on
// load and dropped on store.
inline bool make_slab_map(CUtensorMap* m, const void* base, int ny, int nz, int nt, int slabs,
                          CUtensorMapL2promotion l2) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)nt, (cuuint64_t)nz, (cuuint64_t)ny, (cuuint64_t)slabs};
  cuuint64_t strides[3] = {(cuuint64_t)nt * 4, (cuuint64_t)nz * nt * 4, (cuuint64_t)ny * nz * nt * 4};
  cuuint32_t box[4] = {32, 16, 8, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// N_t % 4 == 2 (the CO2 grid's 86) with N_z even: a row stride of N_t floats
// is not 16-byte aligned, but two rows are.  Two 4-D maps over (t, z pair, y,
// slab) with row stride 2 N_t: the even map starts at the tensor, the odd map
// 2 floats before the first odd row (16-byte aligned), with inner extent
// N_t + 2, so inner coordinate c is element c - 2 of an odd row.  Box (36, 8,
// 8, 1), no swizzle: a 32-t block of an odd row sits 8 bytes into its 144-byte
// line.  Out-of-range t, z and y are zero-filled by the map bounds.
inline bool make_slab_pair_maps(CUtensorMap* even, CUtensorMap* odd, const void* base, int ny, int nz, int nt,
                                int slabs) {
  auto enc = tensor_map_encoder();
  if (!enc || nt % 4 != 2 || nz % 2 != 0 || ((uintptr_t)base & 15)) return false;
  cuuint64_t strides[3] = {(cuuint64_t)2 * nt * 4, (cuuint64_t)nz * nt * 4, (cuuint64_t)ny * nz * nt * 4};
  cuuint32_t box[4] = {36, 8, 8, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  cuuint64_t de[4] = {(cuuint64_t)nt, (cuuint64_t)(nz / 2), (cuuint64_t)ny, (cuuint64_t)slabs};
  cuuint64_t dodd[4] = {(cuuint64_t)nt + 2, (cuuint64_t)(nz / 2), (cuuint64_t)ny, (cuuint64_t)slabs};
  const char* ob = static_cast<const char*>(base) + (nt - 2) * 4;
  return enc(even, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), de, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
         enc(odd, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<char*>(ob), dodd, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D fp32 map over (point, row) of a (rows, npts) tensor, box (128, box_rows),
// no swizzle: rows of a channel-major activation viewed as (b * c, points).
inline bool make_rows_map(CUtensorMap* m, const void* base, long long npts, long long rows, int box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc || (npts * 4) % 16 != 0 || ((uintptr_t)base & 15) || box_rows > 256) return false;
  cuuint64_t dims[2] = {(cuuint64_t)npts, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)npts * 4};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace dfno
