// tcgen05 (5th-generation tensor core) path for the truncated yzt DFT.
// Placeholder until the 3xTF32 kernels land: reports the geometry as outside
// its envelope so dispatch uses the SIMT kernels.
#include "common.cuh"

namespace dfno {
int yzt_fwd_tc(const dfno_geom&, const void*, const void*, int, double, void*, cudaStream_t) {
  return DFNO_ERR_UNSUPPORTED;
}
int yzt_inv_tc(const dfno_geom&, const void*, double, void*, cudaStream_t) { return DFNO_ERR_UNSUPPORTED; }
}  // namespace dfno
