// C ABI entry points of libdfno.so (declared in include/dfno.h): argument
// validation, status strings, buffer sizing and kernel dispatch.
#include <string.h>

#include "common.cuh"

namespace dfno {
template <typename R>
int yzt_fwd_simt(const dfno_geom&, const void*, const void*, int, double, void*, cudaStream_t);
template <typename R>
int yzt_inv_simt(const dfno_geom&, const void*, double, void*, cudaStream_t);
template <typename R>
int xspec_fwd_simt(const dfno_geom&, const void*, const void*, void*, void*, cudaStream_t);
template <typename R>
int xspec_bwd_simt(const dfno_geom&, const void*, const void*, const void*, void*, void*, cudaStream_t);
// tcgen05 paths (dft_fwd_tc.cu, dft_inv_tc3.cu); DFNO_ERR_UNSUPPORTED outside
// their envelope (r > 16 or shared memory), which the SIMT kernels cover
int yzt_fwd_tc2(const dfno_geom&, const void*, const void*, int, double, void*, cudaStream_t);
int yzt_inv_tc3(const dfno_geom&, const void*, double, void*, cudaStream_t);
// streamed x-spectral stage (xspec_stream.cu)
size_t xspec_stream_workspace(const dfno_geom&);
int xspec_fwd_stream(const dfno_geom&, const void*, const void*, void*, void*, void*, cudaStream_t);
int xspec_bwd_stream(const dfno_geom&, const void*, const void*, const void*, void*, void*, void*, cudaStream_t);
int xdft_stage(const dfno_geom&, const void*, float, void*, cudaStream_t);
int xidft_stage(const dfno_geom&, const void*, float, void*, cudaStream_t);
int xmix_fwd_stage(const dfno_geom&, const void*, const void*, void*, cudaStream_t);
int xmix_bwd_stage(const dfno_geom&, const void*, const void*, const void*, void*, void*, cudaStream_t);
}  // namespace dfno

using namespace dfno;

namespace {

int retained(int n, int m) { return (2 * m < n) ? 2 * m : n; }

// Remainder-first block boundaries (reference d/partition.py:47-66).
bool check_blocks(const int32_t* starts, int extent, int P) {
  if (P < 1 || P > extent) return false;
  const int base = extent / P, rem = extent % P;
  int cur = 0;
  for (int r = 0; r < P; ++r) {
    if (starts[r] != cur) return false;
    cur += base + (r < rem ? 1 : 0);
  }
  return starts[P] == extent;
}

}  // namespace

extern "C" int dfno_abi_version(void) { return DFNO_ABI_VERSION; }

extern "C" const char* dfno_build_info(void) {
#define DFNO_STR2(x) #x
#define DFNO_STR(x) DFNO_STR2(x)
  return "libdfno sm_100a (tcgen05 3xTF32 yzt DFT; SIMT fp32/fp64 generic path), nvcc " DFNO_STR(
      __CUDACC_VER_MAJOR__) "." DFNO_STR(__CUDACC_VER_MINOR__);
}

extern "C" const char* dfno_status_string(int status) {
  switch (status) {
    case DFNO_OK: return "ok";
    case DFNO_ERR_DIMENSION: return "dimension mismatch";
    case DFNO_ERR_DTYPE: return "dtype mismatch (real32 / real64 only)";
    case DFNO_ERR_INFEASIBLE: return "infeasible partition";
    case DFNO_ERR_SHAPE: return "shape mismatch";
    case DFNO_ERR_NULL: return "null pointer argument";
    case DFNO_ERR_CUDA: return "CUDA launch failure";
    case DFNO_ERR_UNSUPPORTED: return "geometry outside the kernel envelope";
    default: return "unknown status";
  }
}

// Feasibility rules of FnoConfig.__post_init__ (reference d/fno.py:77-96).
extern "C" int dfno_geom_validate(const dfno_geom* g) {
  if (!g) return DFNO_ERR_NULL;
  if (g->dtype != DFNO_F32 && g->dtype != DFNO_F64) return DFNO_ERR_DTYPE;
  if (g->batch < 0 || g->c_in < 1 || g->c < 1 || g->c_out < 1) return DFNO_ERR_DIMENSION;
  if (g->nx < 1 || g->ny < 1 || g->nz < 1 || g->nt < 1) return DFNO_ERR_DIMENSION;
  if (g->mx < 1 || g->my < 1 || g->mz < 1 || g->mt < 1) return DFNO_ERR_DIMENSION;
  if (g->act < DFNO_ACT_RELU || g->act > DFNO_ACT_IDENTITY) return DFNO_ERR_DIMENSION;
  if (g->rx != retained(g->nx, g->mx) || g->ry != retained(g->ny, g->my) || g->rz != retained(g->nz, g->mz) ||
      g->rt != retained(g->nt, g->mt))
    return DFNO_ERR_SHAPE;
  if (g->nranks < 1 || g->nranks > DFNO_MAX_RANKS) return DFNO_ERR_INFEASIBLE;
  if (g->nranks > g->nx || g->nranks > g->ry) return DFNO_ERR_INFEASIBLE;
  if (g->rank < 0 || g->rank >= g->nranks) return DFNO_ERR_SHAPE;
  if (!check_blocks(g->x_starts, g->nx, g->nranks)) return DFNO_ERR_SHAPE;
  if (!check_blocks(g->ky_starts, g->ry, g->nranks)) return DFNO_ERR_SHAPE;
  return DFNO_OK;
}

extern "C" int dfno_sizes(const dfno_geom* g, int64_t* xk_elems, int64_t* kx_elems, int64_t* spec_elems,
                          int64_t* wshard_elems) {
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  const int64_t rzt = (int64_t)g->rz * g->rt;
  const int64_t XL = x_local(*g), KYL = ky_local(*g);
  if (xk_elems) *xk_elems = (int64_t)g->batch * g->c * XL * g->ry * rzt;
  if (kx_elems) *kx_elems = (int64_t)g->batch * g->c * g->nx * KYL * rzt;
  if (spec_elems) *spec_elems = (int64_t)g->batch * g->c * g->rx * KYL * rzt;
  if (wshard_elems) *wshard_elems = (int64_t)g->c * g->c * g->rx * KYL * rzt;
  return DFNO_OK;
}

extern "C" int dfno_dft_yzt_fwd(const dfno_geom* g, const void* src, const void* pre, int src_mode, double scale,
                                void* xk_out, void* stream) {
  if (!g || !src || !xk_out) return DFNO_ERR_NULL;
  int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (src_mode == DFNO_SRC_GRAD && !pre) return DFNO_ERR_NULL;
  if (src_mode < DFNO_SRC_ACT || src_mode > DFNO_SRC_RAW) return DFNO_ERR_DIMENSION;
  if (g->batch == 0) return DFNO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->dtype == DFNO_F32) {
    rc = yzt_fwd_tc2(*g, src, pre, src_mode, scale, xk_out, st);
    if (rc != DFNO_ERR_UNSUPPORTED) return rc;
    return yzt_fwd_simt<float>(*g, src, pre, src_mode, scale, xk_out, st);
  }
  return yzt_fwd_simt<double>(*g, src, pre, src_mode, scale, xk_out, st);
}

extern "C" int dfno_dft_yzt_inv(const dfno_geom* g, const void* xk_in, double scale, void* out, void* stream) {
  if (!g || !xk_in || !out) return DFNO_ERR_NULL;
  int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->dtype == DFNO_F32) {
    rc = yzt_inv_tc3(*g, xk_in, scale, out, st);
    if (rc != DFNO_ERR_UNSUPPORTED) return rc;
    return yzt_inv_simt<float>(*g, xk_in, scale, out, st);
  }
  return yzt_inv_simt<double>(*g, xk_in, scale, out, st);
}

extern "C" int dfno_xspec_fwd(const dfno_geom* g, const void* kx_in, const void* w, void* spec, void* kx_out,
                              void* stream) {
  if (!g || !kx_in || !w || !kx_out) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->dtype == DFNO_F32) return xspec_fwd_simt<float>(*g, kx_in, w, spec, kx_out, st);
  return xspec_fwd_simt<double>(*g, kx_in, w, spec, kx_out, st);
}

extern "C" int dfno_xspec_bwd(const dfno_geom* g, const void* kx_in, const void* spec, const void* w, void* gw,
                              void* kx_out, void* stream) {
  if (!g || !kx_in || !spec || !w || !gw || !kx_out) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->dtype == DFNO_F32) return xspec_bwd_simt<float>(*g, kx_in, spec, w, gw, kx_out, st);
  return xspec_bwd_simt<double>(*g, kx_in, spec, w, gw, kx_out, st);
}

extern "C" int dfno_xspec_workspace(const dfno_geom* g, int64_t* bytes) {
  if (!g || !bytes) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  *bytes = (int64_t)xspec_stream_workspace(*g);
  return DFNO_OK;
}

extern "C" int dfno_xspec_fwd_ws(const dfno_geom* g, const void* kx_in, const void* w, void* spec, void* kx_out,
                                 void* work, void* stream) {
  if (!g || !kx_in || !w || !kx_out || !work) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  const int r2 = xspec_fwd_stream(*g, kx_in, w, spec, kx_out, work, (cudaStream_t)stream);
  if (r2 != DFNO_ERR_UNSUPPORTED) return r2;
  return dfno_xspec_fwd(g, kx_in, w, spec, kx_out, stream);
}

extern "C" int dfno_xspec_bwd_ws(const dfno_geom* g, const void* kx_in, const void* spec, const void* w, void* gw,
                                 void* kx_out, void* work, void* stream) {
  if (!g || !kx_in || !spec || !w || !gw || !kx_out || !work) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  const int r2 = xspec_bwd_stream(*g, kx_in, spec, w, gw, kx_out, work, (cudaStream_t)stream);
  if (r2 != DFNO_ERR_UNSUPPORTED) return r2;
  return dfno_xspec_bwd(g, kx_in, spec, w, gw, kx_out, stream);
}

// ---- the x-spectral stage by parts (fp32): lets the caller pipeline the
// x-DFTs of channel groups against the exchanges (fno.py)
extern "C" int dfno_xdft(const dfno_geom* g, const void* kx_in, double scale, void* X, void* stream) {
  if (!g || !kx_in || !X) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  return xdft_stage(*g, kx_in, (float)scale, X, (cudaStream_t)stream);
}

extern "C" int dfno_xidft(const dfno_geom* g, const void* Y, double scale, void* kx_out, void* stream) {
  if (!g || !Y || !kx_out) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  return xidft_stage(*g, Y, (float)scale, kx_out, (cudaStream_t)stream);
}

extern "C" int dfno_xmix_fwd(const dfno_geom* g, const void* X, const void* w, void* Y, void* stream) {
  if (!g || !X || !w || !Y) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  return xmix_fwd_stage(*g, X, w, Y, (cudaStream_t)stream);
}

extern "C" int dfno_xmix_bwd(const dfno_geom* g, const void* spec, const void* D, const void* w, void* gw, void* dX,
                             void* stream) {
  if (!g || !spec || !D || !w || !gw || !dX) return DFNO_ERR_NULL;
  const int rc = dfno_geom_validate(g);
  if (rc != DFNO_OK) return rc;
  if (g->batch == 0) return DFNO_OK;
  return xmix_bwd_stage(*g, spec, D, w, gw, dX, (cudaStream_t)stream);
}
