/*
 * dfno.h -- C ABI of libdfno.so, the sm_100a implementation of the
 * domain-decomposed 4-D Fourier neural operator hot path of arXiv 2211.12709
 * (reference package `distfno`, /root/reference/pkg/src/distfno).
 *
 * Every entry point replaces one numpy stage of the reference's rank-local
 * pipeline; the reference line each one stands in for is cited above it.
 * The reference itself has no FFI (pure Python); INTEGRATION.md shows the
 * ctypes binding a maintainer would add to distfno to call these.
 *
 * Conventions
 *  - All data pointers are DEVICE pointers owned by the caller.  Nothing here
 *    allocates, frees or synchronises; every call enqueues on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).
 *  - Real tensors are row-major (b, ch, x, y, z, t), t fastest (reference
 *    d/tensor.py:1-6, d/bench.py:57).  Complex tensors are interleaved
 *    (re, im) pairs of the real dtype (complex64 / complex128).
 *  - Packed exchange buffers are PEER-MAJOR: chunk p is the contiguous block
 *    this rank sends to (or receives from) rank p in the x<->ky repartition
 *    (reference d/partition.py:135-188, d/comm.py:421-483).  Layouts:
 *      XK layout (yzt-forward output / yzt-inverse input), chunk p =
 *          [b][c][x_local][ky in ky_range(p)][rz][rt]
 *      KX layout (x-spectral input and output), chunk p =
 *          [b][c][x in x_range(p)][ky_local][rz][rt]
 *    At P == 1 both are the reference's (b, c, x, ky, kz, kt) tensor.
 *  - Retained mode j along a dim of extent N with m modes is frequency
 *    j (j < m) or N - 2m + j (j >= m); identity when 2m >= N
 *    (reference d/spectral.py:55-66).
 *  - Return value: DFNO_OK (0) or a negative DFNO_ERR_* code;
 *    dfno_status_string() describes it.  The Python layer maps codes onto the
 *    reference's exception classes (d/errors.py).
 */
#ifndef DFNO_H
#define DFNO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFNO_ABI_VERSION 1
#define DFNO_MAX_RANKS 64

/* status codes -> reference exception (d/errors.py) */
#define DFNO_OK 0
#define DFNO_ERR_DIMENSION (-1)   /* DimensionMismatchError  d/errors.py:10 */
#define DFNO_ERR_DTYPE (-2)       /* DTypeMismatchError      d/errors.py:14 */
#define DFNO_ERR_INFEASIBLE (-3)  /* InfeasiblePartitionError d/errors.py:40 */
#define DFNO_ERR_SHAPE (-4)       /* ShapeMismatchError      d/errors.py:44 */
#define DFNO_ERR_NULL (-5)        /* null pointer argument (DistFnoError) */
#define DFNO_ERR_CUDA (-6)        /* kernel launch failure (DistFnoError) */
#define DFNO_ERR_UNSUPPORTED (-7) /* shape outside the kernel's envelope */

/* dtype codes: reference DType.REAL32 / REAL64 (d/tensor.py:78-82) */
#define DFNO_F32 0
#define DFNO_F64 1

/* activation codes: reference ActivationKind (d/fno.py:36-55) */
#define DFNO_ACT_RELU 0
#define DFNO_ACT_GELU 1
#define DFNO_ACT_IDENTITY 2

/* yzt transform input modes */
#define DFNO_SRC_ACT 0      /* forward: act(src)                d/fno.py:372 */
#define DFNO_SRC_GRAD 1     /* backward: src * act'(pre)        d/fno.py:491 */
#define DFNO_SRC_RAW 2      /* src as is                        d/fno.py:328 */

/*
 * Rank geometry.  Mirrors FnoConfig (d/fno.py:62-132) plus the rank's view of
 * Partition.block(x, nx, P) and Partition.block(ky, ry, P)
 * (d/partition.py:47-66, d/fno.py:124-128).  x_starts / ky_starts hold the
 * P+1 block boundaries (remainder-first, d/partition.py:47-66).
 */
typedef struct dfno_geom {
  int32_t batch;
  int32_t c_in, c, c_out;          /* in / hidden / out channels */
  int32_t nx, ny, nz, nt;          /* global grid */
  int32_t mx, my, mz, mt;          /* retained mode counts per dim */
  int32_t rx, ry, rz, rt;          /* retained extents min(2m, N) */
  int32_t nranks, rank;
  int32_t dtype;                   /* DFNO_F32 / DFNO_F64 */
  int32_t act;                     /* DFNO_ACT_* */
  int32_t x_starts[DFNO_MAX_RANKS + 1];
  int32_t ky_starts[DFNO_MAX_RANKS + 1];
} dfno_geom;

/* ABI / build identification */
int dfno_abi_version(void);
const char* dfno_status_string(int status);
const char* dfno_build_info(void);

/* Validate a geometry (the feasibility rules of FnoConfig.__post_init__,
 * d/fno.py:77-96, and remainder-first partitions, d/partition.py:47-66). */
int dfno_geom_validate(const dfno_geom* g);

/* Element counts of the packed exchange buffers and caches (complex
 * elements; multiply by 2 * sizeof(real) for bytes). */
int dfno_sizes(const dfno_geom* g, int64_t* xk_elems, int64_t* kx_elems,
               int64_t* spec_elems, int64_t* wshard_elems);

/*
 * Point-wise channel mix (encoder / decoder), reference _mix_layer_forward
 * d/fno.py:286-289 -> einsum_channel_mix d/tensor.py:210-228, and the
 * activation d/fno.py:41-46.
 *   pre[b][o][p]  = sum_i f(src[b][i][p]) * w[i][o],  f = act if src_act else id
 *   post[b][o][p] = act(pre)          (post may be NULL)
 * npts = local points per channel (x_local*ny*nz*nt).
 */
int dfno_mix_fwd(const dfno_geom* g, int64_t npts, int cin, int cout,
                 const void* src, int src_act, const void* w,
                 void* pre, void* post, void* stream);

/*
 * Channel-mix backward, reference fno_backward d/fno.py:484-486 / :497-499
 * with _mix_weight_grad d/fno.py:405-406 and _mix_input_grad d/fno.py:409-412.
 *   gp = gout * act'(pre)
 *   gin[b][i][p] = sum_o gp[b][o][p] * w[i][o]            (gin may be NULL)
 *   partials[k][i][o] = CTA k's share of sum_{b,p} f(src[b][i][p]) gp[b][o][p]
 * src_act: 0 f = id, 1 f = act, 2 f = act and gin is returned multiplied by
 * act'(src) -- the gradient w.r.t. src itself, i.e. the decoder backward
 * fused with the last block's activation derivative (fp32 tcgen05 path only;
 * DFNO_ERR_UNSUPPORTED elsewhere, and the caller then uses 1).
 * dfno_mix_bwd_partials() gives the partial-buffer element count;
 * dfno_reduce_partials() then sums the partials in a fixed order
 * (deterministic, bit-identical replicas: d/training.py:77-82).
 */
int dfno_mix_bwd_partials(const dfno_geom* g, int64_t npts, int cin, int cout,
                          int64_t* partial_elems, int* num_partials);
int dfno_mix_bwd(const dfno_geom* g, int64_t npts, int cin, int cout,
                 const void* gout, const void* pre, const void* src, int src_act,
                 const void* w, void* gin, void* partials, void* stream);
int dfno_reduce_partials(const dfno_geom* g, int num_partials, int64_t n,
                         const void* partials, void* out, void* stream);

/*
 * Truncated forward DFT over (y, z, t) of this rank's x-slab, written
 * peer-major (XK layout) for the x->ky repartition.  Replaces
 *   fft_dims(a, (y,z,t)) + truncate_modes   d/fno.py:328-329 (forward)
 *   fft_dims(d, (y,z,t)) / N_yzt + truncate  d/fno.py:446-448 (backward)
 * src_mode: DFNO_SRC_ACT (input = act(src)), DFNO_SRC_GRAD
 * (input = src * act'(pre)), DFNO_SRC_RAW.  out = scale * sum(...).
 */
int dfno_dft_yzt_fwd(const dfno_geom* g, const void* src, const void* pre,
                     int src_mode, double scale, void* xk_out, void* stream);

/*
 * Inverse truncated DFT over (ky, kz, kt) -> real (y, z, t) slab from the
 * XK-layout buffer received in the ky->x repartition.  Replaces
 *   pad_modes + ifft_dims(yzt) + .real       d/fno.py:338-343 (scale 1/N_yzt)
 *   pad + ifft_dims(yzt) * N_yzt + .real      d/fno.py:459-464 (scale 1)
 * out[b][c][x][y][z][t] = scale * Re(sum_k V[k] e^{+2 pi i k.n / N}).
 */
int dfno_dft_yzt_inv(const dfno_geom* g, const void* xk_in, double scale,
                     void* out, void* stream);

/*
 * x-spectral stage on this rank's ky pencil, forward.  Replaces
 *   fft_dims(x) + truncate kx + einsum_spectral + pad kx + ifft_dims(kx)
 *   d/fno.py:331-336, d/tensor.py:231-255.
 * kx_in : KX layout received from the x->ky repartition
 * w     : spectral weight shard (c, c, rx, ky_local, rz, rt) complex
 * spec  : cache of the multiply input (b, c, rx, ky_local, rz, rt), may be NULL
 * kx_out: KX layout to send back in the ky->x repartition
 */
int dfno_xspec_fwd(const dfno_geom* g, const void* kx_in, const void* w,
                   void* spec, void* kx_out, void* stream);

/*
 * x-spectral stage, backward (adjoint chain d/fno.py:450-457 with
 * _spectral_weight_grad / _spectral_input_grad d/fno.py:415-423):
 *   D = fft_x(kx_in)/Nx truncated;  gw = sum_b conj(spec) D;
 *   kx_out = ifft_x(pad(sum_o D conj(w))) * Nx
 */
int dfno_xspec_bwd(const dfno_geom* g, const void* kx_in, const void* spec,
                   const void* w, void* gw, void* kx_out, void* stream);

/*
 * Workspace variants of the x-spectral stage: the DFT along x, the per-mode
 * channel contraction and the inverse DFT run as three bandwidth-shaped
 * kernels with the truncated spectra staged in `work` (caller-owned device
 * memory of dfno_xspec_workspace() bytes).  Same results and reference lines
 * as dfno_xspec_fwd / dfno_xspec_bwd; fp32 with batch <= 4 (other cases fall
 * back to the fused kernel, `work` unused).
 */
int dfno_xspec_workspace(const dfno_geom* g, int64_t* bytes);
int dfno_xspec_fwd_ws(const dfno_geom* g, const void* kx_in, const void* w,
                      void* spec, void* kx_out, void* work, void* stream);
int dfno_xspec_bwd_ws(const dfno_geom* g, const void* kx_in, const void* spec,
                      const void* w, void* gw, void* kx_out, void* work,
                      void* stream);

/*
 * The x-spectral stage by parts, fp32 (DFNO_ERR_UNSUPPORTED otherwise), so a
 * caller can pipeline channel groups against the repartition exchanges: the
 * x-DFTs of a group of channels run on a geometry whose c is the group size
 * with X / Y offset to the group's first channel (b = 1), the contraction on
 * the full geometry.  Same reference lines as dfno_xspec_fwd / _bwd.
 *   dfno_xdft     X  = scale * fft_x(kx_in) truncated   (d/fno.py:331-332, :450-452)
 *   dfno_xmix_fwd Y  = einsum_spectral(X, w)             (d/tensor.py:231-255)
 *   dfno_xmix_bwd gw = sum_b conj(spec) D ; dX = sum_o D conj(w)  (d/fno.py:415-423)
 *   dfno_xidft    kx_out = scale * sum_kx Y e^{+i}       (d/fno.py:335-336, :455-457)
 */
int dfno_xdft(const dfno_geom* g, const void* kx_in, double scale, void* X, void* stream);
int dfno_xmix_fwd(const dfno_geom* g, const void* X, const void* w, void* Y, void* stream);
int dfno_xmix_bwd(const dfno_geom* g, const void* spec, const void* D, const void* w, void* gw, void* dX,
                  void* stream);
int dfno_xidft(const dfno_geom* g, const void* Y, double scale, void* kx_out, void* stream);

/*
 * Training step (reference train_step d/training.py:96-133): fused residual /
 * loss / output gradient, and Adam on the real view of a parameter.
 *   resid = pred - target; grad_out = grad_scale * resid (grad_out may be
 *   NULL); sse_out[0] (double) = sum resid^2, reduced in a fixed order over
 *   dfno_mse_partials() double partials (deterministic).
 *   Adam (d/training.py:52-74): n real elements, step >= 1, every operation
 *   rounded to the parameter dtype in the reference's order.
 */
int dfno_mse_partials(int64_t n, int* num_partials);
int dfno_mse_grad(const dfno_geom* g, int64_t n, const void* pred, const void* target,
                  double grad_scale, void* grad_out, void* partials, void* sse_out,
                  void* stream);
int dfno_adam(const dfno_geom* g, int64_t n, void* param, const void* grad, void* m,
              void* v, double lr, double beta1, double beta2, double eps, int step,
              void* stream);
/* Same update written to param_out (param untouched; the reference returns
 * new parameter arrays, d/training.py:52-74, so no copy pass is needed). */
int dfno_adam_out(const dfno_geom* g, int64_t n, const void* param, void* param_out,
                  const void* grad, void* m, void* v, double lr, double beta1, double beta2,
                  double eps, int step, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DFNO_H */
