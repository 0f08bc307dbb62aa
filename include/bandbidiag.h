/*
 * bandbidiag.h -- C ABI of the B200 (sm_100a) band -> bidiagonal reduction.
 *
 * Operation (arXiv 2510.12705, "A GPU-resident Memory-Aware Algorithm for
 * Accelerating Bidiagonalization of Banded Matrices"; P:n = PAPER.md line n):
 * reduce an n x n UPPER-banded matrix A with b superdiagonals
 * (A[i][j] != 0 only for 0 <= j - i <= b) to UPPER bidiagonal form
 * B = U^T A V (U, V orthogonal, never formed) by Householder bulge chasing
 * (SVD stage 2).  The bandwidth is removed in passes of one inner
 * tilewidth (Alg. 1 line 1: b -> b - tw -> ... -> 1); each pass runs
 * one sweep per row (Alg. 1 line 3), each sweep a chain of row-bulge
 * steps (Alg. 2): a row reflector annihilating tw entries of the
 * anchor row, applied from the right, then a column reflector annihilating
 * the left-most column of the generated bulge, applied from the left.
 * Sweeps run as a device-side wavefront behind a dependency distance
 * ("three-cycle separation").  Only the singular values'
 * carrier (d, e) is returned; no singular vectors.
 *
 * Conventions shared by every entry point:
 *
 *  - Element types: BB_F16 = IEEE binary16 (__half; stored in fp16, computed
 *    in fp32, rounded to nearest-even on every store), BB_F32 = float,
 *    BB_F64 = double.
 *  - INPUT LAYOUT `band`: LAPACK upper-band storage, identical to xGBBRD
 *    with KL = 0, KU = b (and xSBTRD UPLO='U'): column-major with leading
 *    dimension `ldband` >= b + 1,
 *        A(i, j) = band[(b + i - j) + j * ldband],  max(0, j - b) <= i <= j.
 *    Slots outside that range are ignored.  In torch terms: a contiguous
 *    tensor of shape (n, ldband) with t[j, b + i - j] = A[i, j].
 *  - OUTPUT: d_out[0..n-1] = diagonal, e_out[0..n-2] = superdiagonal, in the
 *    input dtype.  Their signs are whatever the reflectors produce (LAPACK
 *    dlarfg convention, beta = -sign(alpha)||x||) unless
 *    BB_FLAG_NONNEG_OUTPUT is set, which returns |d|, |e| (an exact
 *    orthogonal equivalence by diagonal +-1 scalings).  |d|, |e| and the
 *    singular values are unique; the signs are not.
 *  - Batched strides are in ELEMENTS.  Matrix k of a batch reads
 *    band + k*stride_band and writes d_out + k*stride_d, e_out + k*stride_e.
 *  - Pointers: DEVICE pointers unless the function name ends in `_host`.
 *    `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  All device work is enqueued on `stream`; the call returns
 *    without host synchronisation; results are valid once the stream
 *    reaches that point.
 *  - Ownership: the caller owns every buffer.  `band` is read-only (it is
 *    copied into the working band).  The non-_ex forms allocate their
 *    workspace stream-ordered (cudaMallocAsync/cudaFreeAsync on `stream`);
 *    the _ex forms use a caller workspace of at least bb_workspace_size()
 *    bytes, 256-byte aligned, which must not be shared by concurrent calls.
 *  - Errors: no exceptions cross the ABI.  Argument errors are detected
 *    synchronously before any device work: BB_ERR_INVALID_VALUE for n < 0,
 *    b < 0, batch < 0, ldband < b + 1, a null pointer with n > 0 and
 *    batch > 0, overlapping batch strides (stride_band < n*ldband,
 *    stride_d < n, stride_e < n - 1), cfg->tw < 0 or workspace too small;
 *    BB_ERR_NOT_SUPPORTED for an unknown dtype or a step window that does
 *    not fit in one SM's shared memory (reduce tw); BB_ERR_OUT_OF_MEMORY
 *    when stream-ordered allocation fails; BB_ERR_CUDA for a launch / CUDA
 *    runtime failure (cudaGetLastError) or no usable device.
 *  - Edge cases: n == 0 or batch == 0: no-op, BB_SUCCESS.  n == 1: d = a00,
 *    e empty.  b >= n: clamped to n - 1.  b <= 1: already bidiagonal,
 *    copied through bit-exactly.
 */
#ifndef BANDBIDIAG_H
#define BANDBIDIAG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BB_VERSION 300 /* 0.3.0: unit (v5) and segment-ring (v6) pass kernels, stage-3 singular values */

/* Diagnostics read from the environment at call time (never needed for normal
 * use; results are bitwise independent of BB_V4_G):
 *   BB_V4_G=g          cap the sweeps per CTA of the multi-sweep kernel (0: use the
 *                      one-sweep register kernel instead)
 *   BB_TRACE_FILE=f, BB_TRACE_PASS=p
 *                      dump per-step device timestamps of pass p (tools/trace4.py);
 *                      synchronises the stream
 *   BB_DEBUG_SYNC=1    synchronise after every pass and report the failing pass
 *   BB_DEBUG_PASSES=k  run only the first k passes (the result is then not bidiagonal)
 *   BB_DEBUG_MAX_CYCLES=k  (cycle schedule only) run only k cycles of each pass */

typedef enum { BB_F16 = 0, BB_F32 = 1, BB_F64 = 2 } bb_dtype;

typedef enum {
    BB_SUCCESS = 0,
    BB_ERR_INVALID_VALUE = 1,
    BB_ERR_NOT_SUPPORTED = 2,
    BB_ERR_OUT_OF_MEMORY = 3,
    BB_ERR_CUDA = 4,
    BB_ERR_INTERNAL = 5
} bb_status;

/* Scheduling of the sweeps inside one pass (bb_config.schedule). */
#define BB_SCHED_AUTO 0  /* = BB_SCHED_FLAGS                                        */
#define BB_SCHED_FLAGS 1 /* one persistent kernel per pass; CTAs claim sweeps in     */
                         /* order and wait on per-sweep progress flags              */
                         /* (acquire/release): step (r, j) starts once sweep r-1    */
                         /* finished step min(j + s - 1, J_{r-1} - 1)       */
#define BB_SCHED_CYCLE 2 /* the paper's form: one kernel launch per global   */
                         /* cycle T, running every step (r, j) with s*r + j == T.   */
                         /* Slow (about s*n launches per pass); reference/debug.    */

/* bb_config.flags */
#define BB_FLAG_NONNEG_OUTPUT 0x1u /* return |d|, |e|                                    */
#define BB_FLAG_GENERIC_KERNEL 0x2u /* force the generic shared-memory step kernel (the   */
                                   /* register kernel serves tw <= 32); results are      */
                                   /* bitwise identical, for testing                     */
#define BB_FLAG_NO_UNIT_KERNEL 0x4u /* never use the unit kernel (G sweeps advanced one step */
                                    /* at a time, bb_pass_v5.cuh); testing / comparison    */
#define BB_FLAG_NO_SEGMENT_KERNEL 0x8u /* never use the segment-ring kernel of the target-   */
                                       /* bandwidth-1 pass (bb_pass_v6.cuh); results are     */
                                       /* bitwise identical, for testing / comparison        */
#define BB_FLAG_CHECK_ZEROS 0x10u /* debug: after the reduction, verify that every cell of the */
                                  /* working band outside the diagonal and superdiagonal is   */
                                  /* exactly zero (the structural zeros); SYNCHRONISES */
                                  /* `stream`; BB_ERR_INTERNAL if any is not (d, e are still  */
                                  /* written)                                                  */

/* Tuning knobs, the paper's hyperparameter triple.
 * Zero-initialise for defaults. */
typedef struct {
    int32_t tw;                /* inner tilewidth TW; 0 = default (32, measured) */
    int32_t threads_per_block; /* "Threads per block" of the GENERIC step kernel */
                               /* (BB_FLAG_GENERIC_KERNEL); 0 = auto.  The default      */
                               /* kernels size their CTAs from (c, t, G) themselves     */
    int32_t max_blocks_per_sm; /* "Max blocks": resident CTAs per SM; 0 = auto  */
    int32_t dep_distance;      /* s; 0 = auto (2, or 3 when the pass target is 1);      */
                               /* values below auto are raised to auto                  */
    int32_t schedule;          /* BB_SCHED_*                                            */
    uint32_t flags;            /* BB_FLAG_*                                             */
    /* Optional timing hooks (NULL/0 = off): an array of cudaEvent_t (as void*),
     * at least passes + 3 long, recorded on `stream`: [0] before the pack
     * kernel, [1] after it, [1 + p] after pass p (p = 1..passes), [passes + 2]
     * after the extract kernel.  Used by bench.py to time the pass kernels
     * with CUDA events on the launching stream.  Too short an array is
     * BB_ERR_INVALID_VALUE. */
    void **timing_events;
    int32_t num_timing_events;
} bb_config;

/* Plan of one call (host-only arithmetic, no device work). */
typedef struct {
    int64_t passes;          /* bandwidth passes (Alg. 1 line 1)                         */
    int64_t steps;           /* row-bulge steps per matrix                               */
    int64_t critical_cycles; /* per matrix: sum over passes of max_r (s*r + J_r)         */
    double alg_elements;     /* per matrix: sum over steps of the two-sided window size  */
                             /* m*((hi-q+1) + (ce-p+1) - m)                              */
    double alg_bytes;        /* per matrix: 2 * elem_size * alg_elements (read + write)  */
    double alg_flops;        /* per matrix: sum 4m(hi-q) + 4m(ce-p) + 6m                 */
    int32_t tw;              /* resolved tilewidth                                       */
    int32_t threads_per_block; /* threads per CTA the first pass's kernel launches          */
    int64_t ldw;             /* leading dimension of the working band (elements),        */
                             /* >= b_eff + 2 tw + 1, padded so ldw * elem is a multiple  */
                             /* of 16 bytes (TMA column boxes); mat_stride = n * ldw     */
    int64_t ku;              /* storage row of the diagonal in the working band          */
    int64_t mat_stride;      /* elements between consecutive matrices' working bands    */
    size_t workspace_bytes;  /* bytes bb_workspace_size() would return                   */
} bb_plan_stats;

/* Single matrix.  band: n x ldband (see layout above); d_out: n; e_out: n-1. */
bb_status bb_band_to_bidiag(int64_t n, int64_t b, bb_dtype dtype, const void *band, int64_t ldband,
                            void *d_out, void *e_out, void *stream);

/* `batch` independent matrices of equal (n, b), reduced concurrently: their
 * sweeps are interleaved in one persistent launch per pass. */
bb_status bb_band_to_bidiag_batched(int64_t n, int64_t b, bb_dtype dtype, int64_t batch,
                                    const void *band, int64_t ldband, int64_t stride_band,
                                    void *d_out, int64_t stride_d, void *e_out, int64_t stride_e,
                                    void *stream);

/* As above with a config (NULL = defaults) and a caller workspace.
 * Workspace layout (documented so tests can inspect the reduced band): it
 * begins with the working band, batch x n columns of ldw elements of the
 * input dtype; matrix k's A(i, j) lives at element
 *     k*mat_stride + (ku + i - j) + j*ldw,   -tw <= j - i <= b_eff + tw
 * (LAPACK general-band storage with KL = tw, KU = b_eff + tw: the band plus
 * twice the tilewidth of bulge headroom).  ldw, ku and mat_stride come
 * from bb_plan(). */
bb_status bb_band_to_bidiag_ex(int64_t n, int64_t b, bb_dtype dtype, const void *band, int64_t ldband,
                               void *d_out, void *e_out, const bb_config *cfg, void *workspace,
                               size_t workspace_bytes, void *stream);

bb_status bb_band_to_bidiag_batched_ex(int64_t n, int64_t b, bb_dtype dtype, int64_t batch,
                                       const void *band, int64_t ldband, int64_t stride_band,
                                       void *d_out, int64_t stride_d, void *e_out, int64_t stride_e,
                                       const bb_config *cfg, void *workspace, size_t workspace_bytes,
                                       void *stream);

/* End-to-end form with HOST buffers (pageable or pinned): copies the bands
 * host->device, reduces, copies d, e device->host, all on `stream`, and
 * BLOCKS until d_out/e_out are valid on the host.  Device memory: one
 * staging buffer per device (band copy, d, e, workspace), allocated on first
 * use, grown when a larger call needs it, kept until process exit; host
 * calls serialise on it (a mutex), so concurrent calls are safe but not
 * concurrent. */
bb_status bb_band_to_bidiag_host(int64_t n, int64_t b, bb_dtype dtype, int64_t batch,
                                 const void *band_host, int64_t ldband, int64_t stride_band,
                                 void *d_host, int64_t stride_d, void *e_host, int64_t stride_e,
                                 const bb_config *cfg, void *stream);

/* Workspace bytes for an _ex call with these arguments (host-only). */
bb_status bb_workspace_size(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const bb_config *cfg,
                            size_t *bytes);

/* Resolve the config and count the algorithmic work (host-only). */
bb_status bb_plan(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const bb_config *cfg,
                  bb_plan_stats *out);

/* Number of kernel launches one call enqueues (host-only); for the bench's
 * gpu_launches count. */
bb_status bb_launch_count(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const bb_config *cfg,
                          int64_t *launches);

/* ---- SVD stage 3 on the device ----------------------
 * Singular values of the upper bidiagonal B = bidiag(d, e) that stage 2
 * returns (the paper hands (d, e) to LAPACK BDSDC): bisection
 * on the Golub-Kahan tridiagonal (zero diagonal, off-diagonal d_0, e_0, d_1,
 * ..., d_{n-1}, eigenvalues +-sigma_i) with Sturm counts, one thread per
 * singular value, fp64 arithmetic for every dtype; each sigma_i to within
 * ~2 ulp of itself or eps * ||T||_Gershgorin (the normwise bound).
 *   d: n elements, e: n-1 elements (DEVICE, dtype), sigma: n fp64 (DEVICE),
 *   written in DESCENDING order.  Batched: matrix k at d + k*stride_d,
 *   e + k*stride_e, sigma + k*stride_sigma (elements).
 *   workspace: DEVICE, >= bb_bidiag_svals_workspace_size() bytes, caller-owned.
 * Errors: BB_ERR_INVALID_VALUE (negative sizes, NULL pointers with n > 0,
 * short workspace, overlapping batch strides), BB_ERR_NOT_SUPPORTED (dtype,
 * n > 2^28, batch > 65535), BB_ERR_CUDA (launch failure).  Enqueued on
 * `stream`, no host synchronisation. */
bb_status bb_bidiag_svals_workspace_size(int64_t n, int64_t batch, size_t *bytes);
bb_status bb_bidiag_svals(int64_t n, bb_dtype dtype, const void *d, const void *e, double *sigma, void *workspace,
                          size_t workspace_bytes, void *stream);
bb_status bb_bidiag_svals_batched(int64_t n, bb_dtype dtype, int64_t batch, const void *d, int64_t stride_d,
                                  const void *e, int64_t stride_e, double *sigma, int64_t stride_sigma,
                                  void *workspace, size_t workspace_bytes, void *stream);

/* ---- SVD stage 1 on the device ------------------------
 * Dense n x n A (DEVICE, column-major, lda >= n, fp32 or fp64) -> upper band
 * with b superdiagonals, U^T A V = band (U, V orthogonal, not formed), by
 * block Householder reflections: per block column a QR of the column panel
 * and an LQ of the row panel (one-CTA panel kernels, LAPACK dlarfg / dlarft
 * conventions), trailing updates as GEMMs (cuBLAS).  The "classical block
 * Householder" first stage the paper pairs with its bulge chasing (P:42,
 * P:308).  A is OVERWRITTEN (it holds the banded matrix on exit); `band`
 * (DEVICE, LAPACK upper band of the stage-2 input layout, ldband >= b + 1)
 * receives the band.  workspace: DEVICE, >= bb_dense_to_band_workspace_size()
 * bytes.  Errors: BB_ERR_INVALID_VALUE (sizes, NULL pointers, workspace),
 * BB_ERR_NOT_SUPPORTED (fp16), BB_ERR_CUDA.  Enqueued on `stream`; calls on
 * one device serialise on an internal cuBLAS handle. */
bb_status bb_dense_to_band_workspace_size(int64_t n, int64_t b, bb_dtype dtype, size_t *bytes);
bb_status bb_dense_to_band(int64_t n, int64_t b, bb_dtype dtype, void *A, int64_t lda, void *band, int64_t ldband,
                           void *workspace, size_t workspace_bytes, void *stream);

const char *bb_status_string(bb_status s);
int32_t bb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BANDBIDIAG_H */
