/*
 * hdconv.h -- C ABI of libhdconv.so: hybrid-dealiased linear convolution
 * (R. J. George, "Hybrid Dealiased Convolutions", arXiv 2306.10016) on NVIDIA
 * B200 (sm_100a).
 *
 * The operation (Eq. 4, per axis per PAPER.md:716):
 *     h = f * g,   h[o] = sum_a f[a] g[o - a],   extent L_f,i + L_g,i - 1,
 * computed without materialised zero padding: each input of length L on an
 * axis is explicitly padded to p*m (p = ceil(L/m)) and implicitly to
 * M1 = q*m >= M >= L_f + L_g - 1 (q = ceil(M/m)) (hybrid padding,
 * PAPER.md:641; parameters PAPER.md:564-567).  Per residue r < q the input is
 * folded and pre-twiddled, w_s = zeta_{qm}^{rs} sum_t zeta_q^{rt} x_{tm+s}
 * (Forward Eq. PAPER.md:528; Alg. "Forward Routine for 1D" PAPER.md:79-114),
 * transformed by a size-m FFT, multiplied pointwise (and summed over pairs for
 * multi-convolution), inverse transformed, untwiddled and accumulated into the
 * outputs (Backward Eq. PAPER.md:531; Alg. "Backward Routine for 1D"
 * PAPER.md:116-134; Alg. "Main Convolution for 1D" PAPER.md:136-204).
 * N-D problems are separable passes along each axis.
 *
 * Conventions (all entry points):
 *  - Complex data is interleaved (re, im): hd_dtype_t HD_C128 = 2 x double,
 *    HD_C64 = 2 x float.  Arrays are row-major, last axis contiguous, batch
 *    index outermost.  C128 buffers must be 16-byte aligned, C64 8-byte.
 *  - Device entry points take caller-owned DEVICE pointers.  The library never
 *    frees them; inputs are read-only; h must not alias f or g (out-of-place
 *    only, the paper's I parameter is unsupported).
 *  - Calls are asynchronous and ordered on `stream` (a cudaStream_t, NULL =
 *    legacy default stream).  Kernel faults surface at the next sync.
 *  - Status codes only; nothing is thrown across the ABI.  On any validation
 *    failure h is left untouched and hd_last_error() describes the problem.
 *  - Either input may be the longer one on any axis (convolution commutes,
 *    PAPER.md:680 "we can always call the larger array g").
 *  - M[i] = 0 selects the minimal padding M = L_f + L_g - 1 on axis i; a
 *    non-zero M[i] must satisfy M[i] >= L_f,i + L_g,i - 1 (aliases are removed
 *    only then) unless HD_FLAG_ALLOW_ALIAS is set.
 *  - plan = NULL uses the tuned plan cached for this problem, else a default
 *    plan; an explicit plan is honoured exactly (fields p_f, p_g, q, M1 are
 *    recomputed and returned by hd_plan_complete).
 *  - ws = NULL lets the context allocate (and cache) the workspace; otherwise
 *    ws_bytes must be >= hd_workspace_bytes() for the same arguments.  The
 *    context's scratch (workspace, real-path and host-I/O buffers) is shared
 *    by every call that passes no workspace, on whatever stream: each such
 *    call is ordered after the previous one's last use of it (an event wait
 *    on the caller's stream), so calls on different streams serialise on the
 *    device; pass a caller-owned ws per stream for concurrency.  A context may
 *    be used from several host threads (calls hold a per-context lock while
 *    they enqueue).
 *  - No CPU fallback exists: without a CUDA device every compute call returns
 *    HD_ERR_CUDA.
 */
#ifndef HDCONV_H
#define HDCONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HD_ABI_VERSION 1
#define HD_MAX_DIM 3
#define HD_MAX_PAIRS 16

typedef enum { HD_C64 = 1, HD_C128 = 2 } hd_dtype_t;

typedef enum {
  HD_OK = 0,
  HD_ERR_INVALID = 1,      /* bad sizes, pointers, plan */
  HD_ERR_UNSUPPORTED = 2,  /* valid request this build does not implement */
  HD_ERR_CUDA = 3,         /* CUDA runtime error (or no device) */
  HD_ERR_NCCL = 4,         /* NCCL missing or failed (distributed entry points) */
  HD_ERR_WORKSPACE = 5     /* caller workspace too small */
} hd_status_t;

/* Plan flags */
#define HD_FLAG_ALLOW_ALIAS 0x1u   /* test-only: accept M1 < L_out (aliased output, extent min(M1, L_out)) */
#define HD_FLAG_SHARED_G    0x2u   /* batch > 1: one g shared by every batch entry */
#define HD_FLAG_GENERIC_FFT 0x4u   /* force the generic radix-8 shared-memory FFT engine
                                      (default: the warp-level engine where it applies) */
#define HD_FLAG_GRAPH       0x8u   /* hd_conv1d/2d/3d, hd_multiconv, hd_conv_window: the first
                                      call also captures its kernel launches into a CUDA graph;
                                      later calls with identical arguments (pointers, extents,
                                      plan, window, stream) replay it with one graph launch.
                                      Dropped when the context reallocates its workspace or is
                                      destroyed; at most 64 are kept (the cache then starts
                                      over).  Not with profiling enabled. */
#define HD_FLAG_EXPLICIT_PLAN 0x20u /* hd_conv_explicit only: the plan is the PADDED problem's own
                                      (m <= M_exp, C, S, D), e.g. from hd_tune_explicit, rather
                                      than a hybrid plan to derive one from */
#define HD_FLAG_STAGED_ORDER 0x10u /* hd_pass only: the forward / inverse passes may run on the
                                      staged engines (m = 512 complex double with C = 1, D = q,
                                      p <= 8; m = 128 complex float with C = 4), whose spectral
                                      order differs from hd_spectral_permutation: a FWD output
                                      is then valid only as the input of an INV (or CONV) pass
                                      of the same axis, plan and flag.  HD_ERR_UNSUPPORTED when
                                      the staged engine does not apply to the pass. */

/* Per-axis parameters (L, M, C, m, D per dimension).
 *  m  : FFT size, a power of two in [2, 4096]
 *  p_f, p_g : ceil(L_f/m), ceil(L_g/m) (derived, PAPER.md:684-685 with Lambda = 1)
 *  q  : ceil(M/m) residues (derived from M and m)
 *  C  : lines (copies of the FFT computed simultaneously) per CTA in
 *       the passes along this axis: 1, 2, 4, 8 or 16
 *  S  : tile width of the transposed intermediate read by the passes along this
 *       axis (adjacent lines staged together; 1, 2, 4, 8 or 16; unused in 1D)
 *  D  : residues per group, 1 <= D <= q (0 = q)
 *  threads : CTA size of the generic engine (multiple of 32, 0 = automatic)
 *  M1 : q*m (derived) */
typedef struct {
  int32_t m, p_f, p_g, q, C, S, D, threads;
  int64_t M1;
} hd_axis_plan_t;

typedef struct {
  int32_t ndim;
  uint32_t flags;
  hd_axis_plan_t axis[HD_MAX_DIM];
  double tuned_seconds;   /* median seconds of the plan when chosen by hd_tune, else 0 */
} hd_plan_t;

typedef struct hd_ctx* hd_ctx_t;  /* owns twiddle tables, plan cache, scratch; one device */

/* ---- context --------------------------------------------------------------- */
int         hd_abi_version(void);
/* Create a context bound to CUDA device `device`.  Returns HD_ERR_CUDA if the
 * device cannot be selected (e.g. no GPU).  *ctx is NULL on failure. */
hd_status_t hd_create(hd_ctx_t* ctx, int device);
hd_status_t hd_destroy(hd_ctx_t ctx);
/* Message for the last failure on this context (or of hd_create when ctx is NULL). */
const char* hd_last_error(hd_ctx_t ctx);

/* ---- plans (host only, no GPU needed) -------------------------------------- */
/* Default plan for a problem: per-axis m, C/S, D chosen by a static cost model.
 * Lf, Lg, M: ndim extents each (M may be NULL = minimal). */
hd_status_t hd_plan_default(hd_dtype_t dtype, int32_t ndim, int32_t npairs,
                            const int64_t* Lf, const int64_t* Lg, const int64_t* M,
                            hd_plan_t* out);
/* Validate a plan against a problem and fill its derived fields (p_f, p_g, q, M1,
 * D = 0 -> q).  Returns HD_ERR_INVALID with a message on inadmissible plans. */
hd_status_t hd_plan_complete(hd_dtype_t dtype, int32_t ndim, int32_t npairs,
                             const int64_t* Lf, const int64_t* Lg, const int64_t* M,
                             hd_plan_t* plan);
/* Internal spectral order: the forward transforms write residue r's size-m FFT
 * output in digit-reversed order.  perm[pos] = l means slot pos of a residue
 * block holds frequency q*l + r.  (perm has m entries.) */
hd_status_t hd_spectral_permutation(int32_t m, int32_t* perm);

/* Bytes of scratch the device entry points need for these arguments. */
size_t hd_workspace_bytes(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t npairs,
                          int64_t batch, const int64_t* Lf, const int64_t* Lg,
                          const int64_t* M, const hd_plan_t* plan);

/* ---- convolution (device pointers) ----------------------------------------- */
/* 1D: batch independent pairs; f is [batch][Lf], g is [batch][Lg] (or [Lg] with
 * HD_FLAG_SHARED_G), h is [batch][Lf+Lg-1]. */
hd_status_t hd_conv1d(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch,
                      const void* f, int64_t Lf, const void* g, int64_t Lg,
                      void* h, int64_t M, const hd_plan_t* plan,
                      void* ws, size_t ws_bytes, void* stream);
/* 2D: f [batch][Lf0][Lf1], g [batch][Lg0][Lg1], h [batch][Lf0+Lg0-1][Lf1+Lg1-1]. */
hd_status_t hd_conv2d(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch,
                      const void* f, const int64_t Lf[2], const void* g, const int64_t Lg[2],
                      void* h, const int64_t M[2], const hd_plan_t* plan,
                      void* ws, size_t ws_bytes, void* stream);
/* 3D: as 2D with three extents. */
hd_status_t hd_conv3d(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch,
                      const void* f, const int64_t Lf[3], const void* g, const int64_t Lg[3],
                      void* h, const int64_t M[3], const hd_plan_t* plan,
                      void* ws, size_t ws_bytes, void* stream);
/* Multi-convolution h = sum_{k<N} f[k] * g[k] (reading R9); every f[k]
 * has extents Lf, every g[k] extents Lg; ndim in {1,2,3}; 1 <= N <= HD_MAX_PAIRS.
 * f and g are host arrays of N device pointers. */
hd_status_t hd_multiconv(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                         const void* const* f, const int64_t* Lf,
                         const void* const* g, const int64_t* Lg,
                         void* h, const int64_t* M, const hd_plan_t* plan,
                         void* ws, size_t ws_bytes, void* stream);
/* Explicit-dealiasing baseline: materialise zero padding to
 * M_exp,i = next power of two >= L_f,i + L_g,i - 1 and run the same kernels with
 * p = q (no pruned blocks); same output as hd_multiconv.  Measurement only. */
hd_status_t hd_conv_explicit(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                             const void* const* f, const int64_t* Lf,
                             const void* const* g, const int64_t* Lg,
                             void* h, const hd_plan_t* plan, void* stream);

/* Output window (PAPER.md:1482-1489 modes full / same_big / same_small / valid
 * are windows): h = (sum_k f[k] * g[k])[win_lo + w] for
 * 0 <= w_i < win_n[i], h an array of extents [batch] x win_n (device pointer).
 * Only the window is written; the last pass of every axis skips the rest.
 * Requires 0 <= win_lo[i] and win_lo[i] + win_n[i] <= L_f,i + L_g,i - 1.
 * Other arguments as hd_multiconv (N = 1 for a plain convolution) with batch. */
hd_status_t hd_conv_window(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                           int64_t batch, const void* const* f, const int64_t* Lf,
                           const void* const* g, const int64_t* Lg, void* h,
                           const int64_t* M, const int64_t* win_lo, const int64_t* win_n,
                           const hd_plan_t* plan, void* ws, size_t ws_bytes, void* stream);

/* Real inputs: f, g, h REAL arrays of the complex dtype's
 * component type (HD_C128: double, HD_C64: float), device pointers, batch pairs,
 * h = f * g (full, extent L_f + L_g - 1 per axis).  The two halves of f along
 * axis 0 (rows [0, A) and [A, L_f,0), A = ceil(L_f,0 / 2)) are packed as the real
 * and imaginary parts of one complex array z; because g is real, w = z * g (the
 * complex pipeline, hd_conv1d/2d/3d's kernels) holds both half convolutions, and
 * h[y] = Re w[y] + Im w[y - A] (overlap-add of the two halves).  About half the
 * transform work and half the input/output bytes of the complex path.  `plan`
 * is for the packed problem (extents A, L_f,1.. and L_g); NULL = cached/default.
 * 2-D HD_C128 with batch 1, even row lengths and the x axis on the staged q = 9
 * kernel: the pack and the unpack run inside the first and last passes (no z or
 * w array; a fix-up kernel adds the L_g,0 - 1 overlapping rows).  Results are the
 * same either way; the context's real-path buffers are reused across calls. */
hd_status_t hd_conv_real(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int64_t batch,
                         const void* f, const int64_t* Lf, const void* g, const int64_t* Lg,
                         void* h, const hd_plan_t* plan, void* stream);

/* ---- end-to-end with HOST buffers ------------------------------------------ */
/* Same as hd_multiconv with batch (N = 1 for plain conv) but f, g, h are HOST
 * pointers (pinned for best speed).  Copies in, convolves, copies out and
 * synchronises `stream` before returning.  Device buffers are context-owned. */
hd_status_t hd_conv_host(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                         int64_t batch, const void* const* f, const int64_t* Lf,
                         const void* const* g, const int64_t* Lg, void* h,
                         const int64_t* M, const hd_plan_t* plan, void* stream);

/* Asynchronous form of hd_conv_host: enqueues copy-in, convolution and copy-out
 * on one of three context-owned streams with their own device buffers, in turn per
 * call, and returns.  The copy-in of call k+2, the convolution of call k+1 and the
 * copy-out of call k can run at once (the convolutions themselves run one after
 * another: they share the context workspace).  f, g, h must stay valid (and h unread)
 * until hd_host_sync returns; pinned host memory is needed for the copies to overlap.
 * Errors in enqueueing are returned; kernel faults surface at hd_host_sync. */
hd_status_t hd_conv_host_async(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                               int64_t batch, const void* const* f, const int64_t* Lf,
                               const void* const* g, const int64_t* Lg, void* h,
                               const int64_t* M, const hd_plan_t* plan);
/* Wait for every hd_conv_host_async call of this context. */
hd_status_t hd_host_sync(hd_ctx_t ctx);

/* ---- the paper's residue routines, batched (device pointers) --------------- */
/* Forward: for each of nlines lines x[l][0..L) compute every residue block
 * X[l][r*m + pos] = F_{q*perm[pos] + r} of x zero-padded to q*m (
 * Alg. Forward PAPER.md:79-114 with lambda = 1). X is [nlines][q*m]. */
hd_status_t hd_forward_residues(hd_ctx_t ctx, hd_dtype_t dtype, int64_t nlines,
                                const void* x, int64_t L, int32_t m, int32_t q,
                                void* X, void* stream);
/* Backward: x[l][j] = sum over residues of the Backward Eq. without
 * the 1/(qm) factor, for j < Lout <= q*m (Alg. Backward).  Input
 * in the internal order hd_forward_residues writes. */
hd_status_t hd_backward_residues(hd_ctx_t ctx, hd_dtype_t dtype, int64_t nlines,
                                 const void* X, int32_t m, int32_t q, void* x,
                                 int64_t Lout, void* stream);

/* ---- one pass with explicit layouts (building block of the distributed paths) */
/* A pass runs along ONE axis over `nlines` lines (x `nbatch` batch entries) of
 * m-point residue transforms, exactly as one launch of the multi-pass pipeline:
 *   HD_PASS_FWD : fold + forward FFT of every line of in_f (array k = 0..npairs-1)
 *                 -> out (array k): q*m spectral values per line, internal order
 *   HD_PASS_INV : inverse FFT + unfold of every spectral line of in_f -> out
 *                 (out.L values per line; no 1/(qm) factor)
 *   HD_PASS_CONV: fold + FFT of in_f[k] and in_g[k], sum_k product x scale,
 *                 inverse FFT + unfold -> out (one array)
 * Addressing (elements, not bytes), for line l (0..nlines-1) and element j:
 *   ptr[k] + (b/nbi)*s_bo + (b%nbi)*s_b + line(l) + elem(j)
 *   line(l) = tl < 30 ? (l >> tl)*s_t + (l & (2^tl-1))*s_l : l*s_l
 *   elem(j) = jd > 0  ? (j / jd)*s_jt + (j % jd)*s_j       : j*s_j
 * Inputs are zero beyond L; outputs write elements j < L only.  The plan axis
 * gives m, C, D, threads; q = ceil(M/m) for the descriptor's M. */
#define HD_PASS_FWD  0
#define HD_PASS_INV  1
#define HD_PASS_CONV 2
typedef struct {
  void* ptr[HD_MAX_PAIRS];
  int64_t L;
  int64_t nbi, s_bo, s_b;     /* nbi = 0: one batch level (nbi = nbatch) */
  int32_t tl, pad_;
  int64_t s_t, s_l;
  int64_t jd, s_jt, s_j;
} hd_lines_t;
typedef struct {
  int32_t mode;               /* HD_PASS_* */
  int32_t npairs;             /* arrays (FWD/INV) or pairs (CONV), 1..16 */
  int64_t nlines, nbatch;
  int64_t M;                  /* padded length along this axis; q = ceil(M/m) */
  hd_axis_plan_t axis;        /* m, C, D (0 = q), threads (0 = automatic); a D whose group of
                                 C D m elements exceeds the generic engine's shared memory
                                 is lowered until it fits (same results: the groups are
                                 walked in turn) */
  hd_lines_t in_f, in_g, out;
  double scale;               /* CONV: product scale (1 / prod M1 over all axes) */
  int32_t batch_fastest;      /* 1: consecutive CTAs take consecutive batch entries */
  uint32_t flags;             /* HD_FLAG_GENERIC_FFT */
  int32_t r_begin, r_end;     /* CONV only: residues [r_begin, r_end) (0, 0 = all q); the
                                 output is then the partial sum over those residues of
                                 the backward transform -- residue
                                 sharding.  A partial range runs the generic engine. */
} hd_pass_desc_t;
/* Validate and launch one pass on `stream`.  Device pointers.  Returns
 * HD_ERR_INVALID on bad sizes/layouts, HD_ERR_UNSUPPORTED if no kernel exists. */
hd_status_t hd_pass(hd_ctx_t ctx, hd_dtype_t dtype, const hd_pass_desc_t* desc, void* stream);

/* Tune the explicit-padding baseline's own plan (hd_conv_explicit's padded problem,
 * M_exp = next power of two >= L_out per axis): per-axis search over m in {64, ...,
 * min(4096, M_exp)}, C in {1, 2, 4} (C > 1 only for m <= 256), S in {1, 2, 4, 8}
 * (ndim > 1), each timed as whole hd_conv_explicit calls (1 warm-up, median of reps,
 * 0 = 3) on zero operands.  The result (flags = HD_FLAG_EXPLICIT_PLAN) is cached: later
 * hd_conv_explicit calls with plan = NULL use it.  hd_tune_log lists the candidates. */
hd_status_t hd_tune_explicit(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N, const int64_t* Lf,
                             const int64_t* Lg, int32_t reps, void* stream, hd_plan_t* out);

/* ---- image filtering ------------------------
 * The paper's demo convolves every channel of an image with one of eight small named
 * kernels (Identity, Ridge_detection_1, Ridge_detection_2, Sharpen,
 * Box_blur, Gaussian_blur, Gaussian_blur_5, Unsharpen_masking -- ids 0..7 in that order)
 * and keeps the real part of each channel's result.
 * hd_filter_kernel (host only): kernel `id` -> its n x n weights (row-major, scale
 * applied; w may be NULL), n and its name.  hd_filter_image: img is a REAL H x W image
 * with C channels (double for HD_C128, float for HD_C64; channel_last = 1: [H][W][C] as
 * decoded images are, 0: [C][H][W]); every channel is convolved with the kernel through
 * the real-input path (hd_conv_real, the channels as one batch), and the window
 * [win_lo, win_lo + win_n) of the full (H + n - 1) x (W + n - 1) result (NULL = all) is
 * written to out in the same channel layout (real values; the listing's further crop
 * and uint8 cast belong to its PNG round trip, which is not built).  Device pointers;
 * scratch is stream-ordered (cudaMallocAsync).  Errors: hd_filter_last_error(). */
#define HD_FILTER_COUNT 8
hd_status_t hd_filter_kernel(int32_t id, double* w, int32_t* n, const char** name);
hd_status_t hd_filter_image(hd_ctx_t ctx, hd_dtype_t dtype, const void* img, int64_t H, int64_t W, int32_t C,
                            int32_t channel_last, int32_t id, const int64_t* win_lo, const int64_t* win_n,
                            void* out, void* stream);
const char* hd_filter_last_error(void);

/* ---- multi-GPU: one process per GPU, NCCL over NVLink --------
 * Bring-up: rank 0 calls hd_dist_unique_id and broadcasts the 128-byte id to the other
 * ranks (the harness's own channel, e.g. torch.distributed); every rank then calls
 * hd_dist_init on its context (device already selected).  nranks = 1 needs no id and
 * no NCCL (the exchanges become local).  NCCL is bound at run time (libnccl.so.2: the
 * copy already loaded in the process, else the system one); HD_ERR_NCCL if missing.
 * The communicator and a communication stream belong to the context (released by
 * hd_dist_init again or hd_destroy).  Errors of the calls below that are not a pass
 * launch's are described by hd_dist_last_error() (thread-local). */
hd_status_t hd_dist_unique_id(void* id /* 128 bytes out */);
hd_status_t hd_dist_init(hd_ctx_t ctx, const void* id, int32_t nranks, int32_t rank);
const char* hd_dist_last_error(void);
/* The library's contiguous partition of `extent` items: rank gets [lo, hi), blocks of
 * ceil(extent / nranks) (the last ones may be short or empty). */
hd_status_t hd_dist_partition(int64_t extent, int32_t nranks, int32_t rank, int64_t* lo, int64_t* hi);

/* 1-D: batch of independent pairs f[b] * g[b] (BASELINE config 2).
 *  HD_SHARD_BATCH   f, g, h hold ONLY this rank's batch slice [lo, hi) of
 *                   hd_dist_partition(batch): no collective.
 *  HD_SHARD_RESIDUE f, g hold the WHOLE batch on every rank; the q residues of every
 *                   line are split over the ranks (hd_dist_partition(q)) -- residues are
 *                   independent (Forward Eq. PAPER.md:528) -- each rank
 *                   computes its residues' backward contributions for all
 *                   lines and an NCCL reduce-scatter (sum) leaves h = the rank's batch
 *                   slice [lo, hi) of hd_dist_partition(batch), (hi - lo) x (Lf+Lg-1). */
#define HD_SHARD_BATCH   0u
#define HD_SHARD_RESIDUE 1u
hd_status_t hd_conv1d_dist(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, int64_t Lf,
                           const void* g, int64_t Lg, void* h, const hd_plan_t* plan, uint32_t shard,
                           void* stream);

/* 2-D / 3-D slab decomposition along axis 0 (separable passes).
 * hd_dist_slab_plan (host only) gives a rank's share and the exchange layout:
 *  in_lo/in_hi   rows (2-D) / planes (3-D) of f this rank holds (row-major, contiguous)
 *  out_lo/out_hi rows / planes of h it receives
 *  spec_lo/hi    spectral lines of axis 1 (2-D: kx columns; 3-D: ky rows) it convolves
 *  R, Ro, Ks     per-rank input, output and spectral extents (2-D: R padded to a
 *                multiple of nchunks, Ks to nchunks x a multiple of 16); chunk_rows =
 *                R / nchunks, chunk_cols = Ks / nchunks
 *                (3-D: chunk_cols = the kx tile of the exchange blocks)
 *  block1/2      elements of one (sender, receiver) block in the two all-to-alls
 *  bytes_sent    bytes leaving this rank per call (both exchanges, self excluded)
 *  scale         1 / prod M1 (the product's normalisation)
 *  plan          the completed plan of the global problem
 * 2-D overlap: pass A (forward along x) runs by row chunks and each chunk's all-to-all
 * starts on the communication stream as soon as its chunk is written; pass B
 * (convolution along y) runs by column chunks, each chunk's all-to-all likewise; pass C
 * (inverse along x) waits for the second exchange.  nchunks = 0: 2 (1 at nranks = 1). */
typedef struct {
  int32_t ndim, nranks, rank, nchunks;
  int64_t in_lo, in_hi, out_lo, out_hi, spec_lo, spec_hi;
  int64_t R, Ro, Ks, chunk_rows, chunk_cols;
  int64_t block1, block2, bytes_sent;
  double scale;
  hd_plan_t plan;
} hd_slab_plan_t;
hd_status_t hd_dist_slab_plan(hd_dtype_t dtype, int32_t ndim, int32_t nranks, int32_t rank, int32_t nchunks,
                              const int64_t* Lf, const int64_t* Lg, const hd_plan_t* plan, hd_slab_plan_t* out);
/* One rank's compute stages without the exchanges (the building blocks of
 * hd_conv2d_dist / hd_conv3d_dist; also lets a caller run its own exchange, e.g. to
 * check the layouts with emulated ranks).  Device buffers; `S` from hd_dist_slab_plan:
 *   stage 0: in = g (whole)               -> out = transformed g (hd_slab_g_bytes)
 *   stage 1: in = f slab                  -> out = send1 (nranks x block1 elements)
 *   stage 2: in = recv1, gt = stage 0 out -> out = send2 (nranks x block2 elements)
 *   stage 3: in = recv2                   -> out = h slab
 * 2-D exchanges, by pieces of P1 = Ks * chunk_rows (first) and P2 = Ro * chunk_cols
 * (second) elements: send is chunk-major (piece for rank d of chunk c at
 * (c * nranks + d) * P), recv source-major (piece from rank s of chunk c at
 * s * block + c * P); with one chunk this is the plain all-to-all.  3-D: both
 * exchanges are plain all-to-alls (block b of rank k's recv = block k of rank b's send).
 * 3-D stages 0, 1, 3 need `scratch` of hd_slab_scratch_bytes (2-D: unused). */
hd_status_t hd_slab_stage(hd_ctx_t ctx, hd_dtype_t dtype, const hd_slab_plan_t* S, const int64_t* Lf,
                          const int64_t* Lg, int32_t stage, const void* in, const void* gt, void* out,
                          void* scratch, void* stream);
size_t hd_slab_scratch_bytes(hd_dtype_t dtype, const hd_slab_plan_t* S, const int64_t* Lf, const int64_t* Lg);
size_t hd_slab_g_bytes(hd_dtype_t dtype, const hd_slab_plan_t* S, const int64_t* Lg);
/* f_rows: rows [in_lo, in_hi) of f ([rows][Lf[1]], device); g: the whole g on every
 * rank; h_rows: rows [out_lo, out_hi) of h ([rows][Lf[1]+Lg[1]-1]).  Lf, Lg: GLOBAL
 * extents.  Every rank must call with the same extents, plan and nchunks. */
hd_status_t hd_conv2d_dist(hd_ctx_t ctx, hd_dtype_t dtype, const void* f_rows, const int64_t Lf[2],
                           const void* g, const int64_t Lg[2], void* h_rows, const hd_plan_t* plan,
                           int32_t nchunks, void* stream);
/* The same with planes of 3-D arrays (f_planes [planes][Lf1][Lf2], h_planes likewise). */
hd_status_t hd_conv3d_dist(hd_ctx_t ctx, hd_dtype_t dtype, const void* f_planes, const int64_t Lf[3],
                           const void* g, const int64_t Lg[3], void* h_planes, const hd_plan_t* plan,
                           void* stream);

/* ---- tuning (the paper's "experience") -------------------- */
#define HD_TUNE_PER_AXIS   0x0u   /* search each axis independently */
#define HD_TUNE_EXHAUSTIVE 0x1u   /* full cross product (grid search A0) */
/* Time candidate plans on the device (CUDA events, 2 warm-ups, median of `reps`
 * >= 1 runs; 0 = 5) and return the fastest; ties break lexicographically on
 * (m, C, S, D).  Inputs are synthetic scratch of the problem's shape.  The
 * result is cached in the context for plan = NULL calls on the same problem.
 * Search space per axis i (hd_tune_space lists it):
 *   m a power of two in [16, 4096] with q = ceil(M_i / m) <= 1024;
 *   C in {1, 2, 4, 8};  D in {q, ceil(q/2), ceil(q/4), ..., 1};
 *   S in {1, 2, 4, 8, 16} (1 when ndim = 1);
 *   threads in {0 (automatic engine), d, 256} with d the sweep-matched default of
 *   (C, D, m), plus {768, 1024} when C*D*m/8 >= 512 and the pass uses more than half
 *   of the 227 KB of shared memory;
 *   excluding candidates whose generic pass exceeds 227 KB of shared memory:
 *   16 bytes (c128) / 8 (c64) x (r(q) + r(256) + nbuf r(C D m)), r(n) = n rounded up
 *   to a multiple of 64 (c128) / 128 (c64) slots, nbuf = 2 (3 with N > 1) on axis 0,
 *   else 1.
 * Pruning: a candidate whose first warm-up takes more than 3x the best median so far
 * is logged with that time and not repeated; in the per-axis search the candidates
 * come in groups of equal (m, C) (the order above), and when a group's first member
 * is more than 3x slower than the best so far the rest of the group is logged with
 * time +inf (not timed).  Every candidate of the space appears in hd_tune_log.  HD_TUNE_EXHAUSTIVE times the whole
 * cross product of the per-axis spaces and fails (HD_ERR_UNSUPPORTED) above 2^22
 * plans instead of truncating. */
/* Host only: the number of candidates of axis `axis` in the space above (-1 on bad
 * arguments); the first min(cap, count) are written to out (m, C, S, D, threads). */
int32_t hd_tune_space(hd_dtype_t dtype, int32_t ndim, int32_t N, const int64_t* Lf, const int64_t* Lg,
                      const int64_t* M, int32_t axis, hd_axis_plan_t* out, int32_t cap);
hd_status_t hd_tune(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                    int64_t batch, const int64_t* Lf, const int64_t* Lg, const int64_t* M,
                    uint32_t flags, int32_t reps, void* stream, hd_plan_t* out);
/* Extended tuning.  flags:
 *   HD_TUNE_PER_AXIS / HD_TUNE_EXHAUSTIVE as hd_tune;
 *   HD_TUNE_RANDOM: A1 random search: n1 plans sampled uniformly
 *     without replacement from the cross product (all of it when n1 >= its size),
 *     deterministic for a seed (splitmix64); argmin, lexicographic tie-break.
 * proxy_rows > 0 (per-axis search, ndim >= 2): the axes other than 0 are timed on
 *   the skinny proxy problem with min(L, proxy_rows) lines along axis 0 and the
 *   winners reused for the full problem (the L_y = 32 heuristic).
 * fake_cost (testing hook, no device work): 1 = the cost of a plan is a fixed hash
 *   of it (and of seed), 2 = every plan costs the same.
 * The result is cached like hd_tune's; hd_tune_log lists every evaluated plan. */
#define HD_TUNE_RANDOM 0x2u
typedef struct {
  uint32_t flags;
  int32_t reps;          /* timed runs per candidate (median); 0 = 5 */
  int32_t n1;            /* HD_TUNE_RANDOM: sample size (>= 1) */
  int32_t fake_cost;     /* 0: time on the device */
  uint64_t seed;
  int64_t proxy_rows;    /* 0: no proxy */
} hd_tune_opts_t;
hd_status_t hd_tune_ex(hd_ctx_t ctx, hd_dtype_t dtype, int32_t ndim, int32_t N,
                       int64_t batch, const int64_t* Lf, const int64_t* Lg, const int64_t* M,
                       const hd_tune_opts_t* opts, void* stream, hd_plan_t* out);
/* Number of candidates evaluated by the last hd_tune and their (plan, seconds). */
int32_t     hd_tune_log(hd_ctx_t ctx, int32_t max, hd_plan_t* plans, double* seconds);

/* ---- row f1: Lambda > 1 residue matching (1-D) ------------------------------- */
/* Linear convolution of a short input f (L_f) with a long input g (L_g >= L_f) by
 * the unequal-size construction of PAPER.md:680-702 ("Final Algorithm For One
 * Dimension"): p_f = ceil(L_f/m), p_g = ceil(L_g/(Lambda m)), q_g = ceil(M/(Lambda m)),
 * q_f = Lambda q_g.  f is transformed into q_f residues of FFT size
 * m, g into q_g residues of FFT size Lambda m; residue r_g of g meets residues
 * r_f = q_g lambda + r_g of f at l_f = floor(l_g / Lambda), lambda = l_g mod Lambda
 * (q_g l_g + r_g = q_f l_f + r_f); the matched product is inverted
 * with size Lambda m and accumulated over the q_g residues.
 *   f : [batch][L_f], g : [batch][L_g], h : [batch][L_f + L_g - 1], device pointers,
 *       contiguous rows, interleaved complex (HD_C64 / HD_C128), h not aliasing f, g;
 *   M : padded length (0: L_f + L_g - 1; M < L_f + L_g - 1 is rejected);
 *   m, Lambda : powers of two, Lambda m <= 4096 (Lambda = 1: the Lambda = 1 method).
 * Runs as four launches on `stream` (two forward residue passes, the matched product,
 * one backward pass) with a context-owned workspace of 2 batch q_g Lambda m elements.
 * Errors: HD_ERR_INVALID for L_f > L_g, bad m / Lambda, M too small, null pointers. */
hd_status_t hd_conv1d_lambda(hd_ctx_t ctx, hd_dtype_t dtype, int64_t batch, const void* f, int64_t Lf,
                             const void* g, int64_t Lg, void* h, int64_t M, int32_t m, int32_t Lambda,
                             void* stream);

/* ---- measurement hooks ------------------------------------------------------ */
/* When enabled, each kernel launch of the compute entry points is bracketed by
 * CUDA events on its stream; hd_profile_read returns (after a stream sync by the
 * caller) the accumulated per-pass milliseconds, launch counts and names. */
hd_status_t hd_profile_enable(hd_ctx_t ctx, int32_t enable);
int32_t     hd_profile_read(hd_ctx_t ctx, int32_t max, double* ms, int64_t* launches,
                            char* names /* max x 32 bytes */);
hd_status_t hd_profile_reset(hd_ctx_t ctx);
/* Total kernel launches issued by this context since creation. */
int64_t     hd_launch_count(hd_ctx_t ctx);
/* Pass launches issued by this context since creation on one engine (HD_ENGINE_*),
 * or -1 for a null context / unknown engine.  The engine of each pass is chosen
 * automatically per axis (plan threads = 0); this reports which ones ran. */
#define HD_ENGINE_GENERIC 0     /* shared-memory radix-8 engine, any m and dtype */
#define HD_ENGINE_S512 1        /* staged warp engine, m = 512 complex double (C = 1) */
#define HD_ENGINE_S512_MCONV 2  /* its multi-pair convolution pass */
#define HD_ENGINE_S128 3        /* staged engine, m = 128 complex float (C = 4) */
#define HD_ENGINE_S512C 4       /* 1-D pass of long lines on two-CTA clusters, complex double,
                                   m = 512 (12 <= q <= 22) */
#define HD_ENGINE_S2048R 5      /* 1-D pass of long lines, complex double, m = 2048, one CTA per
                                   line, residues in pairs (D = q <= 8, p <= 8) */
#define HD_ENGINE_S4096R 6      /* 1-D pass of long lines, complex double, m = 4096, one CTA per
                                   line, eight warps, one residue at a time (D = q <= 4, p <= 4) */
int64_t     hd_engine_launches(hd_ctx_t ctx, int32_t engine);
/* Calls served by replaying a captured CUDA graph (HD_FLAG_GRAPH) since creation;
 * -1 for a null context.  Replays do not add to hd_launch_count. */
int64_t     hd_graph_replays(hd_ctx_t ctx);

#ifdef __cplusplus
}
#endif
#endif /* HDCONV_H */
