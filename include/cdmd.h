/*
 * cdmd.h — C ABI of libcdmd, the B200 (sm_100a) hot path of compressed dynamic
 * mode decomposition (cDMD, Erichson, Brunton & Kutz, arXiv 1512.04205).
 *
 * Citations "P:n" are lines of the paper's LaTeX source; "Alg. 1" is
 * its Algorithm 1.  Readings of silent/garbled passages: DESIGN.md §4.
 *
 * Conventions shared by every entry point
 *  - Pointers are DEVICE pointers unless the argument says "host".
 *  - The CALLER owns every buffer (video, sketch, model, modes, mask, workspace);
 *    the library keeps only per-handle state (cuBLAS/cuSOLVER handles, the Gaussian
 *    table, a ring of 64 tile counters for the persistent kernels -- each launch of
 *    cdmd_modes / cdmd_foreground takes the next one, so up to 64 such launches of one
 *    handle may be in flight at once on any streams -- and the set of sparse sensing
 *    plans already checked) and never allocates on the hot path.
 *  - Calls are asynchronous on the given stream, except cdmd_fit (it reads the
 *    solver status and the model sizes back to the host once) and cdmd_create.
 *  - Validation happens on the host before any launch; an invalid call returns a
 *    status other than CDMD_OK and launches nothing.
 *  - One handle per device per host thread.  Entry points are reentrant.
 *
 * Data layouts
 *  - Video X (D of Alg. 1): uint8, FRAME-MAJOR, X[t*ld + j] is pixel
 *    (pix0 + j) of frame t+1 (a frame is the paper's column x_t).  A rank
 *    of a pixel-sharded run holds the slab of global pixels [pix0, pix0+n_local).
 *    X must be 16-byte aligned, ld >= n_local and ld % 16 == 0, pix0 % 128 == 0.
 *  - Sketch Y_full = C D: p x m, column-major, Y[r + t*ldy]; int32 for
 *    CDMD_SPIXEL / CDMD_SPARSE / CDMD_RADEMACHER (exact), float for CDMD_GAUSSIAN and
 *    CDMD_SRFT (rows 0 .. p/2-1 = Re, p/2 .. p-1 = Im of the complex measurements).
 *    Y = first m-1 columns, Y' = last m-1 columns (Eq. FullData, reading R2).
 *  - Modes Phi (Eq. cDMDModes): complex n x k with columns in conjugate
 *    pairs, stored FOLDED as k_eff real float columns, Phi[j + c*ldphi]:
 *    real eigenvalue  -> column c = phi_c;
 *    pair (c, c+1)    -> columns c, c+1 = Re phi_c, Im phi_c  (phi_{c+1} = conj phi_c).
 *  - Mask (Eq. thres): bit (j % 32) of uint32 word mask[t*ldw + j/32]
 *    is 1 iff |x_jt - L_jt| > tau.
 */
#ifndef CDMD_H
#define CDMD_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CDMD_API __attribute__((visibility("default")))
#else
#define CDMD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* cdmd_stream;       /* == cudaStream_t; NULL = legacy default stream */
typedef struct cdmd_handle_s* cdmd_handle;

typedef enum {
  CDMD_OK = 0,
  CDMD_ERR_ARG = 1,        /* null / misaligned pointer, bad layout or enum      */
  CDMD_ERR_RANGE = 2,      /* p, s, m, k, K, tau out of range                    */
  CDMD_ERR_NUMERIC = 3,    /* solver non-convergence, every sigma dropped, ...   */
  CDMD_ERR_CUDA = 4,       /* CUDA runtime / cuBLAS / cuSOLVER error             */
  CDMD_ERR_WORKSPACE = 5,  /* workspace or model buffer too small                */
  CDMD_ERR_UNSUPPORTED = 6 /* not built for this device (needs sm_100a)          */
} cdmd_status;

/* Measurement matrix C in R^{p x n} (Alg. 1 step 2, P:334 read as p x n). */
typedef enum {
  CDMD_SPIXEL = 0,     /* C = R, p rows of I_n without replacement            */
  CDMD_SPARSE = 1,     /* +-1 w.p. 1/(2s) each, 0 otherwise                    */
  CDMD_RADEMACHER = 2, /* +-1 (Bernoulli; the s = 1 case of P:386-393)              */
  CDMD_GAUSSIAN = 3,   /* N(0,1) rounded to bf16 (reading R7)                       */
  CDMD_SRFT = 4        /* subsampled random Fourier transform C = R F D, realified:
                          p (even) real rows = Re and Im of p/2 complex measurements; phases
                          quantised to 2^-16 turn, entries fp16 (reading R25)             */
} cdmd_measure;

typedef enum {
  CDMD_BG_STATIC = 0,  /* x_BG = Re(Phi beta), one value per pixel            */
  CDMD_BG_DYNAMIC = 1  /* L_jt = Re sum_{p in S} beta_p phi_jp lambda_p^{t-1} */
} cdmd_bg_mode;

typedef struct {
  const uint8_t* X;   /* device, frame-major, see "Data layouts"                  */
  int64_t n_total;    /* n: pixels per frame of the whole video            */
  int64_t pix0;       /* first global pixel of this slab (multiple of 128)        */
  int64_t n_local;    /* pixels in this slab                                      */
  int64_t m;          /* frames, m >= 2                                    */
  int64_t ld;         /* bytes between frames, >= n_local, multiple of 16         */
} cdmd_video;

typedef struct {
  int32_t kind;       /* cdmd_measure                                             */
  int64_t p;          /* measurements, 1 <= p <= n_total                  */
  double s;           /* sparse rate, > 1; <= 0 selects n_total / ln(n_total)     */
  uint64_t seed;      /* Philox4x32-10 key = (seed & 0xffffffff, seed >> 32)       */
} cdmd_sensing;

/* The fitted model (Alg. 1 outputs Phi, b, V of P:331 in factored form).
 * Bind it to ONE caller-allocated device buffer with cdmd_model_bind(); the
 * pointers below then point into that buffer.  Host fields are written by
 * cdmd_fit before it returns. */
typedef struct {
  /* capacities, set by cdmd_model_bind */
  int32_t k, K;        /* target rank and OMP sparsity             */
  int32_t limbs;       /* int8 limbs of the fixed-point M used by cdmd_modes       */
  int32_t kpad;        /* k rounded up to the MMA column block                     */
  int64_t m, mpad;     /* frames; m - 1 rounded up to 128                          */
  /* device arrays */
  double* lambda;      /* [2k]   eigenvalues lambda_j (re, im)         */
  double* omega;       /* [2k]   omega_j = log(lambda_j)/dt                */
  int32_t* pair;       /* [k]    0 real, +1 first / -1 second member of a pair     */
  double* sigma;       /* [k]    singular values of Y                  */
  double* Mfold;       /* [(m-1) k] folded M = V S^-1 W, column-major, ld m-1      */
  double* beta;        /* [2K]   OMP amplitudes (re, im) on the support    */
  int32_t* support;    /* [K]    selected modes, in selection order                */
  int8_t* Mq;          /* [kpad*limbs][mpad] fixed-point limbs of Mfold            */
  double* Mq_scale;    /* [kpad] per-column dequantisation scales                  */
  float* coef;         /* [2K][m] background coefficients per used Phi column      */
  int32_t* coef_col;   /* [2K]   which folded Phi column each coef row multiplies  */
  int32_t* dev_info;   /* [8]    device-side status words                           */
  /* host outputs of cdmd_fit */
  int32_t k_eff;       /* singular values kept (sigma_j > 1e-6 sigma_1; reading R10) */
  int32_t K_eff;       /* OMP atoms selected (<= K)                                 */
  int32_t n_coef;      /* rows of coef in use (<= 2K)                               */
  int32_t info;        /* 0, or the failing solver's info                           */
  double dt;           /* frame interval used for omega (reading R15: 1)            */
} cdmd_model;

/* ---------------------------------------------------------------- lifecycle */
CDMD_API cdmd_status cdmd_create(int device, cdmd_handle* out);
CDMD_API void cdmd_destroy(cdmd_handle h);
CDMD_API const char* cdmd_status_str(cdmd_status s);
CDMD_API const char* cdmd_version(void);
/* Number of libcdmd kernel launches this process has issued so far (all handles,
 * all streams; cuBLAS / cuSOLVER launches inside cdmd_fit are not counted).
 * Diagnostics: bench.py reports the difference across its timed region.          */
CDMD_API uint64_t cdmd_kernel_launches(void);
/* Eigensolver diagnostics of handle h (cdmd_fit step 4): *runs = fits whose k
 * largest Gram eigenpairs were computed by Lanczos (lanczos.cu),
 * *fallbacks = those of them whose Ritz pairs failed the residual test
 * |beta_{J-1} s_{J-1,i}| <= 1e-9 (theta_i - theta_{k+1}) and were recomputed by the
 * Householder solver.  Either pointer may be NULL.  Errors: CDMD_ERR_ARG (null h).   */
CDMD_API cdmd_status cdmd_eigensolver_stats(cdmd_handle h, uint64_t* runs, uint64_t* fallbacks);

/* Background selection of later cdmd_fit calls on this handle.  omega_eps = 0 (the
 * default): Remark 3's OMP picks at most K modes.  omega_eps > 0: the
 * background is the set of modes with |omega_p| = |log(lambda_p)| / dt < omega_eps
 * ("background modes have |omega_p| ~ 0"), in mode order, at most K (the
 * first K such modes; reading R24), with amplitudes the least-squares fit of the first compressed frame
 * on those modes (the same solve OMP ends with).  Errors: CDMD_ERR_ARG (null
 * handle), CDMD_ERR_RANGE (negative or non-finite omega_eps).                     */
CDMD_API cdmd_status cdmd_set_background_selection(cdmd_handle h, double omega_eps);

/* Spatial SM partition for streaming many batches ("decomposed in consecutive
 * batches"): splits device `device`'s SMs once per process into two green contexts —
 * `fit_sms` SMs (rounded up to the hardware granularity: multiples of 8) reserved for
 * the small solves, the rest for the full-resolution passes — and creates
 * `n_streams` non-blocking streams in each: pass_streams[i] (for cdmd_sketch,
 * cdmd_modes, cdmd_foreground) and fit_streams[i] (for cdmd_fit).  The streams are
 * plain cudaStream_t handles owned by the library for the life of the process.
 * sms[0] / sms[1] receive the SM counts of the solve / pass partitions.  Afterwards the
 * persistent kernels size their grids to sms[1] CTAs on every stream.
 * Errors: CDMD_ERR_ARG (bad pointers or counts, or a partition already exists),
 * CDMD_ERR_RANGE (nothing left for the passes), CDMD_ERR_UNSUPPORTED (driver
 * without green contexts), CDMD_ERR_CUDA.                                        */
CDMD_API cdmd_status cdmd_sm_partition(int device, int fit_sms, int n_streams, void** pass_streams,
                                       void** fit_streams, int* sms);

/* ------------------------------------------------------------------- sketch
 * Y_full = C D (Alg. 1 step 3; Eq. P:286-288), C generated on the fly from
 * Philox4x32-10 and never materialised (single pixel = Feistel
 * permutation rows; sparse = geometric-gap rows; Rademacher = bits; Gaussian =
 * bf16 inverse-CDF table).  Columns of C are indexed by the GLOBAL pixel, so the
 * per-slab partial sketches of a pixel-sharded run SUM to the full sketch
 * (integer kinds bit-exactly).  Y (p x m, ldy >= p) is overwritten.  SRFT: p even,
 * 2 <= p <= 2 n_total, m + 1 <= 512 (the tensor-core kernel), else CDMD_ERR_RANGE /
 * CDMD_ERR_UNSUPPORTED.
 * ws: device workspace of at least cdmd_sketch_workspace_bytes() bytes, 256-B
 * aligned (index lists of C; for Gaussian C also the split-K partial sums, which are
 * reduced in a fixed order so Y is deterministic).  Sparse C: the first call with a
 * given (n_total, p, s, seed) on a handle checks the generated rows against their ELL
 * capacity (mu + 12 sqrt(mu) + 16 entries, mu = n/s) with one stream synchronisation;
 * later calls with that plan do not synchronise (so the first call must not be inside
 * a CUDA graph capture: CDMD_ERR_ARG).  Errors: CDMD_ERR_RANGE if p < 1 or p > n_total,
 * s <= 1 (sparse), m < 2; CDMD_ERR_ARG on layout violations; CDMD_ERR_WORKSPACE;
 * CDMD_ERR_NUMERIC if a sparse row exceeds its capacity (Y is not written). */
CDMD_API size_t cdmd_sketch_workspace_bytes(const cdmd_video* v, const cdmd_sensing* c);
CDMD_API cdmd_status cdmd_sketch(cdmd_handle h, const cdmd_video* v, const cdmd_sensing* c,
                        void* Y, int64_t ldy, void* ws, size_t ws_bytes, cdmd_stream st);

/* ---------------------------------------------------------------------- fit
 * The small solve on Y_full (replicated on every rank after the all-reduce):
 * Alg. 1 step 4 truncated SVD (computed from the Gram matrix Y^T Y, the
 * method of snapshots), step 6 A~ = U* Y' V S^-1, step 7 eig (
 * cuSOLVER), M = V S^-1 W (P:346 without X'), Remark 3 OMP on Phi_Y = Y' M
 * against y_1 (Gram form of Rubinstein et al.), omega =
 * log(lambda)/dt, the background coefficient table, and the
 * fixed-point limbs of M for cdmd_modes.  Target rank: k > 0 fixes it (the
 * configs); k < 0 chooses it by the Gavish-Donoho optimal hard threshold (Remark 2,
 * P:361; the paper's evaluation settings): sigma_j > omega(beta) median(sigma)
 * over all min(p, m-1) singular values of Y, omega(b) = 0.56 b^3 - 0.95 b^2 + 1.82 b
 * + 1.43, b = min(p, m-1) / max(p, m-1), at most -k and at least 1; the result is
 * model->k_eff.  BLOCKING: returns after the model is complete.  Errors:
 * CDMD_ERR_RANGE if |k| < 1, |k| > min(p, m-1), K < 1 or K > |k|;
 * CDMD_ERR_NUMERIC if the eigensolvers fail or every sigma is dropped (model->info
 * holds the solver info).  Symmetric eigensolve (the k largest pairs of Y^T Y): by
 * Lanczos with full reorthogonalisation on one 16-CTA cluster (m - 1 <= 512,
 * 2.25 k + 9 <= 144), accepted only if every Ritz pair passes the residual test (see
 * cdmd_eigensolver_stats), else by the 8-CTA Householder solver (m - 1 <= 510; also for
 * k < 0, which needs every eigenvalue), else cuSOLVER's (syevdx for the k largest;
 * syevd for k < 0).
 * Under stream capture (a CUDA graph of a whole step) cdmd_fit reads nothing back to the
 * host: it keeps the model's sizes from the previous eager fit of the same (p, m, k, K)
 * (k_eff, K_eff, n_coef; CDMD_ERR_UNSUPPORTED if there was none, for k < 0, or when a
 * cuSOLVER path would be needed), takes the symmetric solver the last eager fit of that
 * shape ended with (Lanczos, or Householder after a fallback) and runs no fallback of its
 * own; every replay re-checks
 * itself and sets bit 16 (FLAG_GRAPH_STALE) of model->dev_info[3] when this run's sizes
 * differ, the Lanczos residual test failed or a solver reported an error -- then refit
 * eagerly and recapture. */
CDMD_API size_t cdmd_model_bytes(int k, int K, int64_t m);
CDMD_API cdmd_status cdmd_model_bind(cdmd_model* model, void* dev_buf, size_t bytes, int k, int K, int64_t m);
CDMD_API size_t cdmd_fit_workspace_bytes(cdmd_handle h, int64_t p, int64_t m, int k);
CDMD_API cdmd_status cdmd_fit(cdmd_handle h, const void* Y, int64_t ldy, int32_t kind, int64_t p, int64_t m,
                     int k, int K, double dt, cdmd_model* model, void* ws, size_t ws_bytes,
                     cdmd_stream st);

/* -------------------------------------------------------------------- modes
 * Phi = X' V S^-1 W = X' M (Alg. 1 step 8, Eq. cDMDModes), X' = frames
 * 2..m of the slab; written folded (see "Data layouts"), n_local x
 * k_eff, ldphi >= n_local.  tcgen05 int8 tensor cores on sm_100a: uint8 pixels
 * times int8 limbs of M, exact int32 accumulation, fp32 output. */
CDMD_API cdmd_status cdmd_modes(cdmd_handle h, const cdmd_video* v, const cdmd_model* model,
                       float* Phi, int64_t ldphi, cdmd_stream st);

/* --------------------------------------------------------------- background
 * Background frames t0+1 .. t0+nt of the slab, frame-major L[t*ldl + j]:
 * STATIC  L_j  = Re sum_{p in S} beta_p phi_jp              (every t)
 * DYNAMIC L_jt = Re sum_{p in S} beta_p phi_jp lambda_p^(t-1) (Eq. DMDTerms)
 * Phi as written by cdmd_modes.  Only for inspection: cdmd_foreground fuses it. */
CDMD_API cdmd_status cdmd_background(cdmd_handle h, const float* Phi, int64_t ldphi, int64_t n_local,
                            const cdmd_model* model, int32_t mode, int64_t t0, int64_t nt,
                            float* L, int64_t ldl, cdmd_stream st);

/* --------------------------------------------------------------- foreground
 * One pass over X: background (as cdmd_background), residual |x_jt - L_jt| and
 * threshold tau (Eq. thres, strict >) for all m frames, bit-packed.
 * mask: ldw >= ceil(n_local/32) uint32 words per frame.  Errors: CDMD_ERR_RANGE
 * if tau <= 0. */
CDMD_API cdmd_status cdmd_foreground(cdmd_handle h, const cdmd_video* v, const cdmd_model* model,
                            const float* Phi, int64_t ldphi, int32_t mode, float tau,
                            uint32_t* mask, int64_t ldw, cdmd_stream st);

/* --------------------------------------------------------------- amplitudes
 * Full-state amplitudes b = lstsq(Phi, x_1) (Alg. 1 step 9: "compute
 * amplitudes using x_1 as initial condition"; the paper's alternative to the OMP
 * amplitudes of Remark 3, which cdmd_fit computes on the compressed modes).  Two
 * phases so a pixel-row-sharded run exchanges only k_eff (k_eff + 1) doubles:
 *
 * cdmd_amplitudes_gram: G = [F^T F | F^T x_1] over this slab, F = the folded Phi
 *   of cdmd_modes (n_local x k_eff, ldphi), x_1 = frame 1 of the slab (v->X).  G:
 *   device, k_eff x (k_eff + 1) doubles, column-major, ld k_eff, overwritten.  fp32
 *   sums within 128-pixel tiles, fp64 across tiles, fixed-order reduction
 *   (deterministic).
 *   ws: device, >= cdmd_amplitudes_workspace_bytes(h, k_eff) bytes.  Sum G over the
 *   slabs (e.g. an all-reduce) before the solve.
 * cdmd_amplitudes_solve: Cholesky of F^T F (fp64, one CTA), then b: device,
 *   2 k_eff doubles (re, im) in the mode order of the model; conjugate pairs get
 *   conjugate amplitudes.  A column of F dependent on earlier ones (pivot^2 <=
 *   1e-12 (F^T F)_jj) gets c_j = 0 (a least-squares solution, not lstsq's minimum-
 *   norm one; reading R23); dropped (device int32, may be NULL) receives
 *   how many.  Errors: CDMD_ERR_ARG on null pointers, ldphi < n_local or a model
 *   cdmd_fit has not filled; CDMD_ERR_RANGE if k_eff > 128; CDMD_ERR_WORKSPACE. */
CDMD_API size_t cdmd_amplitudes_workspace_bytes(cdmd_handle h, int k);
CDMD_API cdmd_status cdmd_amplitudes_gram(cdmd_handle h, const cdmd_video* v, const cdmd_model* model,
                                          const float* Phi, int64_t ldphi, double* G, void* ws,
                                          size_t ws_bytes, cdmd_stream st);
CDMD_API cdmd_status cdmd_amplitudes_solve(cdmd_handle h, const cdmd_model* model, const double* G,
                                           double* b, int32_t* dropped, cdmd_stream st);

/* Which kernel a call would run (diagnostics for reports): cdmd_modes -> 1 the
 * tcgen05 kernel (kpad <= 64, m up to 512: SMEM-resident limbs), 2 the 4-CTA cluster
 * tcgen05 kernel (64 < kpad <= 128, m up to ~1500: X' tiles multicast to four CTAs
 * that own 32 columns each), 0 the CUDA-core (dp4a) kernel; cdmd_foreground -> 2 tcgen05 dynamic,
 * 1 CUDA-core dynamic, 0 static.  Negative on invalid arguments. */
CDMD_API int32_t cdmd_modes_path(const cdmd_model* model);
CDMD_API int32_t cdmd_foreground_path(const cdmd_video* v, const cdmd_model* model, int32_t mode);

/* ------------------------------------------- foreground with the median fused
 * The fused single pass (cdmd_foreground with Phi = NULL, N11) with the 3x3 median
 * post-filter of Fig. 7 (as cdmd_mask_median3, zero outside the frame) folded into
 * the same kernel: tiles are 128-pixel chunks of image rows; once every tile of image
 * rows y-1, y, y+1 has written its raw mask words, the CTA that completes them filters
 * row y for all m frames.  Whole frames only: v->pix0 == 0, v->n_local == v->n_total
 * == width * height, width % 32 == 0.
 * raw: the unfiltered mask (m frames of ldw words, as cdmd_foreground writes it);
 * out: the filtered mask (same layout, must not alias raw); ws: device, >=
 * cdmd_foreground_median3_ws_bytes(width, height) bytes (row counters).
 * Errors: CDMD_ERR_ARG (null / aliasing / layout), CDMD_ERR_RANGE (tau <= 0),
 * CDMD_ERR_UNSUPPORTED (width % 32 != 0, or the fused pass unsupported: n_coef > 16 or
 * m > 512), CDMD_ERR_WORKSPACE. */
CDMD_API size_t cdmd_foreground_median3_ws_bytes(int64_t width, int64_t height);
CDMD_API cdmd_status cdmd_foreground_median3(cdmd_handle h, const cdmd_video* v, const cdmd_model* model,
                                             int32_t mode, float tau, int64_t width, int64_t height, uint32_t* raw,
                                             uint32_t* out, int64_t ldw, void* ws, size_t ws_bytes, cdmd_stream st);

/* ------------------------------------------------------------ median post-filter
 * The "in addition median filtered foreground mask" (Fig. 7): a 3x3 spatial
 * median of every frame's mask (on a binary image: bit = 1 iff >= 5 of the 3x3
 * neighbourhood are set), zero outside the frame (reading R22).  mask and
 * out: m frames of ldw uint32 words (bit j % 32 of word j / 32, pixel j = y width + x)
 * covering WHOLE frames (n = width * height pixels, ldw >= ceil(n / 32)); out must
 * not alias mask.  A pixel-row-sharded run needs the neighbouring image rows, so
 * call it on gathered whole frames.  Errors: CDMD_ERR_ARG on null pointers, aliasing
 * or ldw too small; CDMD_ERR_RANGE if width, height or m < 1. */
CDMD_API cdmd_status cdmd_mask_median3(const uint32_t* mask, int64_t ldw, int64_t width, int64_t height,
                                       int64_t m, uint32_t* out, cdmd_stream st);

/* ------------------------------------------------ test hooks (same contract)
 * Export what the device generates so tests can compare it bit for bit with the
 * oracle's definitions. */
/* out: device uint32 [4*count]; ctr: device uint32 [4*count]. */
CDMD_API cdmd_status cdmd_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                        int64_t count, cdmd_stream st);
/* out: device uint16 [65536] bf16 bit patterns of the Gaussian table. */
CDMD_API cdmd_status cdmd_gaussian_table(cdmd_handle h, uint16_t* out, cdmd_stream st);
/* out: device uint16 [16385] fp16 bit patterns of the SRFT quarter wave
 * Q[r] = fp16_RNE(cos(2 pi r / 2^16)), r = 0 .. 2^14 (reading R25). */
CDMD_API cdmd_status cdmd_srft_table(cdmd_handle h, uint16_t* out, cdmd_stream st);
/* Single pixel: rows (device int32 [p]).  SRFT: the p/2 frequencies of R (device int32
 * [p/2]).  Sparse: device int32 [p*cap] ELL of (pos << 1 | negative) and int32 counts
 * [p]; cap from cdmd_sparse_cap(). */
CDMD_API int64_t cdmd_sparse_cap(int64_t n_total, int64_t p, double s);
CDMD_API cdmd_status cdmd_sensing_rows(cdmd_handle h, int64_t n_total, const cdmd_sensing* c,
                              int32_t* rows_or_ell, int32_t* counts, cdmd_stream st);
/* Modes through the CUDA-core (dp4a) reference kernel: bit-identical to
 * cdmd_modes (both accumulate exactly in int32). */
CDMD_API cdmd_status cdmd_modes_simt(cdmd_handle h, const cdmd_video* v, const cdmd_model* model,
                            float* Phi, int64_t ldphi, cdmd_stream st);

/* The on-device small nonsymmetric eigensolver cdmd_fit uses for A~ (k <= 118):
 * A: device k x k column-major (not modified); W: device 2k (re, im), complex
 * pairs consecutive (+im first); VR: device k x k column-major, LAPACK real-geev
 * layout (pair j, j+1 -> Re, Im columns); info: device int, 0 on success. */
CDMD_API cdmd_status cdmd_eig(const double* A, int k, double* W, double* VR, int32_t* info,
                              cdmd_stream st);

#ifdef __cplusplus
}
#endif
#endif /* CDMD_H */
