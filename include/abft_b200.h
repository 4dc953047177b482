/*
 * abft_b200.h — C-ABI of the B200-native ABFT-protected blocked factorization
 * library (libabft_b200.so). Plain pointers and sizes only; no torch types.
 *
 * The reference (`slackwise`, pure Python/numpy) has no FFI; its "operator
 * API" for this hot path is the set of Python names listed in SURVEY.md §8b.
 * Each entry point below names the reference interface it replaces
 * (file:line under /root/reference/pkg/src/slackwise/). The Python mirror in
 * paper_2301_03166_b200/ binds these with ctypes (INTEGRATION.md shows the
 * binding a maintainer would add to the reference).
 *
 * All matrices are column-major (Fortran order, as the reference's
 * `np.asfortranarray` / `order="F"` working copy, linalg.py:78,180), float64.
 * Return codes: 0 on success, negative on error (see ABFT_E_*); the message
 * is available from abft_last_error() on the calling thread.
 */
#ifndef ABFT_B200_H
#define ABFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define ABFT_API __attribute__((visibility("default")))
#else
#define ABFT_API
#endif

/* error codes -------------------------------------------------------------- */
#define ABFT_OK 0
#define ABFT_E_INVALID (-1)   /* ValueError (e.g. encode with scheme NONE, abft.py:97-98) */
#define ABFT_E_DIM (-2)       /* InvalidDimensionError (linalg.py:37-38, :52-53, :313-316) */
#define ABFT_E_BREAKDOWN (-3) /* NumericBreakdownError (linalg.py:41-43, :223-224, :234-235) */
#define ABFT_E_RANGE (-4)     /* IndexError: fault outside matrix (abft.py:287-288) */
#define ABFT_E_INCOMPLETE (-5)/* reconstruct before completion (linalg.py:341-342) */
#define ABFT_E_OVERFLOW (-6)  /* event buffer too small */
/* <= -1000: CUDA runtime error (-1000 - cudaError_t) */

/* enums mirror DecompositionKind / ChecksumScheme / ErrorKind / TaskKind ---- */
enum { ABFT_CHOLESKY = 0, ABFT_LU = 1, ABFT_QR = 2 };          /* linalg.py:24-27 */
enum { ABFT_NONE = 0, ABFT_SINGLE = 1, ABFT_FULL = 2 };         /* abft.py:36-39 */
enum { ABFT_D0 = 0, ABFT_D1 = 1, ABFT_D2 = 2 };                 /* abft.py:42-45 */
enum { ABFT_TASK_PD = 0, ABFT_TASK_PU = 1, ABFT_TASK_TMU = 2 };  /* linalg.py:30-34 */

/* One planned fault (InjectedFault, abft.py:48-57). Two magnitude forms:
 *  absolute != 0: `magnitude` is applied as given (inject_faults, abft.py:283-307)
 *  absolute == 0: magnitude = (u * 1e-3) * max(scale, 1), negated if `negate`,
 *                 with scale = max|region| computed on the device after the
 *                 trailing update — exactly sample_fault_plan's formula
 *                 (abft.py:319-321, simulator.py:159-162); the host draws
 *                 (row, col, u, negate) with the caller's numpy Generator. */
typedef struct {
  int32_t kind;        /* ABFT_D0/D1/D2 */
  int32_t orientation; /* 0 = "col", 1 = "row" (1-D streak direction) */
  int64_t row;         /* global row */
  int64_t col;         /* global column */
  int32_t extent;
  int32_t absolute;
  double u;
  int32_t negate;
  int32_t _pad;
  double magnitude;
} abft_fault;

/* One CorrectionReport location (abft.py:60-84): (row, col, kind, flag). For a
 * corrected 0-D element row/col are the element's global indices; otherwise
 * the block's top-left corner. `detected_kind` is the ErrorKind counted in
 * report.detected for this event; `corrected` says report.corrected was
 * incremented; `uncorrectable` says report.uncorrectable was set. */
typedef struct {
  int64_t row;
  int64_t col;
  int32_t kind;
  int32_t flag;
  int32_t detected_kind;
  int32_t corrected;
  int32_t uncorrectable;
  int32_t block_row; /* region-local block indices (ordering key) */
  int32_t block_col;
  int32_t seq;
} abft_location;

typedef struct {
  int64_t detected[3];
  int64_t corrected[3];
  int32_t uncorrectable;
  int32_t n_locations; /* events produced (may exceed the caller's buffer) */
} abft_report;

/* library ------------------------------------------------------------------ */
ABFT_API int abft_version(void);
ABFT_API const char* abft_last_error(void);
ABFT_API int abft_device_count(int* count);
/* kernels launched by this library so far (process-wide counter) */
ABFT_API long long abft_launch_count(void);
/* Diagnostic: while enabled, every verify launch records the largest
 * |delta| / tau among checks that did NOT trip (column sums, row sums,
 * index-weighted column sums) on the current device: the rounding-noise
 * margin of the threshold rule (abft.py:161-163); out3[3] (a 4th slot) is the
 * largest |dw/dp - round(dw/dp)| seen by SINGLE's index recovery
 * (abft.py:208-213). `out3` holds 4 doubles. No reference counterpart. */
ABFT_API int abft_noise_stats(int enable);
ABFT_API int abft_noise_read(double* out3, int reset);

/* device-pointer primitive (for integrators that own device memory):
 * D = beta*C + alpha*op(A)*op(B) on `stream` (cudaStream_t, may be NULL). */
ABFT_API int abft_dev_dgemm(void* stream, char transa, char transb, int64_t m, int64_t n,
                            int64_t k, double alpha, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double beta, const double* C,
                            int64_t ldc, double* D, int64_t ldd);

/* fp32 device-pointer GEMM on the tcgen05 tensor cores (kind::tf32 with a
 * 3xTF32 split for fp32 accuracy): D = beta*C + alpha*op(A)*op(B). */
ABFT_API int abft_dev_sgemm(void* stream, char transa, char transb, int64_t m, int64_t n,
                            int64_t k, float alpha, const float* A, int64_t lda, const float* B,
                            int64_t ldb, float beta, const float* C, int64_t ldc, float* D,
                            int64_t ldd);

/* the same with an explicit split-K factor: `splits` K-slices accumulate in
 * separate tensor-core chains, reduced in a fixed order (the s* Cholesky /
 * QR deep-K updates use this internally). */
ABFT_API int abft_dev_sgemm_splitk(void* stream, char transa, char transb, int64_t m, int64_t n,
                                   int64_t k, float alpha, const float* A, int64_t lda,
                                   const float* B, int64_t ldb, float beta, const float* C,
                                   int64_t ldc, float* D, int64_t ldd, int splits);

/* diagonal-block factorization on device pointers: the PD kernel of
 * linalg.py:219-238 (mode 0 LU unpivoted, 1 Cholesky) and mode 2, the
 * sign-shifted LU of the QR panel's Householder reconstruction (linalg.py:
 * 260-300). D (w x w, w <= 256) in place; Linv = L^{-1}, Uinv = U^{-1} (LU
 * modes; may be NULL); sgn: the mode-2 signs. variant 0 = one CTA, 1 = the
 * thread-block-cluster kernel. info_dev: device int set to 1 + the column of
 * the first breakdown (LU pivot 0 / non-finite, Cholesky pivot <= 0). */
ABFT_API int abft_dev_diag_factor(void* stream, int variant, int mode, int64_t w, double* D,
                                  int64_t ld, double* Linv, int64_t ldl, double* Uinv,
                                  int64_t ldu, int* info_dev, double* sgn);
ABFT_API int abft_dev_sdiag_factor(void* stream, int variant, int mode, int64_t w, float* D,
                                   int64_t ld, float* Linv, int64_t ldl, float* Uinv, int64_t ldu,
                                   int* info_dev, float* sgn);

/* factorization context: replaces Factorization (linalg.py:159-359) -------- */
typedef struct abft_ctx abft_ctx;

/* Factorization(kind, a0, b).__post_init__ (linalg.py:175-180). */
ABFT_API int abft_create(abft_ctx** ctx, int kind, int64_t n, int64_t b, int device);
ABFT_API int abft_destroy(abft_ctx* ctx);
/* copy the host input (column-major, leading dim lda) into the device working matrix */
ABFT_API int abft_set_matrix(abft_ctx* ctx, const double* a, int64_t lda);
/* like abft_set_matrix, but the copy happens inside the next abft_factorize
 * call, column block by column block on a copy stream, overlapped with the
 * factorization (Cholesky copies only rows >= j*b of block column j, the lower
 * block triangle it reads, and waits per block; LU / QR wait for the whole
 * matrix). `a` (pinned for an asynchronous copy) must stay valid until that
 * call returns; other entries that touch the matrix copy it first. Replaces
 * the host-to-device half of the e2e round trip (bench.py run_e2e). */
ABFT_API int abft_set_matrix_streamed(abft_ctx* ctx, const double* a, int64_t lda);
/* keep a device copy of the input for abft_residual(ctx, NULL, ...) */
ABFT_API int abft_keep_input(abft_ctx* ctx, int keep);
/* restore the working matrix from the kept input (needs abft_keep_input) */
ABFT_API int abft_reset(abft_ctx* ctx);
/* the context's cudaStream_t (for timing with events on the launching stream) */
ABFT_API void* abft_stream(abft_ctx* ctx);
/* m <- m m^T + n I on the device (SPD construction of linalg.py:74-75) */
ABFT_API int abft_make_spd(abft_ctx* ctx);
/* Factorization.m (host mirror): copy the device working matrix out */
ABFT_API int abft_get_matrix(abft_ctx* ctx, double* m, int64_t ldm);
/* Factorization.k_done */
ABFT_API int64_t abft_k_done(abft_ctx* ctx);
ABFT_API int abft_set_k_done(abft_ctx* ctx, int64_t k);
/* task_pd / task_pu / task_tmu (linalg.py:192-258), unprotected */
ABFT_API int abft_task(abft_ctx* ctx, int64_t k, int task);
/* run_numeric_iteration (simulator.py:97-121): PD/PU + protected TMU with the
 * fault plan injected between maintenance and verification. Synchronous;
 * fills `rep` and up to `max_locs` locations in reference order. */
ABFT_API int abft_iteration(abft_ctx* ctx, int64_t k, int scheme, const abft_fault* plan,
                            int nplan, int correct, abft_report* rep, abft_location* locs,
                            int max_locs);
/* Whole remaining factorization in one call (no per-iteration host sync).
 * schemes[k] per iteration (NULL: `scheme` for all); faults are given as a
 * flat plan with plan_iter[i] = iteration of fault i (plans pre-drawn on the
 * host in sample_fault_plan order). reports: n_blocks entries (may be NULL). */
ABFT_API int abft_factorize(abft_ctx* ctx, int scheme, const int32_t* schemes,
                            const abft_fault* plan, const int64_t* plan_iter, int nplan,
                            int correct, abft_report* reports, abft_location* locs,
                            int max_locs, int* n_locs);
/* stream the finished factor to `host` (ldh) during the next abft_factorize
 * calls: each column block is copied on a copy stream as soon as it is final,
 * overlapping the rest of the factorization (NULL: off) */
ABFT_API int abft_stream_out(abft_ctx* ctx, double* host, int64_t ldh);
/* QR side data: qr_t[k] (w x w) and _qr_vs[k] (nk x w) (linalg.py:294-308) */
ABFT_API int abft_qr_panels(abft_ctx* ctx);
/* `del qr_t[n:]` / _qr_vs truncation in _Run._restore (simulator.py:431-435) */
ABFT_API int abft_set_qr_panels(abft_ctx* ctx, int count);
ABFT_API int abft_get_qr_panel(abft_ctx* ctx, int64_t k, double* V, int64_t ldv, double* T,
                               int64_t ldt);
/* per-task device timers (CUDA events): enable/reset, then read
 * ms[0]=PD, ms[1]=PU, ms[2]=TMU GEMMs, ms[3]=ABFT encode/maintain/verify/inject */
ABFT_API int abft_profile(abft_ctx* ctx, int enable);
ABFT_API int abft_profile_read(abft_ctx* ctx, double* ms);
/* LU with partial pivoting (LAPACK dgetrf semantics, P A = L U), an option:
 * the reference factors LU unpivoted (linalg.py:230-238); set before
 * iteration 0. abft_get_pivots: n global 0-based rows (row i interchanged
 * with piv[i], in order; LAPACK ipiv - 1), identity when off. */
ABFT_API int abft_set_pivoting(abft_ctx* ctx, int enable);
ABFT_API int abft_get_pivots(abft_ctx* ctx, int32_t* piv);
/* per-iteration device times since abft_profile(ctx, 1): out[4k + t], t = PD
 * (a look-ahead's side-stream panel included), PU, TMU GEMMs, ABFT work */
ABFT_API int abft_profile_read_iters(abft_ctx* ctx, double* out, int64_t nb);
/* per-iteration SMs left to the panel work beside a look-ahead update (QR:
 * the side-stream panel; LU: >= ceil(b/32) selects the multi-CTA diagonal
 * factor); NULL / 0 = built-in choice. The run modes' slack-reclamation lever
 * (replaces the reference's DVFS decisions, scheduler.py:84-146). */
ABFT_API int abft_set_side_sms(abft_ctx* ctx, const int32_t* sms, int64_t nb);
/* streamed input of LU / QR (abft_set_matrix_streamed): block columns
 * [0, split b) are factored chunk by chunk (`chunk` block columns each,
 * left-looking over the chunks) while the input arrives; the rest receives
 * their updates as it arrives, in `right_chunk` block-column pieces (0: all
 * at once). chunk = 0 waits for the whole input. -1 = built-in: LU chunk
 * n_blocks / 8, split 3 n_blocks / 8, right part at once; QR chunk 1, split
 * 3, right_chunk n_blocks / 8 (its panels serialise inside chunks). Same
 * factor and reports either way. Used only when no fault is planned before
 * iteration `split`. */
ABFT_API int abft_set_input_chunks(abft_ctx* ctx, int chunk, int64_t split, int right_chunk);
/* FP64 DMMA issue-rate probe (TFLOP/s) over all SMs: the roofline denominator */
ABFT_API int abft_probe_dmma_peak(int iters, double* tflops);
/* in-device snapshot slots replacing _Run._snapshot/_restore (simulator.py:420-436) */
ABFT_API int abft_snapshot(abft_ctx* ctx, int slot);
ABFT_API int abft_restore(abft_ctx* ctx, int slot);
/* residual(a, factors) (linalg.py:362-368); a0 == NULL uses the kept input */
ABFT_API int abft_residual(abft_ctx* ctx, const double* a0, int64_t lda, double* out);
/* Factorization.reconstruct() (linalg.py:340-359) into a host n x n array */
ABFT_API int abft_reconstruct(abft_ctx* ctx, double* out, int64_t ldo);
/* test/debug accessor for the device checksum arrays (see ctx.cu) */
ABFT_API int abft_debug_array(abft_ctx* ctx, int which, double* out, int64_t* rows,
                              int64_t* cols);
/* column index of the last NumericBreakdownError */
ABFT_API int64_t abft_breakdown_column(abft_ctx* ctx);
/* synchronize the context stream and return accumulated device time (ms) of
 * the last abft_factorize/abft_iteration call, measured with CUDA events */
ABFT_API int abft_last_elapsed_ms(abft_ctx* ctx, double* ms);

/* 1-D block-cyclic distribution over G processes, one GPU each (SURVEY.md
 * §8e; no reference counterpart: the reference is single-process). Rank g
 * owns global column blocks j with j mod G == g, stored contiguously. The
 * exchange step is the caller's (torch.distributed / NCCL) on the device
 * buffer `xbuf` (abft_dist_xbuf_elems(k) doubles) between the phases:
 *   LU/QR : begin (owner of k packs the factored panel) -> broadcast from
 *           owner k mod G -> update -> [all-reduce MAX of *local_max when
 *           faults are planned] -> finish
 *   Chol. : begin (every rank: partial left-looking products) -> sum-reduce
 *           to owner k mod G -> update -> [all-reduce MAX] -> finish
 * One iteration = run_numeric_iteration (simulator.py:97-121) with the same
 * host-drawn plan on every rank (abft.py:310-333). ----------------------- */
typedef struct abft_dist abft_dist;
ABFT_API int abft_dist_create(abft_dist** d, int kind, int64_t n, int64_t b, int device, int rank,
                              int world);
ABFT_API int abft_dist_destroy(abft_dist* d);
ABFT_API int64_t abft_dist_local_cols(abft_dist* d);
ABFT_API void* abft_dist_stream(abft_dist* d);
/* doubles exchanged at iteration k (0: no exchange) */
ABFT_API int64_t abft_dist_xbuf_elems(abft_dist* d, int64_t k);
/* owned column blocks of the host global matrix (column-major, lda) -> device */
ABFT_API int abft_dist_set_matrix(abft_dist* d, const double* a, int64_t lda);
/* keep a device copy of the local input; abft_dist_reset restores it */
ABFT_API int abft_dist_keep_input(abft_dist* d, int keep);
ABFT_API int abft_dist_reset(abft_dist* d);
/* the rank's own column blocks (n x local_cols, ldl) -> device */
ABFT_API int abft_dist_set_local(abft_dist* d, const double* local, int64_t ldl);
/* local columns (n x local_cols) -> host */
ABFT_API int abft_dist_get_matrix(abft_dist* d, double* out, int64_t ldo);
ABFT_API int abft_dist_begin(abft_dist* d, int64_t k, int scheme, double* xbuf);

/* The exchange step of iteration k (between abft_dist_begin and
 * abft_dist_update): returns 0 none, 1 broadcast from *root, 2 sum-reduce
 * to *root (left-looking Cholesky, ABFT_DIST_CHOL=left), over
 * abft_dist_xbuf_elems(k) doubles. Right-looking Cholesky (default)
 * broadcasts panel k-1 from its owner at iteration k. */
ABFT_API int abft_dist_exchange(abft_dist* d, int64_t k, int* root);
ABFT_API int abft_dist_update(abft_dist* d, int64_t k, int scheme, const double* xbuf, int nplan,
                              double* local_max);
/* scale: device pointer to the all-reduced max|region| (NULL if nplan == 0) */
ABFT_API int abft_dist_finish(abft_dist* d, int64_t k, int scheme, const abft_fault* plan,
                              int nplan, int correct, const double* scale);
/* synchronize, check breakdown, drain events (global coordinates; iters[i] = iteration) */
ABFT_API int abft_dist_events(abft_dist* d, abft_location* locs, int64_t* iters, int max_locs,
                              int* n_out);
ABFT_API int64_t abft_dist_k_done(abft_dist* d);
ABFT_API int abft_dist_get_qr_panel(abft_dist* d, int64_t k, double* V, int64_t ldv, double* T,
                                    int64_t ldt);
/* LU look-ahead across ranks: before update(k), hand the buffer for panel
 * k+1; its owner factors and packs it mid-update, then the caller broadcasts
 * it from rank (k+1) mod G on abft_dist_comm_stream() and calls
 * abft_dist_comm_done(); begin(k+1) waits for that broadcast. */
ABFT_API int abft_dist_lookahead(abft_dist* d, int64_t k, double* xnext);
ABFT_API void* abft_dist_comm_stream(abft_dist* d);
ABFT_API int abft_dist_comm_done(abft_dist* d);
/* device time from the first begin(0) to the last finish (CUDA events) */
ABFT_API int abft_dist_elapsed_ms(abft_dist* d, double* ms);
/* single-context QR panel setter (rebuild a gathered factorization for the residual) */
ABFT_API int abft_set_qr_panel(abft_ctx* ctx, int64_t k, const double* V, int64_t ldv,
                               const double* T, int64_t ldt);

/* single precision (the s* variants: sgetrf / spotrf / sgeqrf) ------------
 * Same task order, regions, fault plan semantics, events and error codes as
 * the fp64 context above; fp32 data (tcgen05 kind::tf32 GEMMs with a 3xTF32
 * split), fp64 block checksums, tau = 50 * b * max(max|blk|, 1) * eps32;
 * the QR Householder panel is factored in fp64 from the widened fp32 panel.
 * The reference has no fp32 path (parity unpinned). */
typedef struct abft_sctx abft_sctx;
ABFT_API int abft_s_create(abft_sctx** ctx, int kind, int64_t n, int64_t b, int device);
/* streamed fp32 input: as abft_set_input_chunks (sgetrf; built-in chunk and split
 * n_blocks / 4; QR is not chunked in fp32) */
ABFT_API int abft_s_set_input_chunks(abft_sctx* ctx, int chunk, int64_t split, int right_chunk);
ABFT_API int abft_s_destroy(abft_sctx* ctx);
ABFT_API void* abft_s_stream(abft_sctx* ctx);
ABFT_API int64_t abft_s_k_done(abft_sctx* ctx);
ABFT_API int abft_s_keep_input(abft_sctx* ctx, int keep);
ABFT_API int abft_s_set_matrix(abft_sctx* ctx, const float* a, int64_t lda);
/* fp32 twin of abft_set_matrix_streamed */
ABFT_API int abft_s_set_matrix_streamed(abft_sctx* ctx, const float* a, int64_t lda);
ABFT_API int abft_s_reset(abft_sctx* ctx);
ABFT_API int abft_s_make_spd(abft_sctx* ctx);
ABFT_API int abft_s_get_matrix(abft_sctx* ctx, float* m, int64_t ldm);
ABFT_API int abft_s_iteration(abft_sctx* ctx, int64_t k, int scheme, const abft_fault* plan,
                              int nplan, int correct, abft_report* rep, abft_location* locs,
                              int max_locs);
ABFT_API int abft_s_factorize(abft_sctx* ctx, int scheme, const int32_t* schemes,
                              const abft_fault* plan, const int64_t* plan_iter, int nplan,
                              int correct, abft_report* reports, abft_location* locs,
                              int max_locs, int* n_locs);
ABFT_API int abft_s_last_elapsed_ms(abft_sctx* ctx, double* ms);
/* one in-device snapshot slot (the recompute recovery policy) */
ABFT_API int abft_s_snapshot(abft_sctx* ctx);
ABFT_API int abft_s_restore(abft_sctx* ctx);
/* stream the finished factor to `host` during the next abft_s_factorize calls */
ABFT_API int abft_s_stream_out(abft_sctx* ctx, float* host, int64_t ldh);
ABFT_API int abft_s_profile(abft_sctx* ctx, int enable);
ABFT_API int abft_s_profile_read(abft_sctx* ctx, double* ms);
ABFT_API int abft_s_residual(abft_sctx* ctx, const float* a0, int64_t lda, double* out);
ABFT_API int64_t abft_s_breakdown_column(abft_sctx* ctx);

/* region ABFT on host arrays: encode / maintain_gemm / verify_correct /
 * inject_faults (abft.py:118-307), executed on the device. Checksums are
 * column-major arrays: col_plain/col_weighted (nbr x cols, ld nbr),
 * row_plain/row_weighted (rows x nbc, ld rows), block_max (nbr x nbc). ------ */
ABFT_API int abft_region_encode(const double* m, int64_t ldm, int64_t rows, int64_t cols,
                                int64_t b, int scheme, double* col_plain, double* col_weighted,
                                double* row_plain, double* row_weighted);
ABFT_API int abft_region_maintain(int64_t rows, int64_t cols, int64_t kdim, int64_t b, int scheme,
                                  const double* left, int64_t ldl, const double* right,
                                  int64_t ldr, double* col_plain, double* col_weighted,
                                  double* row_plain, double* row_weighted);
ABFT_API int abft_region_verify(double* m, int64_t ldm, int64_t rows, int64_t cols, int64_t b,
                                int scheme, int correct, int64_t r0, int64_t c0,
                                const double* col_plain, const double* col_weighted,
                                const double* row_plain, abft_report* rep, abft_location* locs,
                                int max_locs);
ABFT_API int abft_inject(double* m, int64_t ldm, int64_t n_rows, int64_t n_cols,
                         const abft_fault* plan, int nplan, double scale);

#ifdef __cplusplus
}
#endif
#endif /* ABFT_B200_H */
