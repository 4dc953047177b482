// Factorization context + protected-iteration driver (C-ABI).
//
// Restates, on one B200, the reference's numeric engine and protected
// iteration (/root/reference/pkg/src/slackwise/):
//   Factorization            linalg.py:159-359
//   _tmu_region              simulator.py:86-94
//   run_numeric_iteration    simulator.py:97-121
//   _protected_tmu           simulator.py:124-167
//   residual / reconstruct   linalg.py:340-368
// Device data layout: the working matrix is column-major with
// an even leading dimension (TMA stride rule); per-block checksums live on the
// GLOBAL b-grid so the verify pass of iteration k is the encode of k+1 for LU
// and QR (their next region is a block-aligned sub-grid untouched by PD/PU).
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "abft_b200.h"
#include "abft_kernels.cuh"
#include "gemm.cuh"
#include "panel.cuh"

using namespace abft;

namespace {

inline int64_t round_even(int64_t x) { return (x + 1) / 2 * 2; }
inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

enum { PROF_PD = 0, PROF_PU = 1, PROF_TMU = 2, PROF_ABFT = 3, PROF_N = 4 };

struct Snapshot {
  double* m = nullptr;
  double* chol_rs = nullptr;
  bool chol_rs_valid = false;
  int64_t k_done = 0;
  int qr_count = 0;
  bool used = false;
};

}  // namespace

struct abft_ctx {
  int kind = 0;
  int64_t n = 0, b = 0, nb = 0, ld = 0;
  int device = 0;
  cudaStream_t st = nullptr;

  double* m = nullptr;
  double* a0 = nullptr;  // kept input (optional)
  bool keep_input = false;

  // checksums on the global block grid
  double* gcsw = nullptr;  // (2nb) x n, ld_cs: row 2*gbi plain, 2*gbi+1 weighted
  int64_t ld_cs = 0;
  double* grs = nullptr;   // n x nb row sums, ld
  double* gmax = nullptr;
  double* fpart = nullptr;  // fused-epilogue per-strip row sums (ld x 4nb, region-local)
  double* fmaxp = nullptr;  // fused-epilogue per-strip max (ld_max x 4nb)  // nb x nb, ld_max
  int64_t ld_max = 0;
  double* csm = nullptr;   // maintained col sums of the current region (2nb x n, ld_cs)
  double* rsm = nullptr;   // maintained row sums (n x nb, ld)
  double* el = nullptr;    // operand block-row sums (2nb x b, ld_cs)
  double* er = nullptr;    // R * E_R (b x nb, ld_t)
  double* chol_rs = nullptr;  // Cholesky running row checksums of future panels (n x nb)
  bool chol_rs_valid = false;

  // workspaces
  int64_t ld_t = 0;     // leading dim of b x b / b x n buffers
  double* lw = nullptr;    // n x b
  double* uw = nullptr;    // b x n (ld_t)
  double* linv = nullptr;  // b x b
  double* uinv = nullptr;  // b x b
  double* vstore = nullptr;  // QR V panels (n x n, ld)
  double* tstore = nullptr;  // QR T factors (nb of b x b, ld_t)
  double* betas = nullptr;
  double* qr_part = nullptr;
  int64_t qr_part_elems = 0;
  double* qr_rowbuf = nullptr;
  double* qr_part2 = nullptr;  // 148 x 32 x b block-update partials
  double* qr_wfin = nullptr;   // 32 x b
  double* gram = nullptr;    // b x b
  double* qr_small = nullptr;  // QR_SMALL_BUFS x (ld_t x b): panel fast path
  QrPanelWork qrw;             // qr_panel_factor workspace (Q1 = lw)
  double* ww = nullptr;      // b x n
  double* mid = nullptr;     // b x n
  double* scratch = nullptr; // 4096 doubles
  GemmWorkspace gws;

  // events / lists
  Event* ev = nullptr;
  int32_t* counters = nullptr;  // [0] events, [1] dirty
  int ev_cap = 0;
  int32_t* dirty = nullptr;
  int dirty_cap = 0;
  DevFault* dplan = nullptr;
  int dplan_cap = 0;
  int32_t* dlist = nullptr;
  int dlist_cap = 0;
  int* info = nullptr;

  // host state
  int64_t k_done = 0;
  bool sums_valid = false;
  int64_t breakdown_col = -1;
  int qr_count = 0;
  std::vector<Snapshot> snaps;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool timed = false;
  int32_t cur_iter = 0;
  bool fuse_enabled = true;       // ABFT_NO_FUSE=1 disables (A/B testing)
  bool want_chol_rs = false;      // abft_factorize: a later iteration uses FULL
  bool lookahead_enabled = true;  // ABFT_NO_LOOKAHEAD=1 disables
  int64_t pd_ready = -1;          // panel already factored by the look-ahead
  int64_t pu_ready = -1;          // PU already applied by the LU look-ahead (depth 2)
  bool lu_la2 = false;            // LU look-ahead also forms PU(k+1), L21(k+1) on the side
                                  // stream beside the update (ABFT_LU_LA2=1). Off: measured
                                  // slower (dgetrf N = 32768 845 -> 850 ms: the side chain's
                                  // SMs cost the update more than the serial PU / L21 did)
  int64_t chol_part = -1;         // Cholesky: panel whose update from panels 0..k-2 is done
  bool chol_enc_ahead = false;    // ... and whose encode ran with it
  int next_scheme = 0;            // scheme of the next iteration (abft_factorize)
  GemmWorkspace gws2;             // split-K workspace of the side stream
  int qr_la_sms = 16;             // QR look-ahead: SMs left to the side-stream panel
  bool qr_la_sms_fixed = false;   // ABFT_QR_LA_SMS=R fixes it; else qr_panel_sms's model
  bool pivot = false;             // LU with partial pivoting (abft_set_pivoting)
  int32_t* ipiv = nullptr;        // n: panel-local pivot rows of each panel
  double* piv_part = nullptr;     // lu_panel_pivot partials
  int64_t piv_part_elems = 0;
  bool lu_coop = true;            // late LU look-ahead iterations: multi-CTA diagonal factor
                                  // (ABFT_LU_COOP=0: always the one-CTA kernel)
  bool chol_cluster = false;      // Cholesky PD on the cluster kernel, submitted ahead of
                                  // the look-ahead update (ABFT_CHOL_CLUSTER=1). Off for
                                  // fp64: PD is hidden behind the K = p update, whose
                                  // 8-SM cap then costs more (dpotrf 27.9 -> 27.0 TF/s)
  // streamed result (abft_stream_out): finished column blocks are copied to
  // this host buffer on a copy stream while the factorization continues
  double* out_host = nullptr;
  int64_t out_ld = 0;
  cudaStream_t st_out = nullptr;
  cudaEvent_t ev_out = nullptr;
  cudaStream_t st2 = nullptr;     // side stream for look-ahead panels
  cudaEvent_t ev_a = nullptr, ev_p = nullptr, ev_r = nullptr;
  // streamed input (abft_set_matrix_streamed): the next abft_factorize call
  // copies the column blocks on st_in (Cholesky: only rows >= j b of block j,
  // the lower block triangle the algorithm reads) and each iteration waits
  // for the block it is about to touch, so the H2D overlaps the factorization
  const double* in_host = nullptr;
  int64_t in_ld = 0;
  bool in_stream = false;         // the running abft_factorize consumes streamed blocks
  cudaStream_t st_in = nullptr;
  std::vector<cudaEvent_t> ev_in;
  std::vector<char> rs_enc;       // streamed Cholesky FULL: block column's row sums added
  double* rs_tmp = nullptr;       // n: fresh row sums of one block column
  // streamed LU input: block columns [0, lu_split b) are factored left-looking
  // in chunks of lu_chunk block columns as they arrive (lu_stream_chunks);
  // L11^{-1} of every panel is kept for the late PU of the next chunks
  int lu_chunk = -1;              // ABFT_STREAM_CHUNK (0: wait for the whole input; -1: LU nb / 8,
                                  // QR 0 -- measured slower, see lu_stream_chunk)
  int64_t lu_split = -1;          // ABFT_STREAM_SPLIT (block columns; -1: 3 nb / 8)
  int lu_rchunk = -1;             // right part's catch-up chunks (0: all of it at once;
                                  // -1: LU 0, QR nb / 8)
  double* linv_store = nullptr;   // nb x (ld_t x b)
  double* el_store = nullptr;     // nb x (ld_cs x b): block-row sums of each L panel
  std::vector<char> el_ok;
  // profiling
  struct ProfPair {
    int cat;
    int32_t iter;
    cudaEvent_t e0, e1;
  };
  std::vector<std::array<double, 4>> prof_iter;  // per-iteration PD/PU/TMU/ABFT ms
  cudaEvent_t prof_open2 = nullptr;              // side-stream (look-ahead) PD bracket
  // per-iteration SMs left to the panel work beside a look-ahead update
  // (abft_set_side_sms; empty = the built-in choice): the run modes' lever
  std::vector<int32_t> side_sms;
  bool prof_on = false;
  double prof_ms[4] = {0, 0, 0, 0};
  std::vector<ProfPair> prof_pending;
  std::vector<cudaEvent_t> prof_free;
  cudaEvent_t prof_open[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

cudaEvent_t prof_event(abft_ctx* c) {
  if (!c->prof_free.empty()) {
    cudaEvent_t e = c->prof_free.back();
    c->prof_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

void prof_mark(abft_ctx* c, int cat, bool begin) {
  if (!c->prof_on) return;
  cudaEvent_t e = prof_event(c);
  cudaEventRecord(e, c->st);
  if (begin) {
    c->prof_open[cat] = e;
  } else {
    c->prof_pending.push_back({cat, c->cur_iter, c->prof_open[cat], e});
    c->prof_open[cat] = nullptr;
  }
}

// Bracket on the side stream (the look-ahead's panel k+1, or Cholesky's
// early update of panel k+1, credited to iteration k+1)
void prof_mark_side(abft_ctx* c, bool begin, int32_t iter, int cat = PROF_PD) {
  if (!c->prof_on) return;
  cudaEvent_t e = prof_event(c);
  cudaEventRecord(e, c->st2);
  if (begin) {
    c->prof_open2 = e;
  } else {
    c->prof_pending.push_back({cat, iter, c->prof_open2, e});
    c->prof_open2 = nullptr;
  }
}

namespace {

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool poison_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ABFT_POISON");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Device allocation; with ABFT_POISON=1 every buffer starts as NaN so a read
// of never-written memory shows up deterministically (debug aid).
int dalloc(double** p, int64_t elems) {
  CUDA_TRY(cudaMalloc(p, std::max<int64_t>(elems, 1) * sizeof(double)));
  if (poison_enabled())
    CUDA_TRY(cudaMemset(*p, 0xFF, std::max<int64_t>(elems, 1) * sizeof(double)));
  if (poison_enabled()) CUDA_TRY(cudaDeviceSynchronize());  // order before non-blocking streams
  return 0;
}

void region_of(const abft_ctx* c, int64_t k, int64_t* r0, int64_t* c0, int64_t* rows,
               int64_t* cols) {
  // _tmu_region (simulator.py:86-94)
  const int64_t p = k * c->b, pe = std::min(p + c->b, c->n);
  if (c->kind == ABFT_CHOLESKY) {
    *r0 = p; *c0 = p; *rows = c->n - p; *cols = pe - p;
  } else if (c->kind == ABFT_LU) {
    *r0 = pe; *c0 = pe; *rows = c->n - pe; *cols = c->n - pe;
  } else {
    *r0 = p; *c0 = pe; *rows = c->n - p; *cols = c->n - pe;
  }
}

// Column block k is final (LU/QR after PD(k), Cholesky after PU(k)): queue
// its device-to-host copy on the copy stream behind the main stream's work.
// Unpivoted LU emits its U rows earlier (emit_rowblock, after each PU), so a
// column block here carries only rows >= k b: the D2H of the late, tall U
// columns no longer piles up behind the last iterations (dgetrf N = 32768:
// the streamed output added 23 ms to the call before).
int emit_column(abft_ctx* c, int64_t k) {
  if (!c->out_host) return 0;
  const int64_t p = k * c->b, w = std::min(c->b, c->n - p);
  const int64_t r0 = (c->kind == ABFT_LU && c->pivot) ? 0 : p;
  CUDA_TRY(cudaEventRecord(c->ev_out, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st_out, c->ev_out, 0));
  CUDA_TRY(cudaMemcpy2DAsync(c->out_host + r0 + p * c->out_ld, c->out_ld * 8, c->m + r0 + p * c->ld,
                             c->ld * 8, (c->n - r0) * 8, w, cudaMemcpyDeviceToHost, c->st_out));
  return 0;
}

// Unpivoted LU: row block k of U over columns [cs, ce) is final after PU(k)
// (nothing updates it again): queue its D2H. Cholesky: the same row block is
// zeroed by PU(k) (linalg.py:251-252) and final too. QR: row block k of R is
// final after the verified TMU(k).
int emit_rowblock(abft_ctx* c, int64_t k, int64_t cs, int64_t ce) {
  if (!c->out_host || c->pivot) return 0;
  const int64_t p = k * c->b, pe = std::min(p + c->b, c->n), w = pe - p;
  cs = std::max(cs, pe);
  ce = std::min(ce, c->n);
  if (cs >= ce) return 0;
  CUDA_TRY(cudaEventRecord(c->ev_out, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st_out, c->ev_out, 0));
  CUDA_TRY(cudaMemcpy2DAsync(c->out_host + p + cs * c->out_ld, c->out_ld * 8, c->m + p + cs * c->ld,
                             c->ld * 8, w * 8, ce - cs, cudaMemcpyDeviceToHost, c->st_out));
  return 0;
}

// SumOut pointing into the global-grid checksum arrays for a b-aligned region.
SumOut sums_for(abft_ctx* c, int64_t r0, int64_t c0, bool rows_too) {
  SumOut o;
  const int64_t gbi = r0 / c->b, gbj = c0 / c->b;
  o.cp = c->gcsw + 2 * gbi + c0 * c->ld_cs;
  o.cp_ld = c->ld_cs;
  o.cp_step = 2;
  o.cw = o.cp + 1;
  o.cw_ld = c->ld_cs;
  o.cw_step = 2;
  if (rows_too) {
    o.rp = c->grs + r0 + gbj * c->ld;
    o.rp_ld = c->ld;
  }
  o.bm = c->gmax + gbi + gbj * c->ld_max;
  o.bm_ld = c->ld_max;
  return o;
}

FusedSums fused_for(abft_ctx* c, int64_t r0, int64_t c0) {
  const SumOut o = sums_for(c, r0, c0, true);
  FusedSums f;
  f.cp = o.cp;
  f.cp_ld = o.cp_ld;
  f.cp_step = o.cp_step;
  f.cw = o.cw;
  f.cw_ld = o.cw_ld;
  f.cw_step = o.cw_step;
  f.rp = o.rp;
  f.rp_ld = o.rp_ld;
  f.bm = o.bm;
  f.bm_ld = o.bm_ld;
  f.rpp = c->fpart;
  f.rpp_ld = c->ld;
  f.bmp = c->fmaxp;
  f.bmp_ld = c->ld_max;
  return f;
}

int check_info(abft_ctx* c) {
  int h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, c->info, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  if (h != 0) {
    c->breakdown_col = h - 1;
    if (c->kind == ABFT_CHOLESKY)
      set_last_error("non-positive pivot at column %lld", (long long)c->breakdown_col);
    else
      set_last_error("zero pivot at column %lld", (long long)c->breakdown_col);
    CUDA_TRY(cudaMemsetAsync(c->info, 0, sizeof(int), c->st));
    return ABFT_E_BREAKDOWN;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// tasks (linalg.py:192-258)
// ---------------------------------------------------------------------------
// Cholesky FULL row checksums, maintained right-looking. chol_rs[r, j] holds,
// for every future panel j, the row sums over panel j's columns of the
// original matrix minus every rank-b update applied so far:
//   after panel k is final, chol_rs[pe:n, j] -= L_k[pe:n, :] * (1^T L_k[block j, :])^T
// for j > k. The reference maintains the same quantity from the operands at
// TMU(j) (maintain_gemm, abft.py:157 with R = L[p:pe, 0:p]^T); accumulating
// it panel by panel avoids re-reading all of L at every iteration.
int chol_rs_encode(abft_ctx* c) {
  Region all{c->m, c->ld, c->n, c->n, c->b};
  SumOut o;
  o.rp = c->chol_rs;
  o.rp_ld = c->ld;
  ABFT_TRY(blocksum(c->st, all, o));
  c->chol_rs_valid = true;
  return 0;
}

int chol_rs_update(abft_ctx* c, int64_t k) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  const int64_t nj = c->nb - (k + 1);
  if (nj <= 0 || pe >= n) return 0;
  // Bc (w x nj): Bc[kk, j] = plain col sum of L over block row (k+1+j), column p+kk
  ABFT_TRY(gather_transpose(c->st, c->gcsw + 2 * (k + 1) + p * c->ld_cs, 2, c->ld_cs, nj, w,
                            c->er, c->ld_t));
  return gemm(c->st, 'N', 'N', (int)(n - pe), (int)nj, (int)w, -1.0, c->m + pe + p * c->ld, c->ld,
              c->er, c->ld_t, 1.0, c->chol_rs + pe + (k + 1) * c->ld, c->ld,
              c->chol_rs + pe + (k + 1) * c->ld, c->ld, &c->gws);
}

// Streamed input: the stream waits until column block j has arrived.
int wait_in(abft_ctx* c, cudaStream_t st, int64_t j) {
  if (!c->in_stream || j < 0 || j >= c->nb) return 0;
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_in[j], 0));
  return 0;
}

// Streamed Cholesky FULL: chol_rs starts at zero and takes the panel updates
// as they come (chol_rs_update); block column j's own row sums are added once
// it has arrived, before anything modifies its rows >= j b (the look-ahead
// update of panel j on st2, else TMU(j)). Same quantity as chol_rs_encode +
// the updates, summed in another order.
int chol_rs_encode_col(abft_ctx* c, cudaStream_t st, int64_t j) {
  if (!c->in_stream || !c->chol_rs_valid || j >= c->nb || c->rs_enc[j]) return 0;
  const int64_t n = c->n, p = j * c->b, w = std::min(c->b, n - p);
  Region reg{c->m + p + p * c->ld, c->ld, n - p, w, c->b};
  SumOut o;
  o.rp = c->rs_tmp;
  o.rp_ld = c->ld;
  ABFT_TRY(blocksum(st, reg, o));
  ABFT_TRY(add_matrix(st, c->rs_tmp, c->ld, c->chol_rs + p + j * c->ld, c->ld, n - p, 1));
  c->rs_enc[j] = 1;
  return 0;
}

// LU panel, part 1: factor the diagonal block and form L11^{-1}, U11^{-1}.
int lu_diag(abft_ctx* c, cudaStream_t st, int64_t k, bool fast = false) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  if (fast)
    return diag_factor_fast(st, c->m + p + p * c->ld, c->ld, (int)w, 0, c->linv, c->ld_t, c->uinv,
                            c->ld_t, c->info, p);
  return diag_factor(st, c->m + p + p * c->ld, c->ld, (int)w, 0, c->linv, c->ld_t, c->uinv,
                     c->ld_t, c->info, p);
}

// LU panel, part 2: L21 = A21 U11^{-1} (GEMM over all SMs).
int lu_l21(abft_ctx* c, int64_t k) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  if (pe >= n) return 0;
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)(n - pe), (int)w, (int)w, 1.0, c->m + pe + p * c->ld, c->ld,
                c->uinv, c->ld_t, 0.0, nullptr, 0, c->lw, c->ld, &c->gws));
  return copy_matrix(c->st, c->lw, c->ld, c->m + pe + p * c->ld, c->ld, n - pe, w);
}

int task_pd(abft_ctx* c, int64_t k) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  double* D = c->m + p + p * c->ld;
  if (c->kind == ABFT_LU && c->pivot) {
    // partial pivoting (LAPACK dgetf2 on the tall panel), the interchanges on
    // every other column (dlaswp), L11^{-1} for PU; the region's rows moved:
    // its checksums are re-encoded by the protected update
    ABFT_TRY(lu_panel_pivot(c->st, D, c->ld, n - p, (int)w, c->ipiv + p, c->piv_part,
                            c->piv_part_elems, c->info, p));
    ABFT_TRY(laswp(c->st, c->m, c->ld, 0, p, p, (int)w, c->ipiv + p));
    ABFT_TRY(laswp(c->st, c->m, c->ld, pe, n - pe, p, (int)w, c->ipiv + p));
    ABFT_TRY(tri_inverse_lower(c->st, D, c->ld, (int)w, true, c->linv, c->ld_t, c->info));
    c->sums_valid = false;
  } else if (c->kind == ABFT_LU) {
    ABFT_TRY(lu_diag(c, c->st, k));
    ABFT_TRY(lu_l21(c, k));
  } else if (c->kind == ABFT_CHOLESKY) {
    const bool side_set = (int64_t)c->side_sms.size() > k && c->side_sms[k] > 0;
    if (side_set ? c->side_sms[k] >= (int)((c->b + 31) / 32) : c->chol_cluster)
      ABFT_TRY(diag_factor_fast(c->st, D, c->ld, (int)w, 1, c->linv, c->ld_t, nullptr, 0, c->info, p));
    else
      ABFT_TRY(diag_factor(c->st, D, c->ld, (int)w, 1, c->linv, c->ld_t, nullptr, 0, c->info, p));
  } else {
    double* V = c->vstore + p + p * c->ld;
    ABFT_TRY(qr_panel_factor(c->st, D, c->ld, n - p, (int)w, V, c->ld,
                             c->tstore + k * c->b * c->ld_t, c->ld_t, c->betas, c->qrw));
    c->qr_count = (int)(k + 1);
  }
  return 0;
}

int task_pu(abft_ctx* c, int64_t k) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  if (c->kind == ABFT_CHOLESKY) {
    if (pe < n) {
      // L21 = A21 L11^{-T}; zero the row block (linalg.py:251-252)
      ABFT_TRY(gemm(c->st, 'N', 'T', (int)(n - pe), (int)w, (int)w, 1.0, c->m + pe + p * c->ld,
                    c->ld, c->linv, c->ld_t, 0.0, nullptr, 0, c->lw, c->ld, &c->gws));
      ABFT_TRY(copy_matrix(c->st, c->lw, c->ld, c->m + pe + p * c->ld, c->ld, n - pe, w));
      ABFT_TRY(fill_matrix(c->st, c->m + p + pe * c->ld, c->ld, w, n - pe, 0.0));
    }
    // block-row checksums of the finished L panel (operand sums for later
    // left-looking maintenance)
    Region reg{c->m + p + p * c->ld, c->ld, n - p, w, c->b};
    SumOut o = sums_for(c, p, p, false);
    o.bm = nullptr;
    ABFT_TRY(blocksum(c->st, reg, o));
    if (c->chol_rs_valid) ABFT_TRY(chol_rs_update(c, k));
  } else if (c->kind == ABFT_LU) {
    if (pe < n) {
      ABFT_TRY(gemm(c->st, 'N', 'N', (int)w, (int)(n - pe), (int)w, 1.0, c->linv, c->ld_t,
                    c->m + p + pe * c->ld, c->ld, 0.0, nullptr, 0, c->uw, c->ld_t, &c->gws));
      ABFT_TRY(copy_matrix(c->st, c->uw, c->ld_t, c->m + p + pe * c->ld, c->ld, w, n - pe));
    }
  }
  return 0;
}

// The trailing-update GEMM(s) of iteration k. Returns in *L/*R the operands
// of `region -= L @ R` for checksum maintenance (simulator.py:135-157).
int tmu_gemm(abft_ctx* c, int64_t k, bool* did) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  *did = false;
  if (c->kind == ABFT_CHOLESKY) {
    if (k == 0) return 0;
    if (c->chol_part == k) {
      // the look-ahead already applied panels 0..k-2: only panel k-1 is left (K = b)
      const double* Lk = c->m + p + (p - c->b) * c->ld;
      ABFT_TRY(gemm(c->st, 'N', 'T', (int)(n - p), (int)w, (int)c->b, -1.0, Lk, c->ld, Lk, c->ld, 1.0,
                    c->m + p + p * c->ld, c->ld, c->m + p + p * c->ld, c->ld, &c->gws));
    } else {
      ABFT_TRY(gemm(c->st, 'N', 'T', (int)(n - p), (int)w, (int)p, -1.0, c->m + p, c->ld, c->m + p,
                    c->ld, 1.0, c->m + p + p * c->ld, c->ld, c->m + p + p * c->ld, c->ld, &c->gws));
    }
  } else if (c->kind == ABFT_LU) {
    if (pe >= n) return 0;
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)(n - pe), (int)(n - pe), (int)w, -1.0,
                  c->m + pe + p * c->ld, c->ld, c->m + p + pe * c->ld, c->ld, 1.0,
                  c->m + pe + pe * c->ld, c->ld, c->m + pe + pe * c->ld, c->ld, &c->gws));
  } else {
    if (pe >= n || k >= c->qr_count) return 0;
    const double* V = c->vstore + p + p * c->ld;
    const double* T = c->tstore + k * c->b * c->ld_t;
    double* C = c->m + p + pe * c->ld;
    ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)(n - pe), (int)(n - p), 1.0, V, c->ld, C, c->ld,
                  0.0, nullptr, 0, c->ww, c->ld_t, &c->gws));
    ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)(n - pe), (int)w, 1.0, T, c->ld_t, c->ww, c->ld_t,
                  0.0, nullptr, 0, c->mid, c->ld_t, &c->gws));
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)(n - p), (int)(n - pe), (int)w, -1.0, V, c->ld, c->mid,
                  c->ld_t, 1.0, C, c->ld, C, c->ld, &c->gws));
  }
  *did = true;
  return 0;
}

// maintain_gemm (abft.py:138-158) for the region of iteration k, from the
// operands of the update. QR needs `mid`, so it runs after the first two QR
// GEMMs (done inside tmu_gemm) -- callers order it accordingly.
int maintain(abft_ctx* c, int64_t k, int scheme, int64_t r0, int64_t c0, int64_t rows,
             int64_t cols) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  const int64_t nbr = (rows + c->b - 1) / c->b, nbc = (cols + c->b - 1) / c->b;
  SumOut enc = sums_for(c, r0, c0, scheme == ABFT_FULL);
  if (c->kind == ABFT_CHOLESKY) {
    // col: CSm = CS - GCSW[2k:, 0:p] * m[p:pe, 0:p]^T   (K = p; K = 0 copies)
    ABFT_TRY(gemm(c->st, 'N', 'T', (int)(2 * nbr), (int)w, (int)p, -1.0, c->gcsw + 2 * k, c->ld_cs,
                  c->m + p, c->ld, 1.0, enc.cp, c->ld_cs, c->csm, c->ld_cs, &c->gws));
    if (scheme == ABFT_FULL) {
      if (c->chol_rs_valid) {
        // running right-looking maintenance (see chol_rs_update): the panel's
        // row checksums already carry every earlier update
        ABFT_TRY(copy_matrix(c->st, c->chol_rs + p + k * c->ld, c->ld, c->rsm, c->ld, rows, nbc));
      } else {
        ABFT_TRY(copy_matrix(c->st, enc.rp, c->ld, c->rsm, c->ld, rows, nbc));
        // row: RSm -= L * rvec, rvec = block-row-k plain sums of L (= R e)
        ABFT_TRY(gemv_sub(c->st, rows, p, c->m + p, c->ld, c->gcsw + 2 * k, c->ld_cs, c->rsm));
      }
    }
    return 0;
  }
  const double* L;
  int64_t ldl;
  const double* R;
  int64_t ldr;
  if (c->kind == ABFT_LU) {
    L = c->m + pe + p * c->ld;
    ldl = c->ld;
    R = c->m + p + pe * c->ld;
    ldr = c->ld;
  } else {
    L = c->vstore + p + p * c->ld;
    ldl = c->ld;
    R = c->mid;
    ldr = c->ld_t;
  }
  // E_L: plain/weighted block-row sums of L (rows x w), interleaved in el
  {
    Region rl{const_cast<double*>(L), ldl, rows, w, c->b};
    SumOut o;
    o.cp = c->el;
    o.cp_ld = c->ld_cs;
    o.cp_step = 2;
    o.cw = c->el + 1;
    o.cw_ld = c->ld_cs;
    o.cw_step = 2;
    ABFT_TRY(blocksum(c->st, rl, o));
  }
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)(2 * nbr), (int)cols, (int)w, -1.0, c->el, c->ld_cs, R, ldr,
                1.0, enc.cp, c->ld_cs, c->csm, c->ld_cs, &c->gws));
  if (scheme == ABFT_FULL) {
    Region rr{const_cast<double*>(R), ldr, w, cols, c->b};
    SumOut o;
    o.rp = c->er;
    o.rp_ld = c->ld_t;
    ABFT_TRY(blocksum(c->st, rr, o));
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)nbc, (int)w, -1.0, L, ldl, c->er, c->ld_t, 1.0,
                  enc.rp, c->ld, c->rsm, c->ld, &c->gws));
  }
  return 0;
}

// Host-side list of region blocks touched by the planned faults.
void touched_blocks(const abft_ctx* c, const abft_fault* plan, int nplan, int64_t r0, int64_t c0,
                    int64_t rows, int64_t cols, std::vector<int32_t>* out) {
  std::vector<std::pair<int32_t, int32_t>> blks;
  for (int f = 0; f < nplan; ++f) {
    const abft_fault& ft = plan[f];
    int64_t er = 1, ec = 1;
    const int64_t ext = std::max<int64_t>(2, ft.extent);
    if (ft.kind == ABFT_D1) {
      if (ft.orientation == 0) er = ext; else ec = ext;
    } else if (ft.kind == ABFT_D2) {
      er = ext;
      ec = ext;
    }
    const int64_t rlo = std::max(ft.row, r0), rhi = std::min(std::min(ft.row + er, c->n), r0 + rows);
    const int64_t clo = std::max(ft.col, c0), chi = std::min(std::min(ft.col + ec, c->n), c0 + cols);
    for (int64_t r = rlo; r < rhi; ++r)
      for (int64_t cc = clo; cc < chi; ++cc)
        blks.emplace_back((int32_t)((r - r0) / c->b), (int32_t)((cc - c0) / c->b));
  }
  std::sort(blks.begin(), blks.end());
  blks.erase(std::unique(blks.begin(), blks.end()), blks.end());
  out->clear();
  for (auto& pr : blks) {
    out->push_back(pr.first);
    out->push_back(pr.second);
  }
}

int upload_plan(abft_ctx* c, const abft_fault* plan, int nplan) {
  if (nplan > c->dplan_cap) {
    if (c->dplan) cudaFree(c->dplan);
    c->dplan_cap = std::max(nplan, 64);
    CUDA_TRY(cudaMalloc(&c->dplan, c->dplan_cap * sizeof(DevFault)));
  }
  std::vector<DevFault> h(nplan);
  for (int i = 0; i < nplan; ++i) {
    h[i].kind = plan[i].kind;
    h[i].orientation = plan[i].orientation;
    h[i].row = plan[i].row;
    h[i].col = plan[i].col;
    h[i].extent = plan[i].extent;
    h[i].absolute = plan[i].absolute;
    h[i].u = plan[i].u;
    h[i].negate = plan[i].negate;
    h[i].pad = 0;
    h[i].magnitude = plan[i].magnitude;
  }
  CUDA_TRY(cudaMemcpyAsync(c->dplan, h.data(), nplan * sizeof(DevFault), cudaMemcpyHostToDevice,
                           c->st));
  // the host vector dies at return: make the copy complete first
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

int upload_list(abft_ctx* c, const std::vector<int32_t>& lst) {
  const int n = (int)lst.size();
  if (n == 0) return 0;
  if (n > c->dlist_cap) {
    if (c->dlist) cudaFree(c->dlist);
    c->dlist_cap = std::max(n, 1024);
    CUDA_TRY(cudaMalloc(&c->dlist, c->dlist_cap * sizeof(int32_t)));
  }
  CUDA_TRY(cudaMemcpyAsync(c->dlist, lst.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

// _protected_tmu (simulator.py:124-167). Events are appended on the device.
int protected_tmu(abft_ctx* c, int64_t k, int scheme, const abft_fault* plan, int nplan,
                  int correct) {
  int64_t r0, c0, rows, cols;
  region_of(c, k, &r0, &c0, &rows, &cols);
  const bool has_region = rows > 0 && cols > 0;
  const bool prot = scheme != ABFT_NONE && has_region;
  Region reg{c->m + r0 + c0 * c->ld, c->ld, rows, cols, c->b};
  const bool full = scheme == ABFT_FULL;
  // LU / QR trailing updates produce the verify sums in the GEMM epilogue
  // (b = 128 / 256); Cholesky's left-looking panel update keeps the pass.
  const bool fuse = prot && c->fuse_enabled && c->kind != ABFT_CHOLESKY && gemm_can_fuse((int)c->b);
  bool fused_done = false;
  if (c->kind == ABFT_CHOLESKY && k == 0 && (scheme == ABFT_FULL || c->want_chol_rs)) {
    prof_mark(c, PROF_ABFT, true);
    if (c->in_stream) {  // block columns add their row sums as they arrive
      CUDA_TRY(cudaMemsetAsync(c->chol_rs, 0, (size_t)c->ld * c->nb * sizeof(double), c->st));
      c->chol_rs_valid = true;
    } else {
      ABFT_TRY(chol_rs_encode(c));
    }
    prof_mark(c, PROF_ABFT, false);
  }
  if (c->kind == ABFT_CHOLESKY) ABFT_TRY(chol_rs_encode_col(c, c->st, k));
  if (prot) {
    // encode (abft.py:118-135): reuse the previous verify's sums when the
    // region is a sub-grid of the last verified region (LU/QR), else a pass
    prof_mark(c, PROF_ABFT, true);
    const bool reuse = (c->sums_valid && c->kind != ABFT_CHOLESKY) ||
                       (c->kind == ABFT_CHOLESKY && c->chol_part == k && c->chol_enc_ahead);
    if (!reuse) ABFT_TRY(blocksum(c->st, reg, sums_for(c, r0, c0, true)));
    if (c->kind != ABFT_QR) ABFT_TRY(maintain(c, k, scheme, r0, c0, rows, cols));
    prof_mark(c, PROF_ABFT, false);
  }
  bool did = false;
  if (prot && c->kind == ABFT_QR) {
    // QR: maintenance needs mid = T^T (V^T C), computed by the first GEMMs
    const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
    if (pe < n && k < c->qr_count) {
      const double* V = c->vstore + p + p * c->ld;
      const double* T = c->tstore + k * c->b * c->ld_t;
      double* C = c->m + p + pe * c->ld;
      prof_mark(c, PROF_TMU, true);
      ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)(n - pe), (int)(n - p), 1.0, V, c->ld, C, c->ld,
                    0.0, nullptr, 0, c->ww, c->ld_t, &c->gws));
      ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)(n - pe), (int)w, 1.0, T, c->ld_t, c->ww,
                    c->ld_t, 0.0, nullptr, 0, c->mid, c->ld_t, &c->gws));
      prof_mark(c, PROF_TMU, false);
      prof_mark(c, PROF_ABFT, true);
      ABFT_TRY(maintain(c, k, scheme, r0, c0, rows, cols));
      prof_mark(c, PROF_ABFT, false);
      prof_mark(c, PROF_TMU, true);
      if (fuse) {
        ABFT_TRY(gemm_fused_sums(c->st, 'N', 'N', (int)(n - p), (int)(n - pe), (int)w, -1.0, V,
                                 c->ld, c->mid, c->ld_t, 1.0, C, c->ld, C, c->ld, (int)c->b,
                                 fused_for(c, r0, c0)));
        fused_done = true;
      } else {
        ABFT_TRY(gemm(c->st, 'N', 'N', (int)(n - p), (int)(n - pe), (int)w, -1.0, V, c->ld,
                      c->mid, c->ld_t, 1.0, C, c->ld, C, c->ld, &c->gws));
      }
      prof_mark(c, PROF_TMU, false);
      did = true;
    } else {
      // no update: maintained == encoded
      SumOut enc = sums_for(c, r0, c0, true);
      const int64_t nbr = (rows + c->b - 1) / c->b, nbc = (cols + c->b - 1) / c->b;
      ABFT_TRY(copy_matrix(c->st, enc.cp, c->ld_cs, c->csm, c->ld_cs, 2 * nbr, cols));
      if (full) ABFT_TRY(copy_matrix(c->st, enc.rp, c->ld, c->rsm, c->ld, rows, nbc));
    }
  } else if (prot && fuse && c->kind == ABFT_LU) {
    // A22 -= L21 U12 with the verify-side block sums produced by the epilogue
    const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
    prof_mark(c, PROF_TMU, true);
    if (pe < n) {
      ABFT_TRY(gemm_fused_sums(c->st, 'N', 'N', (int)(n - pe), (int)(n - pe), (int)w, -1.0,
                               c->m + pe + p * c->ld, c->ld, c->m + p + pe * c->ld, c->ld, 1.0,
                               c->m + pe + pe * c->ld, c->ld, c->m + pe + pe * c->ld, c->ld,
                               (int)c->b, fused_for(c, r0, c0)));
      fused_done = true;
    }
    prof_mark(c, PROF_TMU, false);
  } else {
    prof_mark(c, PROF_TMU, true);
    ABFT_TRY(tmu_gemm(c, k, &did));
    prof_mark(c, PROF_TMU, false);
  }
  (void)did;
  prof_mark(c, PROF_ABFT, true);
  const bool faults = has_region && nplan > 0;
  if (prot && !fused_done) {
    // recomputed sums + block max of the updated region (verify's read)
    ABFT_TRY(blocksum(c->st, reg, sums_for(c, r0, c0, true)));
  } else if (!prot && faults) {
    SumOut o;
    o.bm = c->gmax + (r0 / c->b) + (c0 / c->b) * c->ld_max;
    o.bm_ld = c->ld_max;
    ABFT_TRY(blocksum(c->st, reg, o));
  }
  if (faults) {
    // sample_fault_plan magnitudes from scale = max|region| (simulator.py:159-163)
    for (int f = 0; f < nplan; ++f) {
      if (plan[f].row < 0 || plan[f].row >= c->n || plan[f].col < 0 || plan[f].col >= c->n) {
        set_last_error("fault at (%lld, %lld) outside matrix", (long long)plan[f].row,
                       (long long)plan[f].col);
        return ABFT_E_RANGE;
      }
    }
    ABFT_TRY(upload_plan(c, plan, nplan));
    const int64_t nbr = (rows + c->b - 1) / c->b, nbc = (cols + c->b - 1) / c->b;
    ABFT_TRY(inject(c->st, c->m, c->ld, c->n, c->n, c->dplan, nplan,
                    c->gmax + (r0 / c->b) + (c0 / c->b) * c->ld_max, nbr, nbc, c->ld_max, 0.0));
    if (prot) {
      std::vector<int32_t> lst;
      touched_blocks(c, plan, nplan, r0, c0, rows, cols, &lst);
      if (!lst.empty()) {
        ABFT_TRY(upload_list(c, lst));
        ABFT_TRY(blocksum(c->st, reg, sums_for(c, r0, c0, true), c->dlist, nullptr,
                          (int)(lst.size() / 2)));
      }
    }
  }
  if (prot) {
    Maintained mt;
    mt.cp = c->csm;
    mt.cp_ld = c->ld_cs;
    mt.cp_step = 2;
    mt.cw = c->csm + 1;
    mt.cw_ld = c->ld_cs;
    mt.cw_step = 2;
    mt.rp = c->rsm;
    mt.rp_ld = c->ld;
    EventSink sink{c->ev,    c->counters,     c->ev_cap,  c->dirty,
                   c->counters + 1, c->dirty_cap, c->cur_iter};
    ABFT_TRY(verify_blocks(c->st, reg, c->b, scheme, correct, sums_for(c, r0, c0, true), mt, sink));
    // refresh the sums of repaired blocks so they describe the current data
    ABFT_TRY(blocksum(c->st, reg, sums_for(c, r0, c0, true), c->dirty, c->counters + 1,
                      c->dirty_cap));
    ABFT_TRY(cudaMemsetAsync(c->counters + 1, 0, sizeof(int32_t), c->st) == cudaSuccess ? 0 : -1);
    c->sums_valid = true;
  } else {
    c->sums_valid = false;
  }
  prof_mark(c, PROF_ABFT, false);
  if (c->chol_part == k) {
    c->chol_part = -1;
    c->chol_enc_ahead = false;
  }
  if (c->kind == ABFT_QR) ABFT_TRY(emit_rowblock(c, k, 0, c->n));
  return 0;
}

// Cholesky look-ahead (left-looking, fast path): right after TMU(k), the
// update of panel k+1 by panels 0..k-1 -- final since their PU -- runs on the
// side stream on all SMs but one, while the one-CTA diagonal factorization
// PD(k) runs on the main stream; the panel-(k+1) encode goes with it. PU(k)
// waits for the side stream (it needs the whole GPU), TMU(k+1) then only
// applies panel k (K = b). Same operations as simulator.py:135-167, split.
// With chol_cluster the caller records ev_a (after TMU(k)), submits PD(k)
// -- the cluster diagonal factorization, ceil(b/32) SMs -- and only then this
// update, capped to leave those SMs: both become ready together and the
// cluster, first in submission order, is placed before the persistent GEMM
// fills the GPU.
int chol_lookahead(abft_ctx* c, int64_t k, int scheme_next, bool ev_recorded = false) {
  const int64_t n = c->n, pk = k * c->b, p1 = (k + 1) * c->b;
  const int64_t pe1 = std::min(p1 + c->b, n), w1 = pe1 - p1;
  if (!ev_recorded) CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
  ABFT_TRY(wait_in(c, c->st2, k + 1));
  ABFT_TRY(chol_rs_encode_col(c, c->st2, k + 1));
  c->chol_enc_ahead = false;
  if (scheme_next != ABFT_NONE) {
    Region reg1{c->m + p1 + p1 * c->ld, c->ld, n - p1, w1, c->b};
    ABFT_TRY(blocksum(c->st2, reg1, sums_for(c, p1, p1, true)));
    c->chol_enc_ahead = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  double* P1 = c->m + p1 + p1 * c->ld;
  int keep = c->chol_cluster ? (int)((c->b + 31) / 32) : 1;
  if ((int64_t)c->side_sms.size() > k && c->side_sms[k] > 0)
    keep = std::max(1, std::min((int)c->side_sms[k], sms / 2));
  prof_mark_side(c, true, (int32_t)(k + 1), PROF_TMU);
  ABFT_TRY(gemm_capped(c->st2, 'N', 'T', (int)(n - p1), (int)w1, (int)pk, -1.0, c->m + p1, c->ld,
                       c->m + p1, c->ld, 1.0, P1, c->ld, P1, c->ld, &c->gws2, sms - keep));
  prof_mark_side(c, false, (int32_t)(k + 1), PROF_TMU);
  CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  c->chol_part = k + 1;
  return 0;
}

// Verify (and refresh after repairs) the block columns [j0, j0 + ncb) of the
// region of iteration k — a block-aligned sub-region with its own event
// offsets, so the LU look-ahead can release the next panel early.
int verify_sub(abft_ctx* c, int scheme, int correct, int64_t r0, int64_t c0, int64_t rows,
               int64_t cols, int64_t j0, int64_t ncb) {
  const int64_t cbeg = j0 * c->b;
  const int64_t csub = std::min(cols - cbeg, ncb * c->b);
  if (csub <= 0 || rows <= 0) return 0;
  Region sub{c->m + r0 + (c0 + cbeg) * c->ld, c->ld, rows, csub, c->b};
  SumOut rec = sums_for(c, r0, c0 + cbeg, true);
  Maintained mt;
  mt.cp = c->csm + cbeg * c->ld_cs;
  mt.cp_ld = c->ld_cs;
  mt.cp_step = 2;
  mt.cw = mt.cp + 1;
  mt.cw_ld = c->ld_cs;
  mt.cw_step = 2;
  mt.rp = c->rsm + j0 * c->ld;
  mt.rp_ld = c->ld;
  EventSink sink{c->ev,          c->counters,    c->ev_cap,  c->dirty,
                 c->counters + 1, c->dirty_cap,  c->cur_iter, (int32_t)j0, c->b};
  ABFT_TRY(verify_blocks(c->st, sub, c->b, scheme, correct, rec, mt, sink));
  ABFT_TRY(blocksum(c->st, sub, rec, c->dirty, c->counters + 1, c->dirty_cap));
  CUDA_TRY(cudaMemsetAsync(c->counters + 1, 0, sizeof(int32_t), c->st));
  return 0;
}

// Diagonal-factor kernel of PD(k+1) under the LU look-ahead of iteration k
// (and the SMs kept from the update for it). A long update hides the
// one-CTA factor on 2 free SMs; once the update gets short (late iterations)
// the multi-CTA factor (b/32 SMs, ~2x faster) is worth the SMs it takes.
bool lu_la_fast_diag(const abft_ctx* c, int64_t k, int* keep_out) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  const int64_t rows = n - pe, cols = n - pe, wa = std::min<int64_t>(c->b, cols);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const double upd_s = 2.0 * (double)rows * (double)(cols - wa) * (double)w / (30.0e12 * (sms - 2) / 148.0);
  const int nbd = (int)((c->b + 31) / 32);
  bool fast_diag = c->lu_coop && upd_s < 1.0e-3;
  int keep = fast_diag ? nbd : 2;
  if ((int64_t)c->side_sms.size() > k + 1 && c->side_sms[k + 1] > 0) {
    keep = std::max(1, std::min((int)c->side_sms[k + 1], sms / 2));
    fast_diag = keep >= nbd;
  }
  if (keep_out) *keep_out = keep;
  return fast_diag;
}

// verify_sub restricted to block rows [i0, i0 + nrb) of the region.
int verify_rows(abft_ctx* c, int scheme, int correct, int64_t r0, int64_t c0, int64_t rows,
                int64_t cols, int64_t i0, int64_t nrb, int64_t j0, int64_t ncb) {
  const int64_t rbeg = i0 * c->b, cbeg = j0 * c->b;
  const int64_t rsub = std::min(rows - rbeg, nrb * c->b);
  const int64_t csub = std::min(cols - cbeg, ncb * c->b);
  if (csub <= 0 || rsub <= 0) return 0;
  Region sub{c->m + r0 + rbeg + (c0 + cbeg) * c->ld, c->ld, rsub, csub, c->b};
  SumOut rec = sums_for(c, r0 + rbeg, c0 + cbeg, true);
  Maintained mt;
  mt.cp = c->csm + 2 * i0 + cbeg * c->ld_cs;
  mt.cp_ld = c->ld_cs;
  mt.cp_step = 2;
  mt.cw = mt.cp + 1;
  mt.cw_ld = c->ld_cs;
  mt.cw_step = 2;
  mt.rp = c->rsm + rbeg + j0 * c->ld;
  mt.rp_ld = c->ld;
  EventSink sink{c->ev,          c->counters,    c->ev_cap,  c->dirty,
                 c->counters + 1, c->dirty_cap,  c->cur_iter, (int32_t)j0, c->b, (int32_t)i0};
  ABFT_TRY(verify_blocks(c->st, sub, c->b, scheme, correct, rec, mt, sink));
  ABFT_TRY(blocksum(c->st, sub, rec, c->dirty, c->counters + 1, c->dirty_cap));
  CUDA_TRY(cudaMemsetAsync(c->counters + 1, 0, sizeof(int32_t), c->st));
  return 0;
}

// LU protected trailing update with look-ahead (fault-free iterations of the
// one-call path): the next panel's block column is updated and verified
// first, then its diagonal block is factored on a side stream (2 SMs left
// free by the persistent GEMM) while the rest of the trailing matrix updates.
// Same operations and ordering constraints as _protected_tmu
// (simulator.py:124-167); only independent work overlaps.
int protected_tmu_lu_lookahead(abft_ctx* c, int64_t k, int scheme, int correct) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  region_of(c, k, &r0, &c0, &rows, &cols);
  Region reg{c->m + r0 + c0 * c->ld, c->ld, rows, cols, c->b};
  const bool prot = scheme != ABFT_NONE;
  if (prot) {
    prof_mark(c, PROF_ABFT, true);
    if (!c->sums_valid) ABFT_TRY(blocksum(c->st, reg, sums_for(c, r0, c0, true)));
    ABFT_TRY(maintain(c, k, scheme, r0, c0, rows, cols));
    prof_mark(c, PROF_ABFT, false);
  }
  const double* L21 = c->m + pe + p * c->ld;
  const double* U12 = c->m + p + pe * c->ld;
  double* A22 = c->m + pe + pe * c->ld;
  const int64_t wa = std::min<int64_t>(c->b, cols);
  // (a) next panel's block column, plain tiles over all SMs + checksum pass
  prof_mark(c, PROF_TMU, true);
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)wa, (int)w, -1.0, L21, c->ld, U12, c->ld, 1.0, A22,
                c->ld, A22, c->ld, &c->gws));
  prof_mark(c, PROF_TMU, false);
  if (prot) {
    prof_mark(c, PROF_ABFT, true);
    Region ra{A22, c->ld, rows, wa, c->b};
    ABFT_TRY(blocksum(c->st, ra, sums_for(c, r0, c0, true)));
    ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, 0, 1));
    prof_mark(c, PROF_ABFT, false);
  }
  // side stream: diagonal block of panel k+1 (lu_la_fast_diag)
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int keep = 2;
  const bool fast_diag = lu_la_fast_diag(c, k, &keep);
  const int64_t pe1 = std::min(pe + c->b, n), w1 = pe1 - pe;
  // depth 2 (lu_la2): the side stream also forms L21(k+1) and, once block row
  // k+1 is updated and verified, PU(k+1) -- both only read blocks the rest of
  // the update does not touch -- on SMs sized from the flop ratio
  const bool la2 = c->lu_la2 && cols > wa && rows > c->b && pe1 < n;
  if (la2) {
    const double side = 4.0 * (double)(n - pe1) * (double)w1 * (double)w1;
    const double upd = 2.0 * (double)(rows - c->b) * (double)(cols - wa) * (double)w;
    const int ks = (int)std::ceil((double)sms * side / (side + upd)) + 1;
    keep = std::max(keep, std::min(ks, sms / 2));
  }
  CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
  prof_mark_side(c, true, (int32_t)(k + 1));
  ABFT_TRY(lu_diag(c, c->st2, k + 1, fast_diag));
  if (la2) {
    // L21(k+1) = A21 U11^{-1} (lu_l21 on the side stream)
    ABFT_TRY(gemm_reserved(c->st2, 'N', 'N', (int)(n - pe1), (int)w1, (int)w1, 1.0,
                           c->m + pe1 + pe * c->ld, c->ld, c->uinv, c->ld_t, 0.0, nullptr, 0,
                           c->lw, c->ld, keep));
    ABFT_TRY(copy_matrix(c->st2, c->lw, c->ld, c->m + pe1 + pe * c->ld, c->ld, n - pe1, w1));
  }
  if (!la2) prof_mark_side(c, false, (int32_t)(k + 1));
  if (!la2) CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  auto rest = [&](int64_t rb, int64_t nr) -> int {  // rows [rb, rb + nr) x columns [wa, cols)
    const int64_t rr = std::min(rows - rb, nr);
    if (rr <= 0 || cols <= wa) return 0;
    prof_mark(c, PROF_TMU, true);
    if (prot) {
      FusedSums fs = fused_for(c, r0 + rb, c0 + wa);
      ABFT_TRY(gemm_fused_sums(c->st, 'N', 'N', (int)rr, (int)(cols - wa), (int)w, -1.0,
                               L21 + rb, c->ld, U12 + wa * c->ld, c->ld, 1.0,
                               A22 + rb + wa * c->ld, c->ld, A22 + rb + wa * c->ld, c->ld,
                               (int)c->b, fs, sms - keep));
    } else {
      ABFT_TRY(gemm_reserved(c->st, 'N', 'N', (int)rr, (int)(cols - wa), (int)w, -1.0, L21 + rb,
                             c->ld, U12 + wa * c->ld, c->ld, 1.0, A22 + rb + wa * c->ld, c->ld,
                             A22 + rb + wa * c->ld, c->ld, sms - keep));
    }
    prof_mark(c, PROF_TMU, false);
    if (prot) {
      prof_mark(c, PROF_ABFT, true);
      ABFT_TRY(verify_rows(c, scheme, correct, r0, c0, rows, cols, rb / c->b,
                           (rr + c->b - 1) / c->b, 1, (cols + c->b - 1) / c->b));
      prof_mark(c, PROF_ABFT, false);
    }
    return 0;
  };
  if (!la2) {
    // (b) the rest of the trailing matrix with fused checksums
    ABFT_TRY(rest(0, rows));
    c->sums_valid = prot;
    // join, then L21 of panel k+1 on the main stream
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
    prof_mark(c, PROF_PD, true);
    ABFT_TRY(lu_l21(c, k + 1));
    prof_mark(c, PROF_PD, false);
    ABFT_TRY(emit_column(c, k + 1));
    c->pd_ready = k + 1;
    return 0;
  }
  // (b1) block row k+1 of the rest, verified; then PU(k+1) on the side stream
  ABFT_TRY(rest(0, c->b));
  CUDA_TRY(cudaEventRecord(c->ev_r, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_r, 0));
  ABFT_TRY(gemm_reserved(c->st2, 'N', 'N', (int)w1, (int)(n - pe1), (int)w1, 1.0, c->linv, c->ld_t,
                         c->m + pe + pe1 * c->ld, c->ld, 0.0, nullptr, 0, c->uw, c->ld_t, keep));
  ABFT_TRY(copy_matrix(c->st2, c->uw, c->ld_t, c->m + pe + pe1 * c->ld, c->ld, w1, n - pe1));
  prof_mark_side(c, false, (int32_t)(k + 1));
  CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  // (b2) the rows below
  ABFT_TRY(rest(c->b, rows));
  c->sums_valid = prot;
  CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
  ABFT_TRY(emit_column(c, k + 1));
  ABFT_TRY(emit_rowblock(c, k + 1, 0, n));
  c->pd_ready = k + 1;
  c->pu_ready = k + 1;
  return 0;
}

// ---------------------------------------------------------------------------
// Streamed LU input. Right-looking LU touches every column in iteration 0, so
// the input cannot be consumed block column by block column in iteration
// order. Instead the left part [0, split b) is processed chunk by chunk as it
// arrives: a chunk first receives the updates of every earlier panel (PU(k)
// and the protected TMU(k) restricted to its columns, k in increasing order),
// then its own panels are factored with the updates restricted to it. Every
// block sees the same sequence of K = b updates, encodes, maintenances and
// verifies as in the iteration-ordered schedule (_protected_tmu,
// simulator.py:124-167, restricted to a block-column window -- checksums,
// maintenance and verify are per b x b block), so factor and reports are the
// same. The right part [split b, n) catches up once the whole input is in;
// iterations split.. then run the ordinary (look-ahead) schedule. Used only
// while no fault is planned before iteration `split` (a fault's magnitude
// depends on max|region| over all columns of that iteration).

// PU(k) restricted to columns [cs, ce): U12 = L11^{-1} A12 with the kept L11^{-1}.
int lu_pu_win(abft_ctx* c, int64_t k, int64_t cs, int64_t ce) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  cs = std::max(cs, pe);
  if (cs >= ce) return 0;
  const double* linv = c->linv_store + k * c->ld_t * c->b;
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)w, (int)(ce - cs), (int)w, 1.0, linv, c->ld_t,
                c->m + p + cs * c->ld, c->ld, 0.0, nullptr, 0, c->uw, c->ld_t, &c->gws));
  ABFT_TRY(copy_matrix(c->st, c->uw, c->ld_t, c->m + p + cs * c->ld, c->ld, w, ce - cs));
  return emit_rowblock(c, k, cs, ce);
}

// maintain() of LU iteration k for the region columns [cs, ce): writes the
// window's part of the region-local maintained sums (csm, rsm).
int lu_maintain_win(abft_ctx* c, int64_t k, int scheme, int64_t r0, int64_t c0, int64_t rows,
                    int64_t cs, int64_t ce) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  const int64_t cw = ce - cs, cbeg = cs - c0, j0 = cbeg / c->b;
  const int64_t nbr = (rows + c->b - 1) / c->b, nbw = (cw + c->b - 1) / c->b;
  SumOut enc = sums_for(c, r0, cs, scheme == ABFT_FULL);
  const double* L = c->m + pe + p * c->ld;
  const double* R = c->m + p + cs * c->ld;
  // E_L of panel k: one pass per panel, kept for every window of iteration k
  double* el = c->el_store + k * c->ld_cs * c->b;
  if (!c->el_ok[k]) {
    Region rl{const_cast<double*>(L), c->ld, rows, w, c->b};
    SumOut o;
    o.cp = el;
    o.cp_ld = c->ld_cs;
    o.cp_step = 2;
    o.cw = el + 1;
    o.cw_ld = c->ld_cs;
    o.cw_step = 2;
    ABFT_TRY(blocksum(c->st, rl, o));
    c->el_ok[k] = 1;
  }
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)(2 * nbr), (int)cw, (int)w, -1.0, el, c->ld_cs, R, c->ld,
                1.0, enc.cp, c->ld_cs, c->csm + cbeg * c->ld_cs, c->ld_cs, &c->gws));
  if (scheme == ABFT_FULL) {
    Region rr{const_cast<double*>(R), c->ld, w, cw, c->b};
    SumOut o;
    o.rp = c->er;
    o.rp_ld = c->ld_t;
    ABFT_TRY(blocksum(c->st, rr, o));
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)nbw, (int)w, -1.0, L, c->ld, c->er, c->ld_t,
                  1.0, enc.rp, c->ld, c->rsm + j0 * c->ld, c->ld, &c->gws));
  }
  return 0;
}

// Does the iteration-ordered schedule run iteration k (fault-free) with the
// LU look-ahead (run_iteration_device)?
bool lu_la_applies(const abft_ctx* c, int64_t k) {
  const int64_t pe = std::min((k + 1) * c->b, c->n);
  return c->lookahead_enabled && pe < c->n && c->fuse_enabled && gemm_can_fuse((int)c->b) &&
         !c->pivot;
}

// The protected TMU(k) of LU restricted to region columns [cs, ce). `encode`:
// the window's blocks were not verified by iteration k-1 (first update of the
// window, or an unprotected k-1), so their checksums come from a pass.
int lu_tmu_win(abft_ctx* c, int64_t k, int scheme, int correct, int64_t cs, int64_t ce,
               bool encode) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  region_of(c, k, &r0, &c0, &rows, &cols);
  cs = std::max(cs, c0);
  ce = std::min(ce, c0 + cols);
  if (cs >= ce || rows <= 0) return 0;
  const int64_t cw = ce - cs, j0 = (cs - c0) / c->b, ncb = (cw + c->b - 1) / c->b;
  const bool prot = scheme != ABFT_NONE;
  Region wreg{c->m + r0 + cs * c->ld, c->ld, rows, cw, c->b};
  const double* L21 = c->m + pe + p * c->ld;
  const double* U12 = c->m + p + cs * c->ld;
  double* A22 = c->m + r0 + cs * c->ld;
  if (prot) {
    prof_mark(c, PROF_ABFT, true);
    if (encode) ABFT_TRY(blocksum(c->st, wreg, sums_for(c, r0, cs, true)));
    ABFT_TRY(lu_maintain_win(c, k, scheme, r0, c0, rows, cs, ce));
    prof_mark(c, PROF_ABFT, false);
  }
  // the iteration-ordered schedule's kernels per block column: its look-ahead
  // (lu_la_applies) updates block column k+1 with the plain GEMM + a pass and
  // verifies it first, factors the diagonal block of panel k+1 on the side
  // stream (lu_la_fast_diag) beside the rest of the update, then L21
  const bool fuse = prot && c->fuse_enabled && gemm_can_fuse((int)c->b);
  const bool la = lu_la_applies(c, k) && cs == c0;
  if (!la) {
    prof_mark(c, PROF_TMU, true);
    if (fuse)
      ABFT_TRY(gemm_fused_sums(c->st, 'N', 'N', (int)rows, (int)cw, (int)w, -1.0, L21, c->ld, U12,
                               c->ld, 1.0, A22, c->ld, A22, c->ld, (int)c->b, fused_for(c, r0, cs)));
    else
      ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)cw, (int)w, -1.0, L21, c->ld, U12, c->ld,
                    1.0, A22, c->ld, A22, c->ld, &c->gws));
    prof_mark(c, PROF_TMU, false);
    if (prot) {
      prof_mark(c, PROF_ABFT, true);
      if (!fuse) ABFT_TRY(blocksum(c->st, wreg, sums_for(c, r0, cs, true)));
      ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, j0, ncb));
      prof_mark(c, PROF_ABFT, false);
    }
    return 0;
  }
  const int64_t wa = std::min<int64_t>(c->b, cw);
  prof_mark(c, PROF_TMU, true);
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)wa, (int)w, -1.0, L21, c->ld, U12, c->ld, 1.0,
                A22, c->ld, A22, c->ld, &c->gws));
  prof_mark(c, PROF_TMU, false);
  if (prot) {
    prof_mark(c, PROF_ABFT, true);
    Region ra{A22, c->ld, rows, wa, c->b};
    ABFT_TRY(blocksum(c->st, ra, sums_for(c, r0, cs, true)));
    ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, 0, 1));
    prof_mark(c, PROF_ABFT, false);
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int keep = 2;
  const bool fast_diag = lu_la_fast_diag(c, k, &keep);
  CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
  prof_mark_side(c, true, (int32_t)(k + 1));
  ABFT_TRY(lu_diag(c, c->st2, k + 1, fast_diag));
  prof_mark_side(c, false, (int32_t)(k + 1));
  CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  if (cw > wa) {
    prof_mark(c, PROF_TMU, true);
    if (prot)
      ABFT_TRY(gemm_fused_sums(c->st, 'N', 'N', (int)rows, (int)(cw - wa), (int)w, -1.0, L21,
                               c->ld, U12 + wa * c->ld, c->ld, 1.0, A22 + wa * c->ld, c->ld,
                               A22 + wa * c->ld, c->ld, (int)c->b, fused_for(c, r0, cs + wa),
                               sms - keep));
    else
      ABFT_TRY(gemm_reserved(c->st, 'N', 'N', (int)rows, (int)(cw - wa), (int)w, -1.0, L21,
                             c->ld, U12 + wa * c->ld, c->ld, 1.0, A22 + wa * c->ld, c->ld,
                             A22 + wa * c->ld, c->ld, sms - keep));
    prof_mark(c, PROF_TMU, false);
    if (prot) {
      prof_mark(c, PROF_ABFT, true);
      ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, 1, ncb - 1));
      prof_mark(c, PROF_ABFT, false);
    }
  }
  CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
  c->cur_iter = (int32_t)(k + 1);
  prof_mark(c, PROF_PD, true);
  ABFT_TRY(lu_l21(c, k + 1));
  prof_mark(c, PROF_PD, false);
  ABFT_TRY(emit_column(c, k + 1));
  c->pd_ready = k + 1;
  return 0;
}

// Block columns of the streamed LU / QR left part (0: not used for this call).
int qr_panel_sms(const abft_ctx* c, int64_t k, int sms);

// Does the iteration-ordered schedule run QR iteration k (fault-free) with
// the QR look-ahead (run_iteration_device)?
bool qr_la_applies(const abft_ctx* c, int64_t k) {
  const int64_t pe = std::min((k + 1) * c->b, c->n);
  return c->lookahead_enabled && pe < c->n && c->qr_la_sms > 0;
}

// The protected TMU(k) of QR restricted to region columns [cs, ce):
// W = V^T C (with the full product's split-K partition), mid = T^T W,
// maintenance from mid, C -= V mid with the look-ahead's kernels mirrored
// (protected_tmu_qr_lookahead) when the window holds block column k+1.
int qr_tmu_win(abft_ctx* c, int64_t k, int scheme, int correct, int64_t cs, int64_t ce,
               bool encode) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  region_of(c, k, &r0, &c0, &rows, &cols);
  cs = std::max(cs, c0);
  ce = std::min(ce, c0 + cols);
  if (cs >= ce || rows <= 0) return 0;
  const int64_t cw = ce - cs, cbeg = cs - c0, j0 = cbeg / c->b, ncb = (cw + c->b - 1) / c->b;
  const bool prot = scheme != ABFT_NONE;
  Region wreg{c->m + r0 + cs * c->ld, c->ld, rows, cw, c->b};
  const double* V = c->vstore + p + p * c->ld;
  const double* T = c->tstore + k * c->b * c->ld_t;
  double* C = c->m + p + cs * c->ld;
  if (prot && encode) {
    prof_mark(c, PROF_ABFT, true);
    ABFT_TRY(blocksum(c->st, wreg, sums_for(c, r0, cs, true)));
    prof_mark(c, PROF_ABFT, false);
  }
  prof_mark(c, PROF_TMU, true);
  const int spl = gemm_effective_splits((int)w, (int)cols, (int)rows, &c->gws);
  ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)cw, (int)rows, 1.0, V, c->ld, C, c->ld, 0.0,
                nullptr, 0, c->ww, c->ld_t, &c->gws, spl));
  const int spl2 = gemm_effective_splits((int)w, (int)cols, (int)w, &c->gws);
  ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)cw, (int)w, 1.0, T, c->ld_t, c->ww, c->ld_t, 0.0,
                nullptr, 0, c->mid, c->ld_t, &c->gws, spl2));
  prof_mark(c, PROF_TMU, false);
  if (prot) {
    // maintain() for the window: E_L of V kept per panel, R = mid
    prof_mark(c, PROF_ABFT, true);
    const int64_t nbr = (rows + c->b - 1) / c->b;
    SumOut enc = sums_for(c, r0, cs, scheme == ABFT_FULL);
    double* el = c->el_store + k * c->ld_cs * c->b;
    if (!c->el_ok[k]) {
      Region rl{const_cast<double*>(V), c->ld, rows, w, c->b};
      SumOut o;
      o.cp = el;
      o.cp_ld = c->ld_cs;
      o.cp_step = 2;
      o.cw = el + 1;
      o.cw_ld = c->ld_cs;
      o.cw_step = 2;
      ABFT_TRY(blocksum(c->st, rl, o));
      c->el_ok[k] = 1;
    }
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)(2 * nbr), (int)cw, (int)w, -1.0, el, c->ld_cs, c->mid,
                  c->ld_t, 1.0, enc.cp, c->ld_cs, c->csm + cbeg * c->ld_cs, c->ld_cs, &c->gws,
                  gemm_effective_splits((int)(2 * nbr), (int)cols, (int)w, &c->gws)));
    if (scheme == ABFT_FULL) {
      Region rr{c->mid, c->ld_t, w, cw, c->b};
      SumOut o;
      o.rp = c->er;
      o.rp_ld = c->ld_t;
      ABFT_TRY(blocksum(c->st, rr, o));
      ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)ncb, (int)w, -1.0, V, c->ld, c->er, c->ld_t,
                    1.0, enc.rp, c->ld, c->rsm + j0 * c->ld, c->ld, &c->gws,
                    gemm_effective_splits((int)rows, (int)((cols + c->b - 1) / c->b), (int)w,
                                          &c->gws)));
    }
    prof_mark(c, PROF_ABFT, false);
  }
  const bool fuse = prot && c->fuse_enabled && gemm_can_fuse((int)c->b);
  if (!(qr_la_applies(c, k) && cs == c0)) {
    prof_mark(c, PROF_TMU, true);
    if (fuse)
      ABFT_TRY(gemm_fused_sums(c->st, 'N', 'N', (int)rows, (int)cw, (int)w, -1.0, V, c->ld,
                               c->mid, c->ld_t, 1.0, C, c->ld, C, c->ld, (int)c->b,
                               fused_for(c, r0, cs)));
    else
      ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)cw, (int)w, -1.0, V, c->ld, c->mid, c->ld_t,
                    1.0, C, c->ld, C, c->ld, &c->gws));
    prof_mark(c, PROF_TMU, false);
    if (prot) {
      prof_mark(c, PROF_ABFT, true);
      if (!fuse) ABFT_TRY(blocksum(c->st, wreg, sums_for(c, r0, cs, true)));
      ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, j0, ncb));
      prof_mark(c, PROF_ABFT, false);
    }
    return emit_rowblock(c, k, cs, ce);
  }
  const int64_t wa = std::min<int64_t>(c->b, cw);
  prof_mark(c, PROF_TMU, true);
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)wa, (int)w, -1.0, V, c->ld, c->mid, c->ld_t, 1.0,
                C, c->ld, C, c->ld, &c->gws));
  prof_mark(c, PROF_TMU, false);
  if (prot) {
    prof_mark(c, PROF_ABFT, true);
    Region ra{C, c->ld, rows, wa, c->b};
    ABFT_TRY(blocksum(c->st, ra, sums_for(c, r0, cs, true)));
    ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, 0, 1));
    prof_mark(c, PROF_ABFT, false);
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int res = qr_panel_sms(c, k, sms);
  CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
  {
    const int64_t p1 = pe, pe1 = std::min(p1 + c->b, n), w1 = pe1 - p1;
    QrPanelWork q = c->qrw;
    q.gws = &c->gws2;
    prof_mark_side(c, true, (int32_t)(k + 1));
    ABFT_TRY(qr_panel_factor(c->st2, c->m + p1 + p1 * c->ld, c->ld, n - p1, (int)w1,
                             c->vstore + p1 + p1 * c->ld, c->ld,
                             c->tstore + (k + 1) * c->b * c->ld_t, c->ld_t, c->betas, q, res));
    prof_mark_side(c, false, (int32_t)(k + 1));
  }
  CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  if (cw > wa) {
    prof_mark(c, PROF_TMU, true);
    const double* midb = c->mid + wa * c->ld_t;
    double* Cb = C + wa * c->ld;
    if (fuse) {
      ABFT_TRY(gemm_fused_sums(c->st, 'N', 'N', (int)rows, (int)(cw - wa), (int)w, -1.0, V, c->ld,
                               midb, c->ld_t, 1.0, Cb, c->ld, Cb, c->ld, (int)c->b,
                               fused_for(c, r0, cs + wa), sms - res));
      prof_mark(c, PROF_TMU, false);
    } else {
      ABFT_TRY(gemm_reserved(c->st, 'N', 'N', (int)rows, (int)(cw - wa), (int)w, -1.0, V, c->ld,
                             midb, c->ld_t, 1.0, Cb, c->ld, Cb, c->ld, sms - res));
      prof_mark(c, PROF_TMU, false);
      if (prot) {
        Region rb{Cb, c->ld, rows, cw - wa, c->b};
        ABFT_TRY(blocksum(c->st, rb, sums_for(c, r0, cs + wa, true)));
      }
    }
    if (prot) {
      prof_mark(c, PROF_ABFT, true);
      ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, 1, ncb - 1));
      prof_mark(c, PROF_ABFT, false);
    }
  }
  ABFT_TRY(emit_rowblock(c, k, cs, ce));
  CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
  c->qr_count = (int)(k + 2);
  ABFT_TRY(emit_column(c, k + 1));
  c->pd_ready = k + 1;
  return 0;
}

// Defaults measured on dgetrf N = 32768 b = 256 (nb = 128; e2e ms, H2D of
// 8.6 GB at ~50 GB/s): wait-for-all 1022, chunk 16 / split 48 902, split 32
// 946, split 64 914, chunk 8 906, chunk 32 922 (profiles/lu_stream_r02.txt).
// QR (same windows, qr_tmu_win; bit-identical too) keeps the chunked part
// short: each in-chunk panel runs beside only a window's update on the SMs
// the look-ahead's model leaves it, so the panels serialise. dgeqrf N = 32768
// e2e: wait-for-all 1748 ms; split 32 / 48 / 64 (chunk 16) 1923 / 2058 /
// 2168 ms; split 3 with 1-block chunks and the right part in nb/8 pieces as
// it arrives 1653 ms (split 1 / 2 / 4 / 6 / 8: 1713 / 1684 / 1669 / 1723 /
// 1777; profiles/lu_stream_r02.txt).
int lu_stream_chunk(const abft_ctx* c) {
  if (c->lu_chunk >= 0) return c->lu_chunk;
  return c->kind == ABFT_LU ? (int)std::max<int64_t>(1, c->nb / 8) : 1;
}

int64_t lu_stream_split(const abft_ctx* c) {
  if (c->kind == ABFT_CHOLESKY || c->pivot || lu_stream_chunk(c) <= 0 || c->nb < 4) return 0;
  int64_t s = c->lu_split >= 0 ? c->lu_split : (c->kind == ABFT_LU ? 3 * c->nb / 8 : 3);
  return std::max<int64_t>(1, std::min(s, c->nb - 1));
}

int64_t lu_stream_rchunk(const abft_ctx* c) {
  if (c->lu_rchunk > 0) return c->lu_rchunk;
  if (c->lu_rchunk == 0 || c->kind == ABFT_LU) return c->nb;
  return std::max<int64_t>(1, c->nb / 8);
}

// Iterations 0..split-1 of a streamed LU (see above); returns with the
// matrix in the state of the iteration-ordered schedule after TMU(split-1).
int lu_stream_chunks(abft_ctx* c, int64_t split, int scheme, const int32_t* schemes, int correct) {
  const int64_t b = c->b, n = c->n;
  auto sch = [&](int64_t k) { return schemes ? schemes[k] : scheme; };
  if (c->kind == ABFT_LU && !c->linv_store) ABFT_TRY(dalloc(&c->linv_store, c->ld_t * b * c->nb));
  if (!c->el_store) ABFT_TRY(dalloc(&c->el_store, c->ld_cs * b * c->nb));
  c->el_ok.assign(c->nb, 0);
  c->pd_ready = -1;
  c->pu_ready = -1;
  const bool lu = c->kind == ABFT_LU;
  auto run = [&](int64_t k, int64_t cs, int64_t ce) -> int {
    c->cur_iter = (int32_t)k;
    const bool enc = k == 0 || sch(k - 1) == ABFT_NONE;
    if (!lu) return qr_tmu_win(c, k, sch(k), correct, cs, ce, enc);
    prof_mark(c, PROF_PU, true);
    ABFT_TRY(lu_pu_win(c, k, cs, ce));
    prof_mark(c, PROF_PU, false);
    return lu_tmu_win(c, k, sch(k), correct, cs, ce, enc);
  };
  // the first chunk is a quarter of the others: the GPU starts early
  const int64_t chunk = lu_stream_chunk(c), first = std::max<int64_t>(1, chunk / 4);
  for (int64_t q0 = 0, q1 = 0; q0 < split; q0 = q1) {
    q1 = std::min<int64_t>(q0 + (q0 == 0 ? first : chunk), split);
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_in[q1 - 1], 0));
    for (int64_t k = 0; k < q1; ++k) {
      if (k >= q0) {
        c->cur_iter = (int32_t)k;
        if (c->pd_ready != k) {  // else formed by the look-ahead of TMU(k-1)
          prof_mark(c, PROF_PD, true);
          ABFT_TRY(task_pd(c, k));
          prof_mark(c, PROF_PD, false);
          ABFT_TRY(emit_column(c, k));
        }
        c->pd_ready = -1;
        if (lu)
          ABFT_TRY(copy_matrix(c->st, c->linv, c->ld_t, c->linv_store + k * c->ld_t * b, c->ld_t,
                               b, b));
      }
      ABFT_TRY(run(k, q0 * b, q1 * b));
    }
  }
  // the right part: every earlier panel's update, chunk by chunk as it arrives
  const int64_t rch = lu_stream_rchunk(c);
  for (int64_t q0 = split; q0 < c->nb; q0 += rch) {
    const int64_t q1 = std::min<int64_t>(q0 + rch, c->nb);
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_in[q1 - 1], 0));
    for (int64_t k = 0; k < split; ++k) ABFT_TRY(run(k, q0 * b, std::min(q1 * b, n)));
  }
  c->sums_valid = sch(split - 1) != ABFT_NONE;
  // pd_ready == split when the look-ahead of TMU(split-1) formed PD(split)
  return 0;
}

// SMs for the look-ahead's side-stream QR panel of iteration k (the B200
// form of the reference's slack reclamation, scheduler.py:84-146: the stream
// with slack gets fewer resources). A per-iteration model at the measured
// per-SM DMMA rate: panel(R) = four tall GEMM passes (8 m b^2 flops) on R
// SMs + the latency of its small factorizations; update(R) = C -= V mid on
// the other SMs; R minimises max(panel, update). ABFT_QR_LA_SMS > 0 fixes R.
int qr_panel_sms(const abft_ctx* c, int64_t k, int sms) {
  if ((int64_t)c->side_sms.size() > k + 1 && c->side_sms[k + 1] > 0)
    return std::max(1, std::min((int)c->side_sms[k + 1], sms / 2));
  if (c->qr_la_sms_fixed) return std::max(1, std::min(c->qr_la_sms, sms / 2));
  const double rate = 30.0e12 / 148.0;  // fused trailing-update rate per SM (bench_lu32k_r02)
  static const double lat = [] {        // three multi-CTA diagonal factors + small GEMMs
    const char* e = getenv("ABFT_QR_LA_LAT_US");  // A/B knob
    return (e ? atof(e) : 800.0) * 1e-6;
  }();
  const double n = (double)c->n, b = (double)c->b, p = (double)(k * c->b);
  const double m1 = n - p - b;          // rows of panel k+1
  const double cols = n - p - 2 * b;    // columns left to part (b) of the update
  int best = 16;
  double best_t = 1e30;
  for (int R = 8; R <= 48 && R < sms / 2; R += 4) {
    const double tp = 8.0 * m1 * b * b / (R * rate) + lat;
    const double tu = cols > 0 ? 2.0 * (n - p) * cols * b / ((sms - R) * rate) : 0.0;
    const double t = std::max(tp, tu);
    if (t < 0.995 * best_t) {
      best_t = t;
      best = R;
    }
  }
  return best;
}

// QR protected trailing update with look-ahead (fault-free iterations of the
// one-call path), the LU scheme restated for Householder updates: W = V^T C
// and mid = T^T W over the whole region and the maintained sums first; then
// the next panel's block column C[:, 0:b] -= V mid[:, 0:b] (plain GEMM over
// all SMs) + checksum pass + verify; panel k+1 (qr_panel_factor, every GEMM
// capped at qr_la_sms CTAs) is then factored on the side stream while the
// rest of the region takes C -= V mid with fused sums on the other SMs.
// Same operations and ordering constraints as _protected_tmu
// (simulator.py:124-167) and PD(k+1) (linalg.py:260-300); only independent
// work overlaps.
int protected_tmu_qr_lookahead(abft_ctx* c, int64_t k, int scheme, int correct) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  region_of(c, k, &r0, &c0, &rows, &cols);
  Region reg{c->m + r0 + c0 * c->ld, c->ld, rows, cols, c->b};
  const bool prot = scheme != ABFT_NONE;
  const double* V = c->vstore + p + p * c->ld;
  const double* T = c->tstore + k * c->b * c->ld_t;
  double* C = c->m + p + pe * c->ld;
  if (prot && !c->sums_valid) {
    prof_mark(c, PROF_ABFT, true);
    ABFT_TRY(blocksum(c->st, reg, sums_for(c, r0, c0, true)));
    prof_mark(c, PROF_ABFT, false);
  }
  prof_mark(c, PROF_TMU, true);
  ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)cols, (int)rows, 1.0, V, c->ld, C, c->ld, 0.0,
                nullptr, 0, c->ww, c->ld_t, &c->gws));
  ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)cols, (int)w, 1.0, T, c->ld_t, c->ww, c->ld_t, 0.0,
                nullptr, 0, c->mid, c->ld_t, &c->gws));
  prof_mark(c, PROF_TMU, false);
  if (prot) {
    prof_mark(c, PROF_ABFT, true);
    ABFT_TRY(maintain(c, k, scheme, r0, c0, rows, cols));
    prof_mark(c, PROF_ABFT, false);
  }
  const int64_t wa = std::min<int64_t>(c->b, cols);
  // (a) the next panel's block column
  prof_mark(c, PROF_TMU, true);
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)wa, (int)w, -1.0, V, c->ld, c->mid, c->ld_t, 1.0,
                C, c->ld, C, c->ld, &c->gws));
  prof_mark(c, PROF_TMU, false);
  if (prot) {
    prof_mark(c, PROF_ABFT, true);
    Region ra{C, c->ld, rows, wa, c->b};
    ABFT_TRY(blocksum(c->st, ra, sums_for(c, r0, c0, true)));
    ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, 0, 1));
    prof_mark(c, PROF_ABFT, false);
  }
  // side stream: panel k+1 on qr_la_sms SMs
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int res = qr_panel_sms(c, k, sms);
  CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
  {
    const int64_t p1 = pe, pe1 = std::min(p1 + c->b, n), w1 = pe1 - p1;
    QrPanelWork q = c->qrw;
    q.gws = &c->gws2;
    prof_mark_side(c, true, (int32_t)(k + 1));
    ABFT_TRY(qr_panel_factor(c->st2, c->m + p1 + p1 * c->ld, c->ld, n - p1, (int)w1,
                             c->vstore + p1 + p1 * c->ld, c->ld,
                             c->tstore + (k + 1) * c->b * c->ld_t, c->ld_t, c->betas, q, res));
    prof_mark_side(c, false, (int32_t)(k + 1));
  }
  CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  // (b) the rest of the region
  if (cols > wa) {
    prof_mark(c, PROF_TMU, true);
    const double* midb = c->mid + wa * c->ld_t;
    double* Cb = C + wa * c->ld;
    if (prot && c->fuse_enabled && gemm_can_fuse((int)c->b)) {
      ABFT_TRY(gemm_fused_sums(c->st, 'N', 'N', (int)rows, (int)(cols - wa), (int)w, -1.0, V,
                               c->ld, midb, c->ld_t, 1.0, Cb, c->ld, Cb, c->ld, (int)c->b,
                               fused_for(c, r0, c0 + wa), sms - res));
      prof_mark(c, PROF_TMU, false);
    } else {
      ABFT_TRY(gemm_reserved(c->st, 'N', 'N', (int)rows, (int)(cols - wa), (int)w, -1.0, V, c->ld,
                             midb, c->ld_t, 1.0, Cb, c->ld, Cb, c->ld, sms - res));
      prof_mark(c, PROF_TMU, false);
      if (prot) {
        Region rb{Cb, c->ld, rows, cols - wa, c->b};
        ABFT_TRY(blocksum(c->st, rb, sums_for(c, r0, c0 + wa, true)));
      }
    }
    if (prot) {
      prof_mark(c, PROF_ABFT, true);
      ABFT_TRY(verify_sub(c, scheme, correct, r0, c0, rows, cols, 1, (cols + c->b - 1) / c->b));
      prof_mark(c, PROF_ABFT, false);
    }
  }
  c->sums_valid = prot;
  ABFT_TRY(emit_rowblock(c, k, 0, n));
  CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
  c->qr_count = (int)(k + 2);
  ABFT_TRY(emit_column(c, k + 1));
  c->pd_ready = k + 1;
  return 0;
}

// Per-task device timers (CUDA events on the context stream), enabled by
// abft_profile(ctx, 1): PD, PU, TMU GEMM(s) and the ABFT work around them.

// One iteration in the reference's task order. `sync_checks`: read the
// breakdown flag right after PD (per-iteration API); otherwise it is checked
// once at the end of abft_factorize.
int run_iteration_device(abft_ctx* c, int64_t k, int scheme, const abft_fault* plan, int nplan,
                         int correct, bool sync_checks, bool lookahead = false) {
  auto pd = [&]() -> int {
    if (c->pd_ready == k) {  // produced by the previous iteration's look-ahead
      c->pd_ready = -1;
      return 0;
    }
    prof_mark(c, PROF_PD, true);
    ABFT_TRY(task_pd(c, k));
    prof_mark(c, PROF_PD, false);
    if (sync_checks) ABFT_TRY(check_info(c));
    if (c->kind != ABFT_CHOLESKY) ABFT_TRY(emit_column(c, k));
    return 0;
  };
  auto pu = [&]() -> int {
    if (c->pu_ready == k) {  // applied by the previous iteration's look-ahead
      c->pu_ready = -1;
      return 0;
    }
    prof_mark(c, PROF_PU, true);
    ABFT_TRY(task_pu(c, k));
    prof_mark(c, PROF_PU, false);
    if (c->kind == ABFT_CHOLESKY) ABFT_TRY(emit_column(c, k));
    ABFT_TRY(emit_rowblock(c, k, 0, c->n));
    return 0;
  };
  if (c->kind == ABFT_CHOLESKY) {
    ABFT_TRY(wait_in(c, c->st, k));
    ABFT_TRY(protected_tmu(c, k, scheme, plan, nplan, correct));
    const bool la = lookahead && c->lookahead_enabled && k >= 1 && k + 1 < c->nb;
    const bool side_set = (int64_t)c->side_sms.size() > k && c->side_sms[k] > 0;
    const bool fast_pd = side_set ? c->side_sms[k] >= (int)((c->b + 31) / 32) : c->chol_cluster;
    if (la && fast_pd) {
      CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
      ABFT_TRY(pd());
      ABFT_TRY(chol_lookahead(c, k, c->next_scheme, true));
    } else {
      if (la) ABFT_TRY(chol_lookahead(c, k, c->next_scheme));
      ABFT_TRY(pd());
    }
    if (la) CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
    ABFT_TRY(pu());
  } else if (c->kind == ABFT_LU) {
    ABFT_TRY(pd());
    ABFT_TRY(pu());
    const int64_t pe = std::min((k + 1) * c->b, c->n);
    const bool la = lookahead && nplan == 0 && pe < c->n && c->fuse_enabled &&
                    gemm_can_fuse((int)c->b) && !c->pivot;
    if (la)
      ABFT_TRY(protected_tmu_lu_lookahead(c, k, scheme, correct));
    else
      ABFT_TRY(protected_tmu(c, k, scheme, plan, nplan, correct));
  } else {
    ABFT_TRY(pd());
    const int64_t pe = std::min((k + 1) * c->b, c->n);
    const bool la = lookahead && c->lookahead_enabled && nplan == 0 && pe < c->n &&
                    k < c->qr_count && c->qr_la_sms > 0;
    if (la)
      ABFT_TRY(protected_tmu_qr_lookahead(c, k, scheme, correct));
    else
      ABFT_TRY(protected_tmu(c, k, scheme, plan, nplan, correct));
  }
  return 0;
}

// Pull device events, translate to reference locations, order like the
// reference (block row, block col, column), fill the report.
int collect_events(abft_ctx* c, const std::vector<int64_t>& r0s, const std::vector<int64_t>& c0s,
                   const std::vector<int32_t>* iter_of_event, abft_report* rep, abft_location* locs,
                   int max_locs, std::vector<Event>* raw_out) {
  int32_t cnt[2];
  CUDA_TRY(cudaMemcpyAsync(cnt, c->counters, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  if (cnt[0] > c->ev_cap) {
    set_last_error("ABFT event buffer overflow (%d events)", cnt[0]);
    return ABFT_E_OVERFLOW;
  }
  std::vector<Event> evs(cnt[0]);
  if (cnt[0] > 0)
    CUDA_TRY(cudaMemcpy(evs.data(), c->ev, cnt[0] * sizeof(Event), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemsetAsync(c->counters, 0, 2 * sizeof(int32_t), c->st));
  (void)iter_of_event;
  if (raw_out) *raw_out = evs;
  std::sort(evs.begin(), evs.end(), [](const Event& a, const Event& b) {
    if (a.bi != b.bi) return a.bi < b.bi;
    if (a.bj != b.bj) return a.bj < b.bj;
    return a.seq < b.seq;
  });
  if (rep) {
    memset(rep, 0, sizeof(*rep));
    rep->n_locations = (int32_t)evs.size();
  }
  for (size_t i = 0; i < evs.size(); ++i) {
    const Event& e = evs[i];
    if (e.kind < 0) {
      set_last_error("index 0 is out of bounds for axis 0 with size 0");
      return ABFT_E_RANGE;
    }
    if (rep) {
      rep->detected[e.detected_kind] += 1;
      if (e.corrected) rep->corrected[e.detected_kind] += 1;
      if (e.uncorrectable) rep->uncorrectable = 1;
    }
    if (locs && (int)i < max_locs) {
      abft_location& L = locs[i];
      L.row = e.row + (r0s.empty() ? 0 : r0s[0]);
      L.col = e.col + (c0s.empty() ? 0 : c0s[0]);
      L.kind = e.kind;
      L.flag = e.flag;
      L.detected_kind = e.detected_kind;
      L.corrected = e.corrected;
      L.uncorrectable = e.uncorrectable;
      L.block_row = e.bi;
      L.block_col = e.bj;
      L.seq = e.seq;
    }
  }
  return 0;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

// A streamed input not yet consumed by abft_factorize: entries that touch
// the matrix otherwise copy it now (the whole matrix, synchronously).
static int flush_pending_input(abft_ctx* c) {
  if (!c->in_host) return 0;
  const double* a = c->in_host;
  c->in_host = nullptr;
  CUDA_TRY(cudaMemcpy2DAsync(c->m, c->ld * 8, a, c->in_ld * 8, c->n * 8, c->n,
                             cudaMemcpyHostToDevice, c->st));
  return 0;
}

ABFT_API int abft_create(abft_ctx** out, int kind, int64_t n, int64_t b, int device) {
  *out = nullptr;
  if (kind < 0 || kind > 2) {
    set_last_error("unknown decomposition kind %d", kind);
    return ABFT_E_INVALID;
  }
  if (n < 1) {
    set_last_error("matrix order must be >= 1");
    return ABFT_E_DIM;
  }
  if (!(1 <= b && b <= n)) {
    set_last_error("block size %lld outside [1, %lld]", (long long)b, (long long)n);
    return ABFT_E_DIM;
  }
  if (b > 256) {
    set_last_error("block size %lld > 256 is not supported by the B200 panel kernels",
                   (long long)b);
    return ABFT_E_INVALID;
  }
  if (n > INT32_MAX / 2) {
    set_last_error("matrix order too large");
    return ABFT_E_INVALID;
  }
  DevGuard g(device);
  abft_ctx* c = new abft_ctx();
  c->kind = kind;
  c->n = n;
  c->b = b;
  c->nb = (n + b - 1) / b;
  c->ld = round_up(n, 16);
  c->device = device;
  c->ld_cs = round_even(2 * c->nb);
  c->ld_max = round_even(c->nb);
  c->ld_t = round_even(b);
  {
    const char* e = getenv("ABFT_NO_FUSE");
    c->fuse_enabled = !(e && e[0] == '1');
    const char* e2 = getenv("ABFT_NO_LOOKAHEAD");
    c->lookahead_enabled = !(e2 && e2[0] == '1');
    const char* e5 = getenv("ABFT_LU_COOP");
    if (e5) c->lu_coop = e5[0] == '1';
    const char* e10 = getenv("ABFT_LU_LA2");
    if (e10) c->lu_la2 = e10[0] == '1';
    const char* e4 = getenv("ABFT_CHOL_CLUSTER");
    if (e4) c->chol_cluster = e4[0] == '1';
    const char* e6 = getenv("ABFT_STREAM_CHUNK");
    if (e6) c->lu_chunk = atoi(e6);
    const char* e7 = getenv("ABFT_STREAM_SPLIT");
    if (e7) c->lu_split = atoll(e7);
    const char* e3 = getenv("ABFT_QR_LA_SMS");
    if (e3) {
      c->qr_la_sms = atoi(e3);  // 0 disables the QR look-ahead
      c->qr_la_sms_fixed = true;
    }
  }
  int rc = 0;
  auto fail = [&](int r) {
    abft_destroy(c);
    return r;
  };
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) {
    set_last_error("cudaStreamCreate failed");
    delete c;
    return -1000;
  }
  const int64_t n_ = n, ld = c->ld;
  if ((rc = dalloc(&c->m, ld * n_))) return fail(rc);
  if ((rc = dalloc(&c->gcsw, c->ld_cs * n_))) return fail(rc);
  if ((rc = dalloc(&c->csm, c->ld_cs * n_))) return fail(rc);
  if ((rc = dalloc(&c->grs, ld * c->nb))) return fail(rc);
  if ((rc = dalloc(&c->rsm, ld * c->nb))) return fail(rc);
  if ((rc = dalloc(&c->gmax, c->ld_max * c->nb))) return fail(rc);
  if ((rc = dalloc(&c->fpart, ld * 4 * c->nb))) return fail(rc);
  if ((rc = dalloc(&c->fmaxp, c->ld_max * 4 * c->nb))) return fail(rc);
  if ((rc = dalloc(&c->el, c->ld_cs * b))) return fail(rc);
  if ((rc = dalloc(&c->er, c->ld_t * std::max<int64_t>(c->nb, b)))) return fail(rc);
  if (kind == ABFT_CHOLESKY && (rc = dalloc(&c->chol_rs, ld * c->nb))) return fail(rc);
  if ((rc = dalloc(&c->lw, ld * b))) return fail(rc);
  if ((rc = dalloc(&c->uw, c->ld_t * n_))) return fail(rc);
  if ((rc = dalloc(&c->linv, c->ld_t * b))) return fail(rc);
  if ((rc = dalloc(&c->uinv, c->ld_t * b))) return fail(rc);
  if ((rc = dalloc(&c->scratch, 4096))) return fail(rc);
  if (kind == ABFT_QR) {
    if ((rc = dalloc(&c->vstore, ld * n_))) return fail(rc);
    if (cudaMemset(c->vstore, 0, ld * n_ * sizeof(double)) != cudaSuccess) return fail(-1000);
    if ((rc = dalloc(&c->tstore, c->nb * b * c->ld_t))) return fail(rc);
    if ((rc = dalloc(&c->betas, b))) return fail(rc);
    c->qr_part_elems = 2 * 160 * (b + 1);
    if ((rc = dalloc(&c->qr_part, c->qr_part_elems))) return fail(rc);
    if ((rc = dalloc(&c->qr_rowbuf, 2 * (b + 1) + 128))) return fail(rc);
    if ((rc = dalloc(&c->qr_part2, 160LL * 32 * b))) return fail(rc);
    if ((rc = dalloc(&c->qr_wfin, 32LL * b))) return fail(rc);
    if ((rc = dalloc(&c->gram, c->ld_t * b))) return fail(rc);
    if ((rc = dalloc(&c->qr_small, QR_SMALL_BUFS * c->ld_t * b))) return fail(rc);
    if ((rc = dalloc(&c->ww, c->ld_t * n_))) return fail(rc);
    if ((rc = dalloc(&c->mid, c->ld_t * n_))) return fail(rc);
  }
  // split-K workspace: bounded (falls back to fewer splits when short)
  c->gws.elems = std::min<int64_t>(std::max<int64_t>(8 * ld * b, 1 << 20), int64_t(64) << 20);
  if ((rc = dalloc(&c->gws.ptr, c->gws.elems))) return fail(rc);
  if (kind == ABFT_CHOLESKY || kind == ABFT_QR) {
    c->gws2.elems = c->gws.elems;
    if ((rc = dalloc(&c->gws2.ptr, c->gws2.elems))) return fail(rc);
  }
  c->ev_cap = 1 << 16;
  if (cudaMalloc(&c->ev, c->ev_cap * sizeof(Event)) != cudaSuccess) return fail(-1000);
  if (cudaMalloc(&c->counters, 4 * sizeof(int32_t)) != cudaSuccess) return fail(-1000);
  cudaMemset(c->counters, 0, 4 * sizeof(int32_t));
  c->dirty_cap = 1 << 16;
  if (cudaMalloc(&c->dirty, 2 * c->dirty_cap * sizeof(int32_t)) != cudaSuccess) return fail(-1000);
  if (cudaMalloc(&c->info, 2 * sizeof(int)) != cudaSuccess) return fail(-1000);
  cudaMemset(c->info, 0, 2 * sizeof(int));
  if (kind == ABFT_QR) {
    QrPanelWork& q = c->qrw;
    q.q1 = c->lw;
    q.ldq = ld;
    q.small = c->qr_small;
    q.lds = c->ld_t;
    q.info = c->info + 1;
    q.gws = &c->gws;
    q.part = c->qr_part;
    q.part_elems = c->qr_part_elems;
    q.rowbuf = c->qr_rowbuf;
    q.part2 = c->qr_part2;
    q.wfin = c->qr_wfin;
    q.gram = c->gram;
    q.ldg = c->ld_t;
  }
  cudaEventCreate(&c->e0);
  cudaEventCreate(&c->e1);
  cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c->st_out, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c->st_in, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_p, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_r, cudaEventDisableTiming);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(-1000);
  *out = c;
  return 0;
}

ABFT_API int abft_destroy(abft_ctx* c) {
  if (!c) return 0;
  DevGuard g(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  double* bufs[] = {c->m,     c->a0,     c->gcsw,   c->grs,     c->gmax,  c->csm,  c->rsm,
                    c->fpart, c->fmaxp,
                    c->chol_rs,
                    c->el,    c->er,     c->lw,     c->uw,      c->linv,  c->uinv, c->vstore,
                    c->tstore, c->betas, c->qr_part, c->qr_rowbuf, c->gram, c->ww,  c->mid,
                    c->qr_part2, c->qr_wfin, c->qr_small,
                    c->scratch, c->gws.ptr, c->gws2.ptr, c->linv_store, c->el_store};
  for (double* p : bufs)
    if (p) cudaFree(p);
  if (c->ev) cudaFree(c->ev);
  if (c->counters) cudaFree(c->counters);
  if (c->dirty) cudaFree(c->dirty);
  if (c->dplan) cudaFree(c->dplan);
  if (c->dlist) cudaFree(c->dlist);
  if (c->info) cudaFree(c->info);
  if (c->ipiv) cudaFree(c->ipiv);
  if (c->piv_part) cudaFree(c->piv_part);
  for (auto& s : c->snaps) {
    if (s.m) cudaFree(s.m);
    if (s.chol_rs) cudaFree(s.chol_rs);
  }
  for (auto& pe : c->prof_pending) {
    cudaEventDestroy(pe.e0);
    cudaEventDestroy(pe.e1);
  }
  for (auto e : c->prof_free) cudaEventDestroy(e);
  if (c->st2) {
    cudaStreamSynchronize(c->st2);
    cudaStreamDestroy(c->st2);
  }
  if (c->st_out) {
    cudaStreamSynchronize(c->st_out);
    cudaStreamDestroy(c->st_out);
  }
  if (c->st_in) {
    cudaStreamSynchronize(c->st_in);
    cudaStreamDestroy(c->st_in);
  }
  for (auto e : c->ev_in) cudaEventDestroy(e);
  if (c->rs_tmp) cudaFree(c->rs_tmp);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_p) cudaEventDestroy(c->ev_p);
  if (c->ev_r) cudaEventDestroy(c->ev_r);
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
  return 0;
}

ABFT_API int abft_set_matrix(abft_ctx* c, const double* a, int64_t lda) {
  DevGuard g(c->device);
  c->in_host = nullptr;
  if (lda < c->n) {
    set_last_error("lda < n");
    return ABFT_E_INVALID;
  }
  CUDA_TRY(cudaMemcpy2DAsync(c->m, c->ld * 8, a, lda * 8, c->n * 8, c->n, cudaMemcpyHostToDevice,
                             c->st));
  if (c->keep_input) {
    if (!c->a0) ABFT_TRY(dalloc(&c->a0, c->ld * c->n));
    CUDA_TRY(cudaMemcpy2DAsync(c->a0, c->ld * 8, c->m, c->ld * 8, c->n * 8, c->n,
                               cudaMemcpyDeviceToDevice, c->st));
  }
  CUDA_TRY(cudaStreamSynchronize(c->st));
  c->k_done = 0;
  c->sums_valid = false;
  c->qr_count = 0;
  c->breakdown_col = -1;
  c->pd_ready = -1;
  c->pu_ready = -1;
  c->chol_part = -1;
  c->chol_enc_ahead = false;
  c->chol_rs_valid = false;
  return 0;
}

// Like abft_set_matrix, but the copy is deferred into the next
// abft_factorize call, column block by column block on a copy stream, and
// overlaps the factorization (Cholesky reads only the lower block triangle:
// rows >= j b of block column j are copied, the rest of the device matrix is
// zeroed by the factorization itself). `a` must stay valid (and should be
// pinned) until that call returns. With keep_input (abft_reset) this is a
// plain abft_set_matrix.
ABFT_API int abft_set_matrix_streamed(abft_ctx* c, const double* a, int64_t lda) {
  if (c->keep_input) return abft_set_matrix(c, a, lda);
  DevGuard g(c->device);
  if (lda < c->n) {
    set_last_error("lda < n");
    return ABFT_E_INVALID;
  }
  if (c->kind == ABFT_CHOLESKY && !c->rs_tmp) ABFT_TRY(dalloc(&c->rs_tmp, c->ld));
  c->in_host = a;
  c->in_ld = lda;
  c->k_done = 0;
  c->sums_valid = false;
  c->qr_count = 0;
  c->breakdown_col = -1;
  c->pd_ready = -1;
  c->pu_ready = -1;
  c->chol_part = -1;
  c->chol_enc_ahead = false;
  c->chol_rs_valid = false;
  return 0;
}

// Restore the working matrix from the kept device copy of the input (a new
// factorization of the same matrix without a host round trip).
ABFT_API int abft_reset(abft_ctx* c) {
  DevGuard g(c->device);
  if (!c->a0) {
    set_last_error("abft_reset needs abft_keep_input(ctx, 1) before abft_set_matrix");
    return ABFT_E_INVALID;
  }
  CUDA_TRY(cudaMemcpy2DAsync(c->m, c->ld * 8, c->a0, c->ld * 8, c->n * 8, c->n,
                             cudaMemcpyDeviceToDevice, c->st));
  c->k_done = 0;
  c->sums_valid = false;
  c->qr_count = 0;
  c->breakdown_col = -1;
  c->pd_ready = -1;
  c->pu_ready = -1;
  c->chol_part = -1;
  c->chol_enc_ahead = false;
  c->chol_rs_valid = false;
  return 0;
}

ABFT_API void* abft_stream(abft_ctx* c) { return reinterpret_cast<void*>(c->st); }

// m <- m m^T + n I on the device (generate_test_matrix's SPD construction,
// linalg.py:74-75, with the product on the DMMA GEMM instead of host BLAS);
// the kept input copy (if any) is refreshed.
ABFT_API int abft_make_spd(abft_ctx* c) {
  DevGuard g(c->device);
  ABFT_TRY(flush_pending_input(c));
  double* T = nullptr;
  ABFT_TRY(dalloc(&T, c->ld * c->n));
  int rc = gemm(c->st, 'N', 'T', (int)c->n, (int)c->n, (int)c->n, 1.0, c->m, c->ld, c->m, c->ld,
                0.0, nullptr, 0, T, c->ld, &c->gws);
  if (!rc) rc = add_diag(c->st, T, c->ld, c->n, (double)c->n);
  if (!rc) rc = copy_matrix(c->st, T, c->ld, c->m, c->ld, c->n, c->n, 0);
  if (!rc && c->a0) rc = copy_matrix(c->st, T, c->ld, c->a0, c->ld, c->n, c->n, 0);
  cudaStreamSynchronize(c->st);
  cudaFree(T);
  return rc;
}

ABFT_API int abft_keep_input(abft_ctx* c, int keep) {
  c->keep_input = keep != 0;
  return 0;
}

ABFT_API int abft_get_matrix(abft_ctx* c, double* mh, int64_t ldm) {
  DevGuard g(c->device);
  ABFT_TRY(flush_pending_input(c));
  CUDA_TRY(cudaMemcpy2DAsync(mh, ldm * 8, c->m, c->ld * 8, c->n * 8, c->n, cudaMemcpyDeviceToHost,
                             c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

ABFT_API int64_t abft_k_done(abft_ctx* c) { return c->k_done; }

ABFT_API int abft_set_k_done(abft_ctx* c, int64_t k) {
  c->k_done = k;
  return 0;
}

ABFT_API int abft_task(abft_ctx* c, int64_t k, int task) {
  DevGuard g(c->device);
  ABFT_TRY(flush_pending_input(c));
  if (k < 0 || k >= c->nb) {
    set_last_error("iteration %lld out of range", (long long)k);
    return ABFT_E_DIM;
  }
  if (task == ABFT_TASK_PD) {
    ABFT_TRY(task_pd(c, k));
    ABFT_TRY(check_info(c));
  } else if (task == ABFT_TASK_PU) {
    ABFT_TRY(task_pu(c, k));
  } else if (task == ABFT_TASK_TMU) {
    bool did;
    ABFT_TRY(tmu_gemm(c, k, &did));
    c->sums_valid = false;
  } else {
    set_last_error("unknown task %d", task);
    return ABFT_E_INVALID;
  }
  return 0;
}

ABFT_API int abft_iteration(abft_ctx* c, int64_t k, int scheme, const abft_fault* plan, int nplan,
                            int correct, abft_report* rep, abft_location* locs, int max_locs) {
  DevGuard g(c->device);
  ABFT_TRY(flush_pending_input(c));
  if (k < 0 || k >= c->nb) {
    set_last_error("iteration %lld out of range for %lld blocks", (long long)k, (long long)c->nb);
    return ABFT_E_DIM;
  }
  if (scheme < 0 || scheme > 2) {
    set_last_error("unknown checksum scheme %d", scheme);
    return ABFT_E_INVALID;
  }
  CUDA_TRY(cudaMemsetAsync(c->counters, 0, 2 * sizeof(int32_t), c->st));
  CUDA_TRY(cudaEventRecord(c->e0, c->st));
  c->cur_iter = (int32_t)k;
  int rc = run_iteration_device(c, k, scheme, plan, nplan, correct, true);
  CUDA_TRY(cudaEventRecord(c->e1, c->st));
  c->timed = true;
  if (rc != 0) return rc;
  int64_t r0, c0, rows, cols;
  region_of(c, k, &r0, &c0, &rows, &cols);
  ABFT_TRY(collect_events(c, {r0}, {c0}, nullptr, rep, locs, max_locs, nullptr));
  c->k_done = k + 1;
  return 0;
}

ABFT_API int abft_factorize(abft_ctx* c, int scheme, const int32_t* schemes, const abft_fault* plan,
                            const int64_t* plan_iter, int nplan, int correct, abft_report* reports,
                            abft_location* locs, int max_locs, int* n_locs) {
  DevGuard g(c->device);
  CUDA_TRY(cudaMemsetAsync(c->counters, 0, 2 * sizeof(int32_t), c->st));
  if (n_locs) *n_locs = 0;
  const int64_t k0 = c->k_done;
  c->want_chol_rs = false;
  for (int64_t k = k0; k < c->nb; ++k)
    if ((schemes ? schemes[k] : scheme) == ABFT_FULL) c->want_chol_rs = true;
  CUDA_TRY(cudaEventRecord(c->e0, c->st));
  c->timed = true;
  c->in_stream = false;
  int64_t lu_split = 0;  // streamed LU: iterations [0, lu_split) ran chunk by chunk
  if (c->in_host) {
    // streamed input: every column block goes out now on st_in (in order);
    // Cholesky iterations wait for their own block, LU / QR for all of them
    const bool chol = c->kind == ABFT_CHOLESKY;
    if ((int64_t)c->ev_in.size() < c->nb) {
      for (int64_t j = (int64_t)c->ev_in.size(); j < c->nb; ++j) {
        cudaEvent_t e = nullptr;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_in.push_back(e);
      }
    }
    CUDA_TRY(cudaEventRecord(c->ev_a, c->st));  // the previous use of the matrix is over
    CUDA_TRY(cudaStreamWaitEvent(c->st_in, c->ev_a, 0));
    for (int64_t j = 0; j < c->nb; ++j) {
      const int64_t p = j * c->b, w = std::min(c->b, c->n - p);
      const int64_t r0 = chol ? p : 0;
      CUDA_TRY(cudaMemcpy2DAsync(c->m + r0 + p * c->ld, c->ld * 8, c->in_host + r0 + p * c->in_ld,
                                 c->in_ld * 8, (c->n - r0) * 8, w, cudaMemcpyHostToDevice, c->st_in));
      CUDA_TRY(cudaEventRecord(c->ev_in[j], c->st_in));
    }
    c->in_host = nullptr;
    if (chol) {
      c->in_stream = true;
      c->rs_enc.assign(c->nb, 0);
    } else {
      // LU: chunked left part while the input arrives, if no fault is planned there
      lu_split = k0 == 0 ? lu_stream_split(c) : 0;
      if (plan && plan_iter)
        for (int f = 0; f < nplan; ++f)
          if (plan_iter[f] < lu_split) lu_split = 0;
      if (lu_split == 0) CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_in[c->nb - 1], 0));
    }
  }
  if (lu_split > 0) {
    int rc = lu_stream_chunks(c, lu_split, scheme, schemes, correct);
    if (rc != 0) {
      cudaEventRecord(c->e1, c->st);
      return rc;
    }
  }
  for (int64_t k = std::max(k0, lu_split); k < c->nb; ++k) {
    const int sch = schemes ? schemes[k] : scheme;
    int f0 = 0, f1 = 0;
    if (plan && plan_iter) {
      while (f0 < nplan && plan_iter[f0] < k) ++f0;
      f1 = f0;
      while (f1 < nplan && plan_iter[f1] == k) ++f1;
    }
    c->cur_iter = (int32_t)k;
    c->next_scheme = (k + 1 < c->nb) ? (schemes ? schemes[k + 1] : scheme) : ABFT_NONE;
    int rc = run_iteration_device(c, k, sch, plan ? plan + f0 : nullptr, f1 - f0, correct, false,
                                  c->lookahead_enabled);
    if (rc != 0) {
      cudaEventRecord(c->e1, c->st);
      c->in_stream = false;
      return rc;
    }
  }
  c->in_stream = false;
  if (c->out_host) {  // the streamed result is part of the call
    CUDA_TRY(cudaEventRecord(c->ev_out, c->st_out));
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_out, 0));
  }
  CUDA_TRY(cudaEventRecord(c->e1, c->st));
  // one synchronisation for the whole factorization
  int brk = check_info(c);
  if (brk != 0) {
    c->k_done = c->breakdown_col / c->b;
    return brk;
  }
  // events of all iterations, split per iteration in reference order
  std::vector<Event> evs;
  ABFT_TRY(collect_events(c, {0}, {0}, nullptr, nullptr, nullptr, 0, &evs));
  std::stable_sort(evs.begin(), evs.end(), [](const Event& a, const Event& b) {
    if (a.iter != b.iter) return a.iter < b.iter;
    if (a.bi != b.bi) return a.bi < b.bi;
    if (a.bj != b.bj) return a.bj < b.bj;
    return a.seq < b.seq;
  });
  if (reports)
    for (int64_t k = k0; k < c->nb; ++k) memset(&reports[k], 0, sizeof(abft_report));
  int total = 0;
  for (const Event& e : evs) {
    if (e.kind < 0) {
      set_last_error("index 0 is out of bounds for axis 0 with size 0");
      return ABFT_E_RANGE;
    }
    const int64_t k = e.iter;
    int64_t r0, c0, rows, cols;
    region_of(c, k, &r0, &c0, &rows, &cols);
    if (reports) {
      abft_report& rep = reports[k];
      rep.detected[e.detected_kind] += 1;
      if (e.corrected) rep.corrected[e.detected_kind] += 1;
      if (e.uncorrectable) rep.uncorrectable = 1;
      rep.n_locations += 1;
    }
    if (locs && total < max_locs) {
      abft_location& L = locs[total];
      L.row = e.row + r0;
      L.col = e.col + c0;
      L.kind = e.kind;
      L.flag = e.flag;
      L.detected_kind = e.detected_kind;
      L.corrected = e.corrected;
      L.uncorrectable = e.uncorrectable;
      L.block_row = e.bi;
      L.block_col = e.bj;
      L.seq = e.seq;
    }
    ++total;
  }
  c->k_done = c->nb;
  if (n_locs) *n_locs = total;
  return 0;
}

// Stream the finished factor into `host` (column-major, ldh; pinned memory
// makes the copies asynchronous) during the next abft_factorize calls;
// NULL turns streaming off. Replaces the abft_get_matrix round trip.
ABFT_API int abft_stream_out(abft_ctx* c, double* host, int64_t ldh) {
  if (host && ldh < c->n) {
    set_last_error("ldh < n");
    return ABFT_E_INVALID;
  }
  c->out_host = host;
  c->out_ld = ldh;
  return 0;
}

ABFT_API int abft_profile(abft_ctx* c, int enable) {
  c->prof_on = enable != 0;
  for (int i = 0; i < PROF_N; ++i) c->prof_ms[i] = 0.0;
  c->prof_pending.clear();
  c->prof_iter.assign(c->nb, {0.0, 0.0, 0.0, 0.0});
  return 0;
}

// LU with partial pivoting (LAPACK dgetrf semantics; the reference factors
// unpivoted, linalg.py:230-238). Set before iteration 0.
ABFT_API int abft_set_pivoting(abft_ctx* c, int enable) {
  DevGuard g(c->device);
  if (c->kind != ABFT_LU && enable) {
    set_last_error("partial pivoting is an LU option");
    return ABFT_E_INVALID;
  }
  if (c->k_done != 0) {
    set_last_error("abft_set_pivoting before the first iteration");
    return ABFT_E_INVALID;
  }
  c->pivot = enable != 0;
  if (c->pivot && !c->ipiv) {
    CUDA_TRY(cudaMalloc(&c->ipiv, c->n * sizeof(int32_t)));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    c->piv_part_elems = 2LL * (sms + 1) * (c->b + 2);
    ABFT_TRY(dalloc(&c->piv_part, c->piv_part_elems));
  }
  c->sums_valid = false;
  return 0;
}

// The pivots (global 0-based: row i was interchanged with row piv[i], in
// order; LAPACK ipiv - 1). Valid for the completed panels.
ABFT_API int abft_get_pivots(abft_ctx* c, int32_t* piv) {
  DevGuard g(c->device);
  if (!c->pivot) {
    for (int64_t i = 0; i < c->n; ++i) piv[i] = (int32_t)i;
    return 0;
  }
  CUDA_TRY(cudaMemcpyAsync(piv, c->ipiv, c->n * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  for (int64_t k = 0; k < c->nb; ++k) {
    const int64_t p = k * c->b, w = std::min(c->b, c->n - p);
    for (int64_t j = 0; j < w; ++j) piv[p + j] = (int32_t)(p + piv[p + j]);
  }
  return 0;
}

// Per-iteration device times since abft_profile(ctx, 1): out[4k + t] for
// t = PD (incl. a look-ahead's side-stream panel), PU, TMU, ABFT.
ABFT_API int abft_profile_read_iters(abft_ctx* c, double* out, int64_t nb) {
  double tot[4];
  ABFT_TRY(abft_profile_read(c, tot));
  for (int64_t k = 0; k < nb && k < (int64_t)c->prof_iter.size(); ++k)
    for (int t = 0; t < 4; ++t) out[4 * k + t] = c->prof_iter[k][t];
  return 0;
}

// Per-iteration SMs left to the panel work when iteration k's panel is
// factored beside a look-ahead update (QR: the side-stream panel's GEMMs;
// LU: >= ceil(b/32) selects the multi-CTA diagonal factor). 0 or a null
// array: the built-in choice. The B200 form of the reference's slack
// reclamation (scheduler.py:84-146): the stream with slack gets fewer SMs.
ABFT_API int abft_set_input_chunks(abft_ctx* c, int chunk, int64_t split, int right_chunk) {
  if (chunk < -1 || split < -1 || right_chunk < -1) {
    set_last_error("abft_set_input_chunks: chunk, split, right_chunk >= -1");
    return ABFT_E_INVALID;
  }
  c->lu_chunk = chunk;
  c->lu_split = split;
  c->lu_rchunk = right_chunk;
  return 0;
}

ABFT_API int abft_set_side_sms(abft_ctx* c, const int32_t* sms, int64_t nb) {
  if (!sms || nb <= 0) {
    c->side_sms.clear();
    return 0;
  }
  c->side_sms.assign(sms, sms + nb);
  return 0;
}

// Accumulated per-task device time since abft_profile(ctx, 1):
// ms[0] PD, ms[1] PU, ms[2] TMU GEMMs, ms[3] ABFT (encode/maintain/verify/inject)
ABFT_API int abft_profile_read(abft_ctx* c, double* ms) {
  DevGuard g(c->device);
  CUDA_TRY(cudaStreamSynchronize(c->st));
  if ((int64_t)c->prof_iter.size() < c->nb) c->prof_iter.resize(c->nb, {0.0, 0.0, 0.0, 0.0});
  CUDA_TRY(cudaStreamSynchronize(c->st2));
  for (auto& pe : c->prof_pending) {
    float f = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&f, pe.e0, pe.e1));
    c->prof_ms[pe.cat] += f;
    if (pe.iter >= 0 && pe.iter < c->nb) c->prof_iter[pe.iter][pe.cat] += f;
    c->prof_free.push_back(pe.e0);
    c->prof_free.push_back(pe.e1);
  }
  c->prof_pending.clear();
  for (int i = 0; i < PROF_N; ++i) ms[i] = c->prof_ms[i];
  return 0;
}

ABFT_API int abft_last_elapsed_ms(abft_ctx* c, double* ms) {
  DevGuard g(c->device);
  if (!c->timed) {
    *ms = 0.0;
    return 0;
  }
  CUDA_TRY(cudaEventSynchronize(c->e1));
  float f = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&f, c->e0, c->e1));
  *ms = f;
  return 0;
}

ABFT_API int abft_qr_panels(abft_ctx* c) { return c->qr_count; }

ABFT_API int abft_get_qr_panel(abft_ctx* c, int64_t k, double* V, int64_t ldv, double* T,
                               int64_t ldt) {
  DevGuard g(c->device);
  if (c->kind != ABFT_QR || k < 0 || k >= c->qr_count) {
    set_last_error("no QR panel %lld", (long long)k);
    return ABFT_E_INVALID;
  }
  const int64_t p = k * c->b, pe = std::min(p + c->b, c->n), w = pe - p;
  if (V)
    CUDA_TRY(cudaMemcpy2DAsync(V, ldv * 8, c->vstore + p + p * c->ld, c->ld * 8, (c->n - p) * 8, w,
                               cudaMemcpyDeviceToHost, c->st));
  if (T)
    CUDA_TRY(cudaMemcpy2DAsync(T, ldt * 8, c->tstore + k * c->b * c->ld_t, c->ld_t * 8, w * 8, w,
                               cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

ABFT_API int abft_snapshot(abft_ctx* c, int slot) {
  DevGuard g(c->device);
  ABFT_TRY(flush_pending_input(c));
  if (slot < 0 || slot > 64) {
    set_last_error("bad snapshot slot");
    return ABFT_E_INVALID;
  }
  if ((int)c->snaps.size() <= slot) c->snaps.resize(slot + 1);
  Snapshot& s = c->snaps[slot];
  if (!s.m) ABFT_TRY(dalloc(&s.m, c->ld * c->n));
  CUDA_TRY(cudaMemcpyAsync(s.m, c->m, c->ld * c->n * 8, cudaMemcpyDeviceToDevice, c->st));
  if (c->chol_rs) {
    if (!s.chol_rs) ABFT_TRY(dalloc(&s.chol_rs, c->ld * c->nb));
    CUDA_TRY(cudaMemcpyAsync(s.chol_rs, c->chol_rs, c->ld * c->nb * 8, cudaMemcpyDeviceToDevice,
                             c->st));
  }
  s.chol_rs_valid = c->chol_rs_valid;
  s.k_done = c->k_done;
  s.qr_count = c->qr_count;
  s.used = true;
  return 0;
}

ABFT_API int abft_restore(abft_ctx* c, int slot) {
  DevGuard g(c->device);
  if (slot < 0 || slot >= (int)c->snaps.size() || !c->snaps[slot].used) {
    set_last_error("empty snapshot slot %d", slot);
    return ABFT_E_INVALID;
  }
  Snapshot& s = c->snaps[slot];
  CUDA_TRY(cudaMemcpyAsync(c->m, s.m, c->ld * c->n * 8, cudaMemcpyDeviceToDevice, c->st));
  if (c->chol_rs && s.chol_rs)
    CUDA_TRY(cudaMemcpyAsync(c->chol_rs, s.chol_rs, c->ld * c->nb * 8, cudaMemcpyDeviceToDevice,
                             c->st));
  c->chol_rs_valid = s.chol_rs_valid && s.chol_rs != nullptr;
  c->k_done = s.k_done;
  c->qr_count = s.qr_count;
  c->sums_valid = false;
  c->pd_ready = -1;
  c->pu_ready = -1;
  c->chol_part = -1;
  c->chol_enc_ahead = false;
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

ABFT_API int64_t abft_breakdown_column(abft_ctx* c) { return c->breakdown_col; }

// Debug/test accessor for the device checksum state:
// which = 0 gcsw (2nb x n), 1 csm (2nb x n), 2 grs (n x nb), 3 rsm (n x nb),
// 4 gmax (nb x nb). Copies the full array into `out` (column-major).
ABFT_API int abft_debug_array(abft_ctx* c, int which, double* out, int64_t* rows, int64_t* cols) {
  DevGuard g(c->device);
  ABFT_TRY(flush_pending_input(c));
  const double* src;
  int64_t r, cl, ld;
  switch (which) {
    case 0: src = c->gcsw; r = 2 * c->nb; cl = c->n; ld = c->ld_cs; break;
    case 1: src = c->csm; r = 2 * c->nb; cl = c->n; ld = c->ld_cs; break;
    case 2: src = c->grs; r = c->n; cl = c->nb; ld = c->ld; break;
    case 3: src = c->rsm; r = c->n; cl = c->nb; ld = c->ld; break;
    case 4: src = c->gmax; r = c->nb; cl = c->nb; ld = c->ld_max; break;
    default: set_last_error("bad array id"); return ABFT_E_INVALID;
  }
  *rows = r;
  *cols = cl;
  if (out) {
    CUDA_TRY(cudaStreamSynchronize(c->st));
    CUDA_TRY(cudaMemcpy2D(out, r * 8, src, ld * 8, r * 8, cl, cudaMemcpyDeviceToHost));
  }
  return 0;
}

// reconstruct (linalg.py:340-359) into device buffer `out` (ld = c->ld);
// `tmp` is an n x ld scratch buffer.
static int reconstruct_device(abft_ctx* c, double* out, double* tmp) {
  const int64_t n = c->n, ld = c->ld;
  if (c->kind == ABFT_LU) {
    ABFT_TRY(copy_matrix(c->st, c->m, ld, tmp, ld, n, n, 1));  // L (unit)
    ABFT_TRY(copy_matrix(c->st, c->m, ld, out, ld, n, n, 2));  // U
    // out = L U, computed in place from a copy of U
    double* U = nullptr;
    ABFT_TRY(dalloc(&U, ld * n));
    int rc = copy_matrix(c->st, out, ld, U, ld, n, n, 0);
    if (!rc)
      rc = gemm(c->st, 'N', 'N', (int)n, (int)n, (int)n, 1.0, tmp, ld, U, ld, 0.0, nullptr, 0, out,
                ld, &c->gws);
    // pivoted: A = P^T L U -- undo the interchanges, last panel first
    for (int64_t k = c->nb - 1; c->pivot && !rc && k >= 0; --k) {
      const int64_t p = k * c->b, w = std::min(c->b, n - p);
      rc = laswp(c->st, out, ld, 0, n, p, (int)w, c->ipiv + p, true);
    }
    cudaStreamSynchronize(c->st);
    cudaFree(U);
    return rc;
  }
  if (c->kind == ABFT_CHOLESKY) {
    ABFT_TRY(copy_matrix(c->st, c->m, ld, tmp, ld, n, n, 3));
    return gemm(c->st, 'N', 'T', (int)n, (int)n, (int)n, 1.0, tmp, ld, tmp, ld, 0.0, nullptr, 0,
                out, ld, &c->gws);
  }
  // out = triu(m); for k from last to 0: out[p:n,:] -= V (T (V^T out[p:n,:]))
  ABFT_TRY(copy_matrix(c->st, c->m, ld, out, ld, n, n, 2));
  for (int64_t k = c->qr_count - 1; k >= 0; --k) {
    const int64_t p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
    const double* V = c->vstore + p + p * ld;
    const double* T = c->tstore + k * c->b * c->ld_t;
    double* blk = out + p;
    ABFT_TRY(gemm(c->st, 'T', 'N', (int)w, (int)n, (int)(n - p), 1.0, V, ld, blk, ld, 0.0, nullptr,
                  0, c->ww, c->ld_t, &c->gws));
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)w, (int)n, (int)w, 1.0, T, c->ld_t, c->ww, c->ld_t, 0.0,
                  nullptr, 0, c->mid, c->ld_t, &c->gws));
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)(n - p), (int)n, (int)w, -1.0, V, ld, c->mid, c->ld_t, 1.0,
                  blk, ld, blk, ld, &c->gws));
  }
  return 0;
}

ABFT_API int abft_reconstruct(abft_ctx* c, double* outh, int64_t ldo) {
  DevGuard g(c->device);
  ABFT_TRY(flush_pending_input(c));
  if (c->k_done < c->nb) {
    set_last_error("factorization incomplete");
    return ABFT_E_INCOMPLETE;
  }
  const int64_t n = c->n, ld = c->ld;
  double *X = nullptr, *T = nullptr;
  int rc = dalloc(&X, ld * n);
  if (!rc) rc = dalloc(&T, ld * n);
  if (!rc) rc = reconstruct_device(c, X, T);
  if (!rc && cudaMemcpy2DAsync(outh, ldo * 8, X, ld * 8, n * 8, n, cudaMemcpyDeviceToHost, c->st) !=
                 cudaSuccess)
    rc = -1000;
  cudaStreamSynchronize(c->st);
  if (X) cudaFree(X);
  if (T) cudaFree(T);
  return rc;
}

ABFT_API int abft_set_qr_panel(abft_ctx* c, int64_t k, const double* V, int64_t ldv,
                               const double* T, int64_t ldt) {
  DevGuard g(c->device);
  if (c->kind != ABFT_QR || k < 0 || k >= c->nb || k > c->qr_count) {
    set_last_error("cannot set QR panel %lld", (long long)k);
    return ABFT_E_INVALID;
  }
  const int64_t p = k * c->b, pe = std::min(p + c->b, c->n), w = pe - p;
  CUDA_TRY(cudaMemcpy2DAsync(c->vstore + p + p * c->ld, c->ld * 8, V, ldv * 8, (c->n - p) * 8, w,
                             cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaMemcpy2DAsync(c->tstore + k * c->b * c->ld_t, c->ld_t * 8, T, ldt * 8, w * 8, w,
                             cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  c->qr_count = (int)std::max<int64_t>(c->qr_count, k + 1);
  return 0;
}

ABFT_API int abft_set_qr_panels(abft_ctx* c, int count) {
  if (count < 0 || count > c->qr_count) {
    set_last_error("cannot extend the QR panel list from the host");
    return ABFT_E_INVALID;
  }
  c->qr_count = count;
  return 0;
}

ABFT_API int abft_residual(abft_ctx* c, const double* a0h, int64_t lda, double* out) {
  DevGuard g(c->device);
  ABFT_TRY(flush_pending_input(c));
  if (c->k_done < c->nb) {
    set_last_error("factorization incomplete");
    return ABFT_E_INCOMPLETE;
  }
  const int64_t n = c->n, ld = c->ld;
  double *A = nullptr, *X = nullptr, *T = nullptr;
  bool own_a = false;
  int rc = 0;
  if (a0h) {
    rc = dalloc(&A, ld * n);
    own_a = true;
    if (!rc && cudaMemcpy2DAsync(A, ld * 8, a0h, lda * 8, n * 8, n, cudaMemcpyHostToDevice, c->st) !=
                   cudaSuccess)
      rc = -1000;
  } else if (c->a0) {
    A = c->a0;
  } else {
    set_last_error("no input matrix for the residual");
    return ABFT_E_INVALID;
  }
  if (!rc) rc = dalloc(&X, ld * n);
  if (!rc) rc = dalloc(&T, ld * n);
  double* sq = c->scratch + 2048;
  if (!rc) rc = sumsq(c->st, A, ld, n, n, sq, c->scratch);            // ||A||^2
  if (!rc) rc = reconstruct_device(c, X, T);
  if (!rc) rc = sub_matrix(c->st, A, ld, X, ld, n, n);                // X = rec - A
  if (!rc) rc = sumsq(c->st, X, ld, n, n, sq + 1, c->scratch + 1024);  // ||A - rec||^2
  double h[2] = {0, 0};
  if (!rc && cudaMemcpyAsync(h, sq, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st) !=
                 cudaSuccess)
    rc = -1000;
  cudaStreamSynchronize(c->st);
  if (X) cudaFree(X);
  if (T) cudaFree(T);
  if (own_a && A) cudaFree(A);
  if (rc) return rc;
  const double na = sqrt(h[0]), nd = sqrt(h[1]);
  *out = (na == 0.0) ? nd : nd / na;
  return 0;
}

}  // extern "C"
