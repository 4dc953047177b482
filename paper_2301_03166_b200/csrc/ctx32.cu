// Single-precision factorization context (the s* variants of the north star:
// sgetrf / spotrf) on the tcgen05 fp32 GEMM (sgemm_tc05.cu).
//
// Same algorithm, task order, regions, fault semantics and event order as
// the fp64 context (ctx.cu, restating linalg.py:159-359 and
// simulator.py:86-167); the data is fp32, the block checksums, their
// maintenance and verification stay fp64 (abft.py:118-276 with tau on eps32,
// the reference has no fp32 path, so parity is unpinned and
// checked against the fp64 oracle's fault outcomes).
//   LU       right-looking: PD = diag factor + L21 = A21 U11^{-1} (tcgen05),
//            PU = L11^{-1} A12 (tcgen05), TMU = A22 -= L21 U12 with the block
//            checksums produced in the GEMM epilogue (b = 128).
//   Cholesky left-looking like the reference: TMU = panel -= L L^T (tcgen05),
//            PD = diag factor, PU = L21 = A21 L11^{-T} (tcgen05).
//   QR       compact-WY: the Householder panel is factored in fp64 from the
//            widened fp32 panel (the fp64 cooperative panel kernel + larft,
//            a mixed-precision panel), V / T / R are stored back in fp32, and
//            the trailing update C -= V (T^T (V^T C)) runs on tcgen05 with the
//            fused checksums.
// The maintenance products run on the fp64 DMMA GEMM from widened operands.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "abft_b200.h"
#include "abft_kernels.cuh"
#include "gemm.cuh"
#include "panel.cuh"
#include "sgemm.cuh"

using namespace abft;

namespace {

inline int64_t s_round_even(int64_t x) { return (x + 1) / 2 * 2; }
inline int64_t s_round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct SGuard {
  int prev = -1;
  explicit SGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~SGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename T>
int salloc(T** p, int64_t elems, cudaStream_t st) {
  CUDA_TRY(cudaMalloc(p, std::max<int64_t>(elems, 1) * sizeof(T)));
  CUDA_TRY(cudaMemsetAsync(*p, 0, std::max<int64_t>(elems, 1) * sizeof(T), st));
  return 0;
}

enum { SP_PD = 0, SP_PU = 1, SP_TMU = 2, SP_ABFT = 3 };

}  // namespace

struct abft_sctx {
  int kind = 0;
  int64_t n = 0, b = 0, nb = 0, ld = 0;
  int device = 0;
  cudaStream_t st = nullptr;
  float* m = nullptr;
  float* a0 = nullptr;
  bool keep_input = false;
  // fp64 checksums on the global block grid (as ctx.cu)
  double* gcsw = nullptr;
  int64_t ld_cs = 0;
  double* grs = nullptr;
  double* gmax = nullptr;
  int64_t ld_max = 0;
  double* csm = nullptr;
  double* rsm = nullptr;
  double* el = nullptr;
  double* er = nullptr;
  int64_t ld_t = 0;
  double* lwd = nullptr;  // widened left operand (n x b)
  // QR: fp32 V / T of every panel, fp64 panel workspaces
  float* vstore = nullptr;   // n x n (ld)
  float* tstore = nullptr;   // nb of b x b (ld_t)
  float* ww = nullptr;       // b x n (ld_t)
  float* mid = nullptr;      // b x n (ld_t)
  double* pan64 = nullptr;   // n x b (ld)
  double* v64 = nullptr;     // n x b (ld)
  double* t64 = nullptr;     // b x b (ld_t)
  double* gram = nullptr;    // b x b
  int qr_la_sms = 0;            // QR look-ahead: SMs left to the side-stream panel
                                // (ABFT_QR_LA_SMS=R enables it). Off: the fp32 update is
                                // short, the fp64 panel is the critical path, and taking
                                // SMs from it measured slower (sgeqrf 41.0 -> 35.0 / 37.9
                                // TF/s at R = 16 / 24)
  bool lu_coop = true;          // LU look-ahead diagonal factor on the multi-CTA kernel
                                // beside the update capped at sms - b/32 (ABFT_LU_COOP=0: off)
  bool chol_cluster = true;     // Cholesky PD on the cluster kernel (ABFT_CHOL_CLUSTER=0: off);
                                // spotrf N=16384 32.4 -> 35.4 TF/s (the fp32 update is short,
                                // so the diagonal chain was on the critical path)
  double* qr_q1 = nullptr;     // fp64 n x b: CholeskyQR2 Q of the widened panel
  double* qr_small = nullptr;  // QR_SMALL_BUFS x (ld_t x b)
  QrPanelWork qrw;
  double* betas = nullptr;
  double* qr_part = nullptr;
  int64_t qr_part_elems = 0;
  double* qr_rowbuf = nullptr;
  double* qr_part2 = nullptr;
  double* qr_wfin = nullptr;
  int qr_count = 0;
  double* chol_rs = nullptr;  // Cholesky running row checksums of future panels (n x nb)
  bool chol_rs_valid = false;
  bool want_chol_rs = false;
  double* uwd = nullptr;  // widened right operand (b x n)
  // fp32 workspaces
  float* lw = nullptr;    // n x b
  float* uw = nullptr;    // b x n
  float* linv = nullptr;
  float* uinv = nullptr;
  float* sws = nullptr;   // sgemm split-operand workspace
  int64_t sws_elems = 0;
  int sms = 148;
  // Cholesky: finished L columns kept pre-split for the tensor cores
  // (lsh/lsl[r * ldk + c] = hi/lo of L(r, c)), written once per panel, so
  // the left-looking update reads both operands with no per-iteration split
  float* lsh = nullptr;
  float* lsl = nullptr;
  int64_t ldk = 0;
  double* scratch = nullptr;
  GemmWorkspace gws;
  GemmWorkspace gws2;           // fp64 split-K workspace of the side-stream QR panel
  Event* ev = nullptr;
  int32_t* counters = nullptr;
  int ev_cap = 0;
  int32_t* dirty = nullptr;
  int dirty_cap = 0;
  DevFault* dplan = nullptr;
  int dplan_cap = 0;
  int32_t* dlist = nullptr;
  int dlist_cap = 0;
  int* info = nullptr;
  float* out_host = nullptr;  // streamed result (abft_s_stream_out)
  int64_t out_ld = 0;
  cudaStream_t st_out = nullptr;
  cudaEvent_t ev_out = nullptr;
  // streamed input (abft_s_set_matrix_streamed, as ctx.cu): block columns
  // copied on st_in inside the next abft_s_factorize call
  const float* in_host = nullptr;
  int64_t in_ld = 0;
  bool in_stream = false;
  cudaStream_t st_in = nullptr;
  std::vector<cudaEvent_t> ev_in;
  std::vector<char> rs_enc;
  double* rs_tmp = nullptr;
  // device snapshot slot (replaces _Run._snapshot/_restore, simulator.py:420-436)
  float* snap_m = nullptr;
  double* snap_rs = nullptr;
  bool snap_used = false, snap_rs_valid = false;
  int64_t snap_k = 0;
  int snap_qr = 0;
  int64_t el_for = -1;  // iteration whose operand sums E_L / R E_R came out of the
  int64_t er_for = -1;  // PD / PU GEMM epilogues (no separate checksum pass)
  int64_t k_done = 0;
  bool sums_valid = false;
  int64_t breakdown_col = -1;
  bool fuse_enabled = true;
  bool lookahead_enabled = true;  // ABFT_NO_LOOKAHEAD=1 disables
  int64_t pd_ready = -1;          // panel already factored by the look-ahead
  // streamed LU input (as ctx.cu's lu_stream_chunks): the left `lu_split`
  // block columns are factored chunk by chunk as they arrive
  int lu_chunk = -1;              // ABFT_STREAM_CHUNK (0: wait for all; -1: nb / 4)
  int64_t lu_split = -1;          // ABFT_STREAM_SPLIT (-1: nb / 4)
  int lu_rchunk = -1;             // right part's pieces (0: at once; -1: LU 0, QR nb / 8)
  float* linv_store = nullptr;    // nb x (ld_t x b): L11^{-1} of every panel
  double* el_store = nullptr;     // nb x (ld_cs x b): E_L of every panel
  std::vector<char> el_ok;        // QR windows: E_L of panel k already in el_store
  int64_t chol_part = -1;         // Cholesky: panel already updated by panels 0..k-2
  bool chol_enc_ahead = false;    // ... and encoded before that update
  int next_scheme = 0;            // scheme of the next iteration (abft_s_factorize)
  cudaStream_t st2 = nullptr;     // side stream for the look-ahead diagonal block
  cudaEvent_t ev_a = nullptr, ev_p = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool timed = false;
  bool prof_on = false;
  double prof_ms[4] = {0, 0, 0, 0};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_pending;
  cudaEvent_t prof_open[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

void smark(abft_sctx* c, int cat, bool begin) {
  if (!c->prof_on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, c->st);
  if (begin) {
    c->prof_open[cat] = e;
  } else {
    c->prof_pending.push_back({cat, {c->prof_open[cat], e}});
    c->prof_open[cat] = nullptr;
  }
}

void s_region(const abft_sctx* c, int64_t k, int64_t* r0, int64_t* c0, int64_t* rows, int64_t* cols) {
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
// its device-to-host copy on the copy stream (as ctx.cu).
// LU / Cholesky emit row block k after PU(k), QR after TMU(k) (s_emit_rowblock,
// as ctx.cu), so a column block carries only rows >= k b.
int s_emit_column(abft_sctx* c, int64_t k) {
  if (!c->out_host) return 0;
  const int64_t p = k * c->b, w = std::min(c->b, c->n - p);
  const int64_t r0 = p;
  CUDA_TRY(cudaEventRecord(c->ev_out, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st_out, c->ev_out, 0));
  CUDA_TRY(cudaMemcpy2DAsync(c->out_host + r0 + p * c->out_ld, c->out_ld * 4, c->m + r0 + p * c->ld,
                             c->ld * 4, (c->n - r0) * 4, w, cudaMemcpyDeviceToHost, c->st_out));
  return 0;
}

// LU: row block k of U over columns [cs, ce) is final after PU(k).
int s_emit_rowblock(abft_sctx* c, int64_t k, int64_t cs, int64_t ce) {
  if (!c->out_host) return 0;  // LU: U rows; Cholesky: zeroed rows; QR: R rows after TMU(k)
  const int64_t p = k * c->b, pe = std::min(p + c->b, c->n), w = pe - p;
  cs = std::max(cs, pe);
  ce = std::min(ce, c->n);
  if (cs >= ce) return 0;
  CUDA_TRY(cudaEventRecord(c->ev_out, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st_out, c->ev_out, 0));
  CUDA_TRY(cudaMemcpy2DAsync(c->out_host + p + cs * c->out_ld, c->out_ld * 4, c->m + p + cs * c->ld,
                             c->ld * 4, w * 4, ce - cs, cudaMemcpyDeviceToHost, c->st_out));
  return 0;
}

SumOut s_sums(abft_sctx* c, int64_t r0, int64_t c0, bool rows_too) {
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

// Long reductions are split into K chunks of at most S_KCHUNK, accumulated
// in fp32 through the epilogue (beta = 1): the tensor core's internal
// accumulation of a single long-K MMA chain loses precision roughly linearly
// in K (measured: QR residual ~2e-8 * n with K = n - p), so chunking keeps
// every product fp32-accurate.
constexpr int64_t S_KCHUNK = 512;
// Cholesky's left-looking panel update (K = p, output n-p x b) issues one
// launch per chunk; a deeper chunk keeps it launch-cheap (accuracy measured:
// residual 2.4e-7 at N = 16384)
constexpr int64_t S_KCHUNK_CHOL = 2048;

// Split-K plan of one s_gemm. Narrow outputs with deep K (Cholesky's
// left-looking panel update, QR's V^T C: fewer tiles than SMs) run as one
// split-K launch -- at least ceil(K / kchunk) slices for the chain-depth
// bound, more for parallelism (up to two units per SM). Wide outputs, and
// GEMMs whose epilogue produces the checksums, run the K chunks as
// sequential launches accumulating through beta = 1 (no partial buffers).
void s_gemm_plan(int sms, int64_t M, int64_t N, int64_t K, int64_t kchunk, bool fused, int* splits,
                 int64_t* need) {
  const int64_t tiles = ((M + 127) / 128) * ((N + 127) / 128);
  int64_t S = (K + kchunk - 1) / kchunk;
  if (fused || tiles >= sms) {
    *splits = 1;
    *need = sgemm_workspace_elems((int)M, (int)N, (int)std::min(K, kchunk), 1);
    return;
  }
  // wave model (as gemm_splits_for): units run round-robin over the SMs,
  // each costs its K-slice plus a fixed ~128-deep prologue/epilogue, and
  // every slice adds a partial write + read-back
  const int64_t s_min = std::max<int64_t>(S, 1), s_max = std::max<int64_t>(s_min, std::min<int64_t>(64, K / 128));
  double best_t = 0.0;
  int64_t best = s_min;
  for (int64_t sc = s_min; sc <= s_max; ++sc) {
    const int64_t kps = ((K + sc - 1) / sc + 31) / 32 * 32;
    if ((K + kps - 1) / kps != sc) continue;
    const int64_t waves = (tiles * sc + sms - 1) / sms;
    // seconds: one 128 x 128 x 32 3xTF32 k-block ~ 0.4 us per SM
    double t = (double)waves * ((double)kps / 32.0 + 4.0) * 0.4e-6;
    if (sc > 1) t += (double)sc * M * N * 8.0 / 6.0e12 + 4e-6;
    if (sc == s_min || t < 0.98 * best_t) {
      best = sc;
      best_t = t;
    }
  }
  *splits = (int)best;
  *need = sgemm_workspace_elems((int)M, (int)N, (int)K, *splits);
}

int s_gemm(abft_sctx* c, char ta, char tb, int64_t M, int64_t N, int64_t K, float alpha,
           const float* A, int64_t lda, const float* B, int64_t ldb, float beta, const float* C,
           int64_t ldc, float* D, int64_t ldd, const FusedSums* fs = nullptr, int max_ctas = 0,
           int64_t kchunk = S_KCHUNK, int force_splits = 0) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  int splits;
  int64_t need;
  s_gemm_plan(max_ctas > 0 ? std::min(max_ctas, c->sms) : c->sms, M, N, K, kchunk, fs != nullptr,
              &splits, &need);
  if (force_splits > 0 && !fs) {  // a column window of a wider product: its K partition
    splits = force_splits;
    need = sgemm_workspace_elems((int)M, (int)N, (int)(splits > 1 ? K : std::min(K, kchunk)), splits);
  }
  if (need > c->sws_elems) {
    CUDA_TRY(cudaStreamSynchronize(c->st));
    if (c->sws) cudaFree(c->sws);
    c->sws = nullptr;
    c->sws_elems = need + need / 4;
    CUDA_TRY(cudaMalloc(&c->sws, c->sws_elems * sizeof(float)));
  }
  if (splits > 1 || K <= kchunk)
    return sgemm_tc(c->st, ta, tb, (int)M, (int)N, (int)K, alpha, A, lda, B, ldb, beta, C, ldc, D,
                    ldd, c->sws, c->sws_elems, fs, max_ctas, splits);
  const bool AT = (ta == 'T' || ta == 't'), BT = (tb == 'T' || tb == 't');
  for (int64_t k0 = 0; k0 < K; k0 += kchunk) {
    const int64_t kl = std::min(kchunk, K - k0);
    const float* Ak = AT ? A + k0 : A + k0 * lda;
    const float* Bk = BT ? B + k0 * ldb : B + k0;
    const bool first = k0 == 0, last = k0 + kl >= K;
    ABFT_TRY(sgemm_tc(c->st, ta, tb, (int)M, (int)N, (int)kl, alpha, Ak, lda, Bk, ldb,
                      first ? beta : 1.0f, first ? C : D, first ? ldc : ldd, D, ldd, c->sws,
                      c->sws_elems, last ? fs : nullptr, max_ctas));
  }
  return 0;
}

// Cholesky left-looking panel update P(p:n, p:pe) -= L(p:n, K0:K1) L(p:pe, K0:K1)^T
// from the cached operand splits (split-K, one launch + reduction), on `st`.
// K0:K1 = 0:p normally; the look-ahead applies 0:p-b on the side stream
// and leaves p-b:p (the newest panel) to the main stream.
int s_chol_update(abft_sctx* c, cudaStream_t st, int64_t k, int64_t K0, int64_t K1, int max_ctas) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  const int64_t K = K1 - K0;
  if (K <= 0) return 0;
  int splits;
  int64_t need;
  s_gemm_plan(max_ctas > 0 ? std::min(max_ctas, c->sms) : c->sms, n - p, w, K, S_KCHUNK_CHOL, false,
              &splits, &need);
  need = sgemm_partial_elems((int)(n - p), (int)w, splits) + 128;
  if (need > c->sws_elems) {
    CUDA_TRY(cudaDeviceSynchronize());
    if (c->sws) cudaFree(c->sws);
    c->sws = nullptr;
    c->sws_elems = need;
    CUDA_TRY(cudaMalloc(&c->sws, c->sws_elems * sizeof(float)));
  }
  float* P = c->m + p + p * c->ld;
  const float* ah = c->lsh + p * c->ldk + K0;
  const float* al = c->lsl + p * c->ldk + K0;
  if (splits > 1)
    return sgemm_tc_presplit(st, (int)(n - p), (int)w, (int)K, -1.0f, ah, al, c->ldk, ah, al, c->ldk,
                             1.0f, P, c->ld, P, c->ld, c->sws, c->sws_elems, max_ctas, splits);
  // wide enough for the SMs: the chain-depth bound runs as sequential
  // K chunks accumulating through beta = 1
  for (int64_t k0 = 0; k0 < K; k0 += S_KCHUNK_CHOL) {
    const int64_t kl = std::min<int64_t>(S_KCHUNK_CHOL, K - k0);
    ABFT_TRY(sgemm_tc_presplit(st, (int)(n - p), (int)w, (int)kl, -1.0f, ah + k0, al + k0, c->ldk,
                               ah + k0, al + k0, c->ldk, 1.0f, P, c->ld, P, c->ld, nullptr, 0, max_ctas,
                               1));
  }
  return 0;
}

// Streamed input: the stream waits until column block j has arrived.
int s_wait_in(abft_sctx* c, cudaStream_t st, int64_t j) {
  if (!c->in_stream || j < 0 || j >= c->nb) return 0;
  CUDA_TRY(cudaStreamWaitEvent(st, c->ev_in[j], 0));
  return 0;
}

// Streamed Cholesky FULL (as ctx.cu chol_rs_encode_col): block column j's
// row sums join chol_rs (zeroed at k = 0, panel updates already applied)
// before anything modifies its rows >= j b.
int s_chol_rs_encode_col(abft_sctx* c, cudaStream_t st, int64_t j) {
  if (!c->in_stream || !c->chol_rs_valid || j >= c->nb || c->rs_enc[j]) return 0;
  const int64_t n = c->n, p = j * c->b, w = std::min(c->b, n - p);
  RegionF reg{c->m + p + p * c->ld, c->ld, n - p, w, c->b};
  SumOut o;
  o.rp = c->rs_tmp;
  o.rp_ld = c->ld;
  ABFT_TRY(blocksum(st, reg, o));
  ABFT_TRY(add_matrix(st, c->rs_tmp, c->ld, c->chol_rs + p + j * c->ld, c->ld, n - p, 1));
  c->rs_enc[j] = 1;
  return 0;
}

// Cholesky look-ahead (as ctx.cu): right after TMU(k) the update of panel
// k+1 by panels 0..k-1 -- final since their PU -- runs on the side stream
// (encode of panel k+1 first, when its iteration is protected) while the
// main stream factors panel k; TMU(k+1) then applies panel k alone.
// (chol_cluster: the caller records ev_a after TMU(k) and submits the cluster
// PD(k) first, as ctx.cu's chol_lookahead)
int s_chol_lookahead(abft_sctx* c, int64_t k, int scheme_next, bool ev_recorded = false) {
  const int64_t n = c->n, pk = k * c->b, p1 = (k + 1) * c->b;
  const int64_t pe1 = std::min(p1 + c->b, n), w1 = pe1 - p1;
  if (!ev_recorded) CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
  ABFT_TRY(s_wait_in(c, c->st2, k + 1));
  ABFT_TRY(s_chol_rs_encode_col(c, c->st2, k + 1));
  c->chol_enc_ahead = false;
  if (scheme_next != ABFT_NONE) {
    RegionF reg1{c->m + p1 + p1 * c->ld, c->ld, n - p1, w1, c->b};
    ABFT_TRY(blocksum(c->st2, reg1, s_sums(c, p1, p1, true)));
    c->chol_enc_ahead = true;
  }
  const int keep = c->chol_cluster ? (int)((c->b + 31) / 32) : 1;
  ABFT_TRY(s_chol_update(c, c->st2, k + 1, 0, pk, c->sms - keep));
  CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  c->chol_part = k + 1;
  return 0;
}

int s_check_info(abft_sctx* c) {
  int h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, c->info, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  if (h != 0) {
    c->breakdown_col = h - 1;
    set_last_error(c->kind == ABFT_CHOLESKY ? "non-positive pivot at column %lld"
                                            : "zero pivot at column %lld",
                   (long long)c->breakdown_col);
    CUDA_TRY(cudaMemsetAsync(c->info, 0, sizeof(int), c->st));
    return ABFT_E_BREAKDOWN;
  }
  return 0;
}

// ---- tasks -------------------------------------------------------------------
int s_lu_diag(abft_sctx* c, cudaStream_t st, int64_t k) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  if (c->lu_coop)
    return diag_factor_fast(st, c->m + p + p * c->ld, c->ld, (int)w, 0, c->linv, c->ld_t, c->uinv,
                            c->ld_t, c->info, p);
  return diag_factor(st, c->m + p + p * c->ld, c->ld, (int)w, 0, c->linv, c->ld_t, c->uinv, c->ld_t,
                     c->info, p);
}

int s_lu_l21(abft_sctx* c, int64_t k) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  if (pe >= n) return 0;
  float* D = c->m + p + p * c->ld;
  // b = 128: the GEMM epilogue also emits the block column sums of L21 =
  // the operand sums E_L of the maintenance of iteration k (abft.py:147-152)
  FusedSums fs;
  const bool fuse = c->fuse_enabled && c->b == 128 && w == 128;
  if (fuse) {
    fs.cp = c->el;
    fs.cp_ld = c->ld_cs;
    fs.cp_step = 2;
    fs.cw = c->el + 1;
    fs.cw_ld = c->ld_cs;
    fs.cw_step = 2;
    fs.rp = c->lwd;  // row sums / maxima are not needed: scratch
    fs.rp_ld = c->ld;
    fs.bm = c->scratch;
    fs.bm_ld = 1;
  }
  // in place: sgemm_tc splits A (= the output block) into its workspace
  // before the tensor-core launch reads anything, so D may alias A
  ABFT_TRY(s_gemm(c, 'N', 'N', n - pe, w, w, 1.0f, D + w, c->ld, c->uinv, c->ld_t, 0.0f, nullptr, 0,
                  D + w, c->ld, fuse ? &fs : nullptr));
  c->el_for = fuse ? k : -1;
  return 0;
}

// Mixed-precision Householder panel k on stream st: widen, factor in fp64
// (qr_panel_factor: tensor-core path + exact fallback; GEMMs capped at
// max_ctas), narrow back into the fp32 matrix / V / T stores.
int s_qr_panel(abft_sctx* c, cudaStream_t st, int64_t k, int max_ctas, GemmWorkspace* gws) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  float* D = c->m + p + p * c->ld;
  const int64_t nk = n - p;
  ABFT_TRY(widen_matrix(st, D, c->ld, c->pan64, c->ld, nk, w));
  ABFT_TRY(fill_matrix(st, c->v64, c->ld, nk, w, 0.0));
  QrPanelWork q = c->qrw;
  q.gws = gws;
  ABFT_TRY(qr_panel_factor(st, c->pan64, c->ld, nk, (int)w, c->v64, c->ld, c->t64, c->ld_t,
                           c->betas, q, max_ctas));
  ABFT_TRY(narrow_matrix(st, c->pan64, c->ld, D, c->ld, nk, w));
  ABFT_TRY(narrow_matrix(st, c->v64, c->ld, c->vstore + p + p * c->ld, c->ld, nk, w));
  return narrow_matrix(st, c->t64, c->ld_t, c->tstore + k * c->b * c->ld_t, c->ld_t, w, w);
}

int s_pd(abft_sctx* c, int64_t k) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  float* D = c->m + p + p * c->ld;
  if (c->kind == ABFT_LU) {
    ABFT_TRY(s_lu_diag(c, c->st, k));
    ABFT_TRY(s_lu_l21(c, k));
  } else if (c->kind == ABFT_CHOLESKY) {
    if (c->chol_cluster)
      ABFT_TRY(diag_factor_fast(c->st, D, c->ld, (int)w, 1, c->linv, c->ld_t, nullptr, 0, c->info, p));
    else
      ABFT_TRY(diag_factor(c->st, D, c->ld, (int)w, 1, c->linv, c->ld_t, nullptr, 0, c->info, p));
  } else {
    ABFT_TRY(s_qr_panel(c, c->st, k, 0, &c->gws));
    c->qr_count = (int)(k + 1);
  }
  return 0;
}

int s_pu(abft_sctx* c, int64_t k) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  if (c->kind == ABFT_LU) {
    if (pe < n) {
      float* U12 = c->m + p + pe * c->ld;
      // b = 128: the epilogue also emits the block row sums of U12 = R E_R
      FusedSums fs;
      const bool fuse = c->fuse_enabled && c->b == 128 && w == 128;
      if (fuse) {
        fs.cp = c->uwd;  // column sums are not needed: scratch
        fs.cp_ld = c->ld_t;
        fs.cp_step = 1;
        fs.cw = c->uwd + 1;
        fs.cw_ld = c->ld_t;
        fs.cw_step = 1;
        fs.rp = c->er;
        fs.rp_ld = c->ld_t;
        fs.bm = c->scratch + 2048;
        fs.bm_ld = 1;
      }
      ABFT_TRY(s_gemm(c, 'N', 'N', w, n - pe, w, 1.0f, c->linv, c->ld_t, U12, c->ld, 0.0f, nullptr, 0,
                      c->uw, c->ld_t, fuse ? &fs : nullptr));
      c->er_for = fuse ? k : -1;
      ABFT_TRY(copy_matrix(c->st, c->uw, c->ld_t, U12, c->ld, w, n - pe));
    }
  } else {
    if (pe < n) {
      float* A21 = c->m + pe + p * c->ld;
      // in place (A is split into the workspace before the launch, as s_lu_l21)
      ABFT_TRY(s_gemm(c, 'N', 'T', n - pe, w, w, 1.0f, A21, c->ld, c->linv, c->ld_t, 0.0f, nullptr, 0,
                      A21, c->ld));
      ABFT_TRY(fill_matrix(c->st, c->m + p + pe * c->ld, c->ld, w, n - pe, 0.0));
    }
    // panel k is final: keep its hi/lo split for the later panel updates
    if (c->lsh) ABFT_TRY(sgemm_split_operand(c->st, c->m + p + p * c->ld, c->ld, (int)(n - p), (int)w, (int)w, 0,
                                 c->lsh + p * c->ldk + p, c->lsl + p * c->ldk + p, c->ldk));
    // block-row sums of the finished panel: operand sums of later maintenance
    RegionF reg{c->m + p + p * c->ld, c->ld, n - p, w, c->b};
    SumOut o = s_sums(c, p, p, false);
    o.bm = nullptr;
    ABFT_TRY(blocksum(c->st, reg, o));
    // chol_rs[pe:n, j] -= L_k[pe:n, :] (1^T L_k[block j, :])^T for j > k
    const int64_t nj = c->nb - (k + 1);
    if (c->chol_rs_valid && nj > 0 && pe < n) {
      ABFT_TRY(gather_transpose(c->st, c->gcsw + 2 * (k + 1) + p * c->ld_cs, 2, c->ld_cs, nj, w, c->er,
                                c->ld_t));
      ABFT_TRY(widen_matrix(c->st, c->m + pe + p * c->ld, c->ld, c->lwd, c->ld, n - pe, w));
      ABFT_TRY(gemm(c->st, 'N', 'N', (int)(n - pe), (int)nj, (int)w, -1.0, c->lwd, c->ld, c->er,
                    c->ld_t, 1.0, c->chol_rs + pe + (k + 1) * c->ld, c->ld,
                    c->chol_rs + pe + (k + 1) * c->ld, c->ld, &c->gws));
    }
  }
  return 0;
}

// maintain_gemm (abft.py:138-158) in fp64 from widened operands.
int s_maintain(abft_sctx* c, int64_t k, int scheme, int64_t r0, int64_t c0, int64_t rows,
               int64_t cols) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  const int64_t nbr = (rows + c->b - 1) / c->b, nbc = (cols + c->b - 1) / c->b;
  SumOut enc = s_sums(c, r0, c0, scheme == ABFT_FULL);
  if (c->kind == ABFT_CHOLESKY) {
    // col: CSm = CS - GCSW[2k:, 0:p] * m[p:pe, 0:p]^T ; row: RSm = RS - L * rvec
    ABFT_TRY(widen_matrix(c->st, c->m + p, c->ld, c->uwd, c->ld_t, w, p));  // R^T rows (w x p)
    ABFT_TRY(gemm(c->st, 'N', 'T', (int)(2 * nbr), (int)w, (int)p, -1.0, c->gcsw + 2 * k, c->ld_cs,
                  c->uwd, c->ld_t, 1.0, enc.cp, c->ld_cs, c->csm, c->ld_cs, &c->gws));
    if (scheme == ABFT_FULL) {
      if (!c->chol_rs_valid) {
        set_last_error("fp32 Cholesky FULL checksums need FULL from the first iteration");
        return ABFT_E_INVALID;
      }
      // running right-looking maintenance (as ctx.cu): the panel's row
      // checksums already carry every earlier update
      ABFT_TRY(copy_matrix(c->st, c->chol_rs + p + k * c->ld, c->ld, c->rsm, c->ld, rows, nbc));
    }
    return 0;
  }
  const float* L = c->kind == ABFT_LU ? c->m + pe + p * c->ld : c->vstore + p + p * c->ld;
  const float* R = c->kind == ABFT_LU ? c->m + p + pe * c->ld : c->mid;
  const int64_t ldr = c->kind == ABFT_LU ? c->ld : c->ld_t;
  if (!(c->kind == ABFT_LU && c->el_for == k)) {
    RegionF rl{const_cast<float*>(L), c->ld, rows, w, c->b};
    SumOut o;
    o.cp = c->el;
    o.cp_ld = c->ld_cs;
    o.cp_step = 2;
    o.cw = c->el + 1;
    o.cw_ld = c->ld_cs;
    o.cw_step = 2;
    ABFT_TRY(blocksum(c->st, rl, o));
  }
  ABFT_TRY(widen_matrix(c->st, R, ldr, c->uwd, c->ld_t, w, cols));
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)(2 * nbr), (int)cols, (int)w, -1.0, c->el, c->ld_cs, c->uwd,
                c->ld_t, 1.0, enc.cp, c->ld_cs, c->csm, c->ld_cs, &c->gws));
  if (scheme == ABFT_FULL) {
    if (!(c->kind == ABFT_LU && c->er_for == k)) {
      RegionF rr{const_cast<float*>(R), ldr, w, cols, c->b};
      SumOut o;
      o.rp = c->er;
      o.rp_ld = c->ld_t;
      ABFT_TRY(blocksum(c->st, rr, o));
    }
    ABFT_TRY(widen_matrix(c->st, L, c->ld, c->lwd, c->ld, rows, w));
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)nbc, (int)w, -1.0, c->lwd, c->ld, c->er, c->ld_t,
                  1.0, enc.rp, c->ld, c->rsm, c->ld, &c->gws));
  }
  return 0;
}

int s_upload_plan(abft_sctx* c, const abft_fault* plan, int nplan) {
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
  CUDA_TRY(cudaMemcpyAsync(c->dplan, h.data(), nplan * sizeof(DevFault), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

int s_touched(abft_sctx* c, const abft_fault* plan, int nplan, int64_t r0, int64_t c0, int64_t rows,
              int64_t cols, int* count) {
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
    for (int64_t r = std::max(ft.row, r0); r < std::min(std::min(ft.row + er, c->n), r0 + rows); ++r)
      for (int64_t cc = std::max(ft.col, c0); cc < std::min(std::min(ft.col + ec, c->n), c0 + cols); ++cc)
        blks.emplace_back((int32_t)((r - r0) / c->b), (int32_t)((cc - c0) / c->b));
  }
  std::sort(blks.begin(), blks.end());
  blks.erase(std::unique(blks.begin(), blks.end()), blks.end());
  *count = (int)blks.size();
  if (blks.empty()) return 0;
  std::vector<int32_t> lst;
  for (auto& pr : blks) {
    lst.push_back(pr.first);
    lst.push_back(pr.second);
  }
  const int nn = (int)lst.size();
  if (nn > c->dlist_cap) {
    if (c->dlist) cudaFree(c->dlist);
    c->dlist_cap = std::max(nn, 1024);
    CUDA_TRY(cudaMalloc(&c->dlist, c->dlist_cap * sizeof(int32_t)));
  }
  CUDA_TRY(cudaMemcpyAsync(c->dlist, lst.data(), nn * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

FusedSums s_fused(abft_sctx* c, int64_t r0, int64_t c0) {
  const SumOut o = s_sums(c, r0, c0, true);
  FusedSums fs;
  fs.cp = o.cp;
  fs.cp_ld = o.cp_ld;
  fs.cp_step = o.cp_step;
  fs.cw = o.cw;
  fs.cw_ld = o.cw_ld;
  fs.cw_step = o.cw_step;
  fs.rp = o.rp;
  fs.rp_ld = o.rp_ld;
  fs.bm = o.bm;
  fs.bm_ld = o.bm_ld;
  return fs;
}

// _protected_tmu (simulator.py:124-167) in fp32 data / fp64 checksums.
int s_protected_tmu(abft_sctx* c, int64_t k, int scheme, const abft_fault* plan, int nplan,
                    int correct) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  s_region(c, k, &r0, &c0, &rows, &cols);
  const bool has = rows > 0 && cols > 0;
  const bool prot = scheme != ABFT_NONE && has;
  RegionF reg{c->m + r0 + c0 * c->ld, c->ld, rows, cols, c->b};
  bool fused = false;
  if (c->kind == ABFT_CHOLESKY && k == 0 && (scheme == ABFT_FULL || c->want_chol_rs)) {
    if (c->in_stream) {  // block columns add their row sums as they arrive
      CUDA_TRY(cudaMemsetAsync(c->chol_rs, 0, (size_t)c->ld * c->nb * sizeof(double), c->st));
    } else {
      RegionF all{c->m, c->ld, n, n, c->b};
      SumOut o;
      o.rp = c->chol_rs;
      o.rp_ld = c->ld;
      ABFT_TRY(blocksum(c->st, all, o));
    }
    c->chol_rs_valid = true;
  }
  if (c->kind == ABFT_CHOLESKY) ABFT_TRY(s_chol_rs_encode_col(c, c->st, k));
  const bool qr_live = c->kind == ABFT_QR && pe < n && k < c->qr_count;
  if (prot) {
    smark(c, SP_ABFT, true);
    const bool reuse = (c->sums_valid && c->kind != ABFT_CHOLESKY) ||
                       (c->kind == ABFT_CHOLESKY && c->chol_part == k && c->chol_enc_ahead);
    if (!reuse) ABFT_TRY(blocksum(c->st, reg, s_sums(c, r0, c0, true)));
    smark(c, SP_ABFT, false);
  }
  if (c->kind == ABFT_QR && qr_live) {
    // W = V^T C, mid = T^T W (maintenance needs mid)
    const float* V = c->vstore + p + p * c->ld;
    const float* T = c->tstore + k * c->b * c->ld_t;
    float* C = c->m + p + pe * c->ld;
    smark(c, SP_TMU, true);
    ABFT_TRY(s_gemm(c, 'T', 'N', w, n - pe, n - p, 1.0f, V, c->ld, C, c->ld, 0.0f, nullptr, 0, c->ww,
                    c->ld_t));
    ABFT_TRY(s_gemm(c, 'T', 'N', w, n - pe, w, 1.0f, T, c->ld_t, c->ww, c->ld_t, 0.0f, nullptr, 0,
                    c->mid, c->ld_t));
    smark(c, SP_TMU, false);
  }
  if (prot) {
    smark(c, SP_ABFT, true);
    if (c->kind != ABFT_QR || qr_live) {
      ABFT_TRY(s_maintain(c, k, scheme, r0, c0, rows, cols));
    } else {
      // no update: maintained == encoded
      SumOut enc = s_sums(c, r0, c0, true);
      const int64_t nbr = (rows + c->b - 1) / c->b, nbc = (cols + c->b - 1) / c->b;
      ABFT_TRY(copy_matrix(c->st, enc.cp, c->ld_cs, c->csm, c->ld_cs, 2 * nbr, cols));
      if (scheme == ABFT_FULL) ABFT_TRY(copy_matrix(c->st, enc.rp, c->ld, c->rsm, c->ld, rows, nbc));
    }
    smark(c, SP_ABFT, false);
  }
  smark(c, SP_TMU, true);
  if (c->kind == ABFT_QR) {
    if (qr_live) {
      const bool fuse = prot && c->fuse_enabled && c->b == 128;
      FusedSums fs;
      if (fuse) fs = s_fused(c, r0, c0);
      float* C = c->m + p + pe * c->ld;
      ABFT_TRY(s_gemm(c, 'N', 'N', n - p, n - pe, w, -1.0f, c->vstore + p + p * c->ld, c->ld, c->mid,
                      c->ld_t, 1.0f, C, c->ld, C, c->ld, fuse ? &fs : nullptr));
      fused = fuse;
    }
  } else if (c->kind == ABFT_LU) {
    if (pe < n) {
      FusedSums fs;
      const bool fuse = prot && c->fuse_enabled && c->b == 128;
      if (fuse) {
        const SumOut o = s_sums(c, r0, c0, true);
        fs.cp = o.cp;
        fs.cp_ld = o.cp_ld;
        fs.cp_step = o.cp_step;
        fs.cw = o.cw;
        fs.cw_ld = o.cw_ld;
        fs.cw_step = o.cw_step;
        fs.rp = o.rp;
        fs.rp_ld = o.rp_ld;
        fs.bm = o.bm;
        fs.bm_ld = o.bm_ld;
      }
      float* A22 = c->m + pe + pe * c->ld;
      ABFT_TRY(s_gemm(c, 'N', 'N', n - pe, n - pe, w, -1.0f, c->m + pe + p * c->ld, c->ld,
                      c->m + p + pe * c->ld, c->ld, 1.0f, A22, c->ld, A22, c->ld,
                      fuse ? &fs : nullptr));
      fused = fuse;
    }
  } else if (k > 0) {
    // after the look-ahead only the newest panel (k-1) is left
    ABFT_TRY(s_chol_update(c, c->st, k, c->chol_part == k ? p - c->b : 0, p, 0));
  }
  smark(c, SP_TMU, false);
  smark(c, SP_ABFT, true);
  const bool faults = has && nplan > 0;
  if (prot && !fused) {
    ABFT_TRY(blocksum(c->st, reg, s_sums(c, r0, c0, true)));
  } else if (!prot && faults) {
    SumOut o;
    o.bm = c->gmax + (r0 / c->b) + (c0 / c->b) * c->ld_max;
    o.bm_ld = c->ld_max;
    ABFT_TRY(blocksum(c->st, reg, o));
  }
  if (faults) {
    for (int f = 0; f < nplan; ++f)
      if (plan[f].row < 0 || plan[f].row >= n || plan[f].col < 0 || plan[f].col >= n) {
        set_last_error("fault at (%lld, %lld) outside matrix", (long long)plan[f].row,
                       (long long)plan[f].col);
        return ABFT_E_RANGE;
      }
    ABFT_TRY(s_upload_plan(c, plan, nplan));
    const int64_t nbr = (rows + c->b - 1) / c->b, nbc = (cols + c->b - 1) / c->b;
    ABFT_TRY(inject(c->st, c->m, c->ld, n, n, c->dplan, nplan,
                    c->gmax + (r0 / c->b) + (c0 / c->b) * c->ld_max, nbr, nbc, c->ld_max, 0.0));
    if (prot) {
      int cnt = 0;
      ABFT_TRY(s_touched(c, plan, nplan, r0, c0, rows, cols, &cnt));
      if (cnt > 0) ABFT_TRY(blocksum(c->st, reg, s_sums(c, r0, c0, true), c->dlist, nullptr, cnt));
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
    EventSink sink{c->ev, c->counters, c->ev_cap, c->dirty, c->counters + 1, c->dirty_cap, (int32_t)k};
    ABFT_TRY(verify_blocks(c->st, reg, c->b, scheme, correct, s_sums(c, r0, c0, true), mt, sink));
    ABFT_TRY(blocksum(c->st, reg, s_sums(c, r0, c0, true), c->dirty, c->counters + 1, c->dirty_cap));
    CUDA_TRY(cudaMemsetAsync(c->counters + 1, 0, sizeof(int32_t), c->st));
  }
  c->sums_valid = prot;
  smark(c, SP_ABFT, false);
  if (c->chol_part == k) {
    c->chol_part = -1;
    c->chol_enc_ahead = false;
  }
  if (c->kind == ABFT_QR) ABFT_TRY(s_emit_rowblock(c, k, 0, n));
  return 0;
}


// Verify (and refresh after repairs) block columns [j0, j0 + ncb) of the
// region of iteration k, with event coordinates relative to the region.
int s_verify_sub(abft_sctx* c, int64_t k, int scheme, int correct, int64_t r0, int64_t c0,
                 int64_t rows, int64_t cols, int64_t j0, int64_t ncb) {
  const int64_t cbeg = j0 * c->b;
  const int64_t csub = std::min(cols - cbeg, ncb * c->b);
  if (csub <= 0 || rows <= 0) return 0;
  RegionF sub{c->m + r0 + (c0 + cbeg) * c->ld, c->ld, rows, csub, c->b};
  SumOut rec = s_sums(c, r0, c0 + cbeg, true);
  Maintained mt;
  mt.cp = c->csm + cbeg * c->ld_cs;
  mt.cp_ld = c->ld_cs;
  mt.cp_step = 2;
  mt.cw = mt.cp + 1;
  mt.cw_ld = c->ld_cs;
  mt.cw_step = 2;
  mt.rp = c->rsm + j0 * c->ld;
  mt.rp_ld = c->ld;
  EventSink sink{c->ev,          c->counters,  c->ev_cap, c->dirty, c->counters + 1,
                 c->dirty_cap,   (int32_t)k,   (int32_t)j0, c->b};
  ABFT_TRY(verify_blocks(c->st, sub, c->b, scheme, correct, rec, mt, sink));
  ABFT_TRY(blocksum(c->st, sub, rec, c->dirty, c->counters + 1, c->dirty_cap));
  CUDA_TRY(cudaMemsetAsync(c->counters + 1, 0, sizeof(int32_t), c->st));
  return 0;
}

// LU trailing update with look-ahead (fault-free iterations of the one-call
// path, as ctx.cu): the next panel's block column is updated and verified
// first, its diagonal block is factored on a side stream while the rest of
// the trailing matrix updates on the remaining SMs.
// fp32 QR look-ahead (fault-free iterations of the one-call path), ctx.cu's
// protected_tmu_qr_lookahead restated: W = V^T C, mid = T^T W and the
// maintained sums over the whole region; the next panel's block column
// first (plain GEMM + checksum pass + verify); panel k+1 (widen, tensor-core
// fp64 panel on qr_la_sms SMs, narrow) on the side stream; the rest of the
// region with fused sums on the other SMs.
int s_tmu_qr_lookahead(abft_sctx* c, int64_t k, int scheme, int correct) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  s_region(c, k, &r0, &c0, &rows, &cols);
  RegionF reg{c->m + r0 + c0 * c->ld, c->ld, rows, cols, c->b};
  const bool prot = scheme != ABFT_NONE;
  const float* V = c->vstore + p + p * c->ld;
  const float* T = c->tstore + k * c->b * c->ld_t;
  float* C = c->m + p + pe * c->ld;
  if (prot && !c->sums_valid) {
    smark(c, SP_ABFT, true);
    ABFT_TRY(blocksum(c->st, reg, s_sums(c, r0, c0, true)));
    smark(c, SP_ABFT, false);
  }
  smark(c, SP_TMU, true);
  ABFT_TRY(s_gemm(c, 'T', 'N', w, cols, rows, 1.0f, V, c->ld, C, c->ld, 0.0f, nullptr, 0, c->ww,
                  c->ld_t));
  ABFT_TRY(s_gemm(c, 'T', 'N', w, cols, w, 1.0f, T, c->ld_t, c->ww, c->ld_t, 0.0f, nullptr, 0, c->mid,
                  c->ld_t));
  smark(c, SP_TMU, false);
  if (prot) {
    smark(c, SP_ABFT, true);
    ABFT_TRY(s_maintain(c, k, scheme, r0, c0, rows, cols));
    smark(c, SP_ABFT, false);
  }
  const int64_t wa = std::min<int64_t>(c->b, cols);
  smark(c, SP_TMU, true);
  ABFT_TRY(s_gemm(c, 'N', 'N', rows, wa, w, -1.0f, V, c->ld, c->mid, c->ld_t, 1.0f, C, c->ld, C,
                  c->ld));
  smark(c, SP_TMU, false);
  if (prot) {
    smark(c, SP_ABFT, true);
    RegionF ra{C, c->ld, rows, wa, c->b};
    ABFT_TRY(blocksum(c->st, ra, s_sums(c, r0, c0, true)));
    ABFT_TRY(s_verify_sub(c, k, scheme, correct, r0, c0, rows, cols, 0, 1));
    smark(c, SP_ABFT, false);
  }
  const int res = std::max(8, std::min(c->qr_la_sms, c->sms / 2));
  CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
  ABFT_TRY(s_qr_panel(c, c->st2, k + 1, res, &c->gws2));
  CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  if (cols > wa) {
    const float* midb = c->mid + wa * c->ld_t;
    float* Cb = C + wa * c->ld;
    const bool fuse = prot && c->fuse_enabled && c->b == 128;
    FusedSums fs;
    if (fuse) fs = s_fused(c, r0, c0 + wa);
    smark(c, SP_TMU, true);
    ABFT_TRY(s_gemm(c, 'N', 'N', rows, cols - wa, w, -1.0f, V, c->ld, midb, c->ld_t, 1.0f, Cb, c->ld,
                    Cb, c->ld, fuse ? &fs : nullptr, c->sms - res));
    smark(c, SP_TMU, false);
    if (prot) {
      smark(c, SP_ABFT, true);
      if (!fuse) {
        RegionF rb{Cb, c->ld, rows, cols - wa, c->b};
        ABFT_TRY(blocksum(c->st, rb, s_sums(c, r0, c0 + wa, true)));
      }
      ABFT_TRY(s_verify_sub(c, k, scheme, correct, r0, c0, rows, cols, 1, (cols + c->b - 1) / c->b));
      smark(c, SP_ABFT, false);
    }
  }
  c->sums_valid = prot;
  ABFT_TRY(s_emit_rowblock(c, k, 0, n));
  CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
  c->qr_count = (int)(k + 2);
  ABFT_TRY(s_emit_column(c, k + 1));
  c->pd_ready = k + 1;
  return 0;
}

int s_tmu_lu_lookahead(abft_sctx* c, int64_t k, int scheme, int correct) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  s_region(c, k, &r0, &c0, &rows, &cols);
  RegionF reg{c->m + r0 + c0 * c->ld, c->ld, rows, cols, c->b};
  const bool prot = scheme != ABFT_NONE;
  if (prot) {
    smark(c, SP_ABFT, true);
    if (!c->sums_valid) ABFT_TRY(blocksum(c->st, reg, s_sums(c, r0, c0, true)));
    ABFT_TRY(s_maintain(c, k, scheme, r0, c0, rows, cols));
    smark(c, SP_ABFT, false);
  }
  const float* L21 = c->m + pe + p * c->ld;
  const float* U12 = c->m + p + pe * c->ld;
  float* A22 = c->m + pe + pe * c->ld;
  const int64_t wa = std::min<int64_t>(c->b, cols);
  const bool fuse_a = prot && c->fuse_enabled && c->b == 128;
  FusedSums fsa;
  if (fuse_a) fsa = s_fused(c, r0, c0);
  smark(c, SP_TMU, true);
  ABFT_TRY(s_gemm(c, 'N', 'N', rows, wa, w, -1.0f, L21, c->ld, U12, c->ld, 1.0f, A22, c->ld, A22,
                  c->ld, fuse_a ? &fsa : nullptr));
  smark(c, SP_TMU, false);
  if (prot) {
    smark(c, SP_ABFT, true);
    if (!fuse_a) {
      RegionF ra{A22, c->ld, rows, wa, c->b};
      ABFT_TRY(blocksum(c->st, ra, s_sums(c, r0, c0, true)));
    }
    ABFT_TRY(s_verify_sub(c, k, scheme, correct, r0, c0, rows, cols, 0, 1));
    smark(c, SP_ABFT, false);
  }
  CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
  CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
  ABFT_TRY(s_lu_diag(c, c->st2, k + 1));
  CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  if (cols > wa) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const bool fuse = prot && c->fuse_enabled && c->b == 128;
    FusedSums fs;
    if (fuse) fs = s_fused(c, r0, c0 + wa);
    smark(c, SP_TMU, true);
    ABFT_TRY(s_gemm(c, 'N', 'N', rows, cols - wa, w, -1.0f, L21, c->ld, U12 + wa * c->ld, c->ld, 1.0f,
                    A22 + wa * c->ld, c->ld, A22 + wa * c->ld, c->ld, fuse ? &fs : nullptr,
                    sms - (c->lu_coop ? (int)((c->b + 31) / 32) : 2)));
    smark(c, SP_TMU, false);
    if (prot) {
      smark(c, SP_ABFT, true);
      if (!fuse) {
        RegionF rb{A22 + wa * c->ld, c->ld, rows, cols - wa, c->b};
        ABFT_TRY(blocksum(c->st, rb, s_sums(c, r0, c0 + wa, true)));
      }
      ABFT_TRY(s_verify_sub(c, k, scheme, correct, r0, c0, rows, cols, 1, (cols + c->b - 1) / c->b));
      smark(c, SP_ABFT, false);
    }
  }
  c->sums_valid = prot;
  CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
  smark(c, SP_PD, true);
  ABFT_TRY(s_lu_l21(c, k + 1));
  smark(c, SP_PD, false);
  ABFT_TRY(s_emit_column(c, k + 1));
  c->pd_ready = k + 1;
  return 0;
}

// ---------------------------------------------------------------------------
// Streamed LU input, fp32 context: ctx.cu's lu_stream_chunks restated over
// s_pu / s_maintain / s_tmu_lu_lookahead restricted to block-column windows.
// Every block gets the same updates, operand sums (E_L from the L21
// epilogue, R E_R from the PU epilogue) and kernels as in the
// iteration-ordered schedule: factor and reports are bit-identical.

// PU(k) for region columns [cs, ce) with the kept L11^{-1}; R E_R from the epilogue.
int s_pu_win(abft_sctx* c, int64_t k, int64_t cs, int64_t ce) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  cs = std::max(cs, pe);
  if (cs >= ce) return 0;
  float* U12 = c->m + p + cs * c->ld;
  FusedSums fs;
  const bool fuse = c->fuse_enabled && c->b == 128 && w == 128;
  if (fuse) {
    fs.cp = c->uwd;  // column sums are not needed: scratch
    fs.cp_ld = c->ld_t;
    fs.cp_step = 1;
    fs.cw = c->uwd + 1;
    fs.cw_ld = c->ld_t;
    fs.cw_step = 1;
    fs.rp = c->er;
    fs.rp_ld = c->ld_t;
    fs.bm = c->scratch + 2048;
    fs.bm_ld = 1;
  }
  ABFT_TRY(s_gemm(c, 'N', 'N', w, ce - cs, w, 1.0f, c->linv_store + k * c->ld_t * c->b, c->ld_t,
                  U12, c->ld, 0.0f, nullptr, 0, c->uw, c->ld_t, fuse ? &fs : nullptr));
  c->er_for = fuse ? k : -1;
  ABFT_TRY(copy_matrix(c->st, c->uw, c->ld_t, U12, c->ld, w, ce - cs));
  return s_emit_rowblock(c, k, cs, ce);
}

// s_maintain of LU iteration k for region columns [cs, ce) (E_L kept per panel).
int s_maintain_win(abft_sctx* c, int64_t k, int scheme, int64_t r0, int64_t c0, int64_t rows,
                   int64_t cs, int64_t ce) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  const int64_t cw = ce - cs, cbeg = cs - c0, j0 = cbeg / c->b;
  const int64_t nbr = (rows + c->b - 1) / c->b, nbw = (cw + c->b - 1) / c->b;
  SumOut enc = s_sums(c, r0, cs, scheme == ABFT_FULL);
  const float* L = c->m + pe + p * c->ld;
  const float* R = c->m + p + cs * c->ld;
  const double* el = c->el_store + k * c->ld_cs * c->b;
  ABFT_TRY(widen_matrix(c->st, R, c->ld, c->uwd, c->ld_t, w, cw));
  ABFT_TRY(gemm(c->st, 'N', 'N', (int)(2 * nbr), (int)cw, (int)w, -1.0, el, c->ld_cs, c->uwd,
                c->ld_t, 1.0, enc.cp, c->ld_cs, c->csm + cbeg * c->ld_cs, c->ld_cs, &c->gws));
  if (scheme == ABFT_FULL) {
    if (c->er_for != k) {
      RegionF rr{const_cast<float*>(R), c->ld, w, cw, c->b};
      SumOut o;
      o.rp = c->er;
      o.rp_ld = c->ld_t;
      ABFT_TRY(blocksum(c->st, rr, o));
    }
    ABFT_TRY(widen_matrix(c->st, L, c->ld, c->lwd, c->ld, rows, w));
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)nbw, (int)w, -1.0, c->lwd, c->ld, c->er, c->ld_t,
                  1.0, enc.rp, c->ld, c->rsm + j0 * c->ld, c->ld, &c->gws));
  }
  return 0;
}

// Protected TMU(k) of LU for region columns [cs, ce); the look-ahead's
// kernels (s_tmu_lu_lookahead) when the window holds block column k+1.
int s_lu_tmu_win(abft_sctx* c, int64_t k, int scheme, int correct, int64_t cs, int64_t ce,
                 bool encode) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  s_region(c, k, &r0, &c0, &rows, &cols);
  cs = std::max(cs, c0);
  ce = std::min(ce, c0 + cols);
  if (cs >= ce || rows <= 0) return 0;
  const int64_t cw = ce - cs, j0 = (cs - c0) / c->b, ncb = (cw + c->b - 1) / c->b;
  const bool prot = scheme != ABFT_NONE;
  RegionF wreg{c->m + r0 + cs * c->ld, c->ld, rows, cw, c->b};
  const float* L21 = c->m + pe + p * c->ld;
  const float* U12 = c->m + p + cs * c->ld;
  float* A22 = c->m + r0 + cs * c->ld;
  if (prot) {
    smark(c, SP_ABFT, true);
    if (encode) ABFT_TRY(blocksum(c->st, wreg, s_sums(c, r0, cs, true)));
    ABFT_TRY(s_maintain_win(c, k, scheme, r0, c0, rows, cs, ce));
    smark(c, SP_ABFT, false);
  }
  const bool fuse = prot && c->fuse_enabled && c->b == 128;
  const bool la = c->lookahead_enabled && pe < n && cs == c0;
  const int64_t wa = la ? std::min<int64_t>(c->b, cw) : 0;
  if (la) {
    FusedSums fsa;
    if (fuse) fsa = s_fused(c, r0, cs);
    smark(c, SP_TMU, true);
    ABFT_TRY(s_gemm(c, 'N', 'N', rows, wa, w, -1.0f, L21, c->ld, U12, c->ld, 1.0f, A22, c->ld, A22,
                    c->ld, fuse ? &fsa : nullptr));
    smark(c, SP_TMU, false);
    if (prot) {
      smark(c, SP_ABFT, true);
      if (!fuse) {
        RegionF ra{A22, c->ld, rows, wa, c->b};
        ABFT_TRY(blocksum(c->st, ra, s_sums(c, r0, cs, true)));
      }
      ABFT_TRY(s_verify_sub(c, k, scheme, correct, r0, c0, rows, cols, 0, 1));
      smark(c, SP_ABFT, false);
    }
    CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
    CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
    ABFT_TRY(s_lu_diag(c, c->st2, k + 1));
    CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  }
  if (cw > wa) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    FusedSums fs;
    if (fuse) fs = s_fused(c, r0, cs + wa);
    smark(c, SP_TMU, true);
    ABFT_TRY(s_gemm(c, 'N', 'N', rows, cw - wa, w, -1.0f, L21, c->ld, U12 + wa * c->ld, c->ld,
                    1.0f, A22 + wa * c->ld, c->ld, A22 + wa * c->ld, c->ld, fuse ? &fs : nullptr,
                    la ? sms - (c->lu_coop ? (int)((c->b + 31) / 32) : 2) : 0));
    smark(c, SP_TMU, false);
    if (prot) {
      smark(c, SP_ABFT, true);
      if (!fuse) {
        RegionF rb{A22 + wa * c->ld, c->ld, rows, cw - wa, c->b};
        ABFT_TRY(blocksum(c->st, rb, s_sums(c, r0, cs + wa, true)));
      }
      ABFT_TRY(s_verify_sub(c, k, scheme, correct, r0, c0, rows, cols, j0 + (wa ? 1 : 0),
                            ncb - (wa ? 1 : 0)));
      smark(c, SP_ABFT, false);
    }
  }
  if (la) {
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
    smark(c, SP_PD, true);
    ABFT_TRY(s_lu_l21(c, k + 1));
    smark(c, SP_PD, false);
    ABFT_TRY(s_emit_column(c, k + 1));
    c->pd_ready = k + 1;
  }
  return 0;
}

// Defaults nb / 4 and nb / 4 (sgetrf N = 16384 b = 128 e2e: wait-for-all 82.5 ms,
// 32/32 77.9, 16/32 78.1, 12/24 79.6, 16/48 80.3, 16/16 81.1): the fp32
// iterations are launch-latency bound, so every extra window costs more
// than in fp64 and a short left part with few chunks wins.
// Protected TMU(k) of QR for region columns [cs, ce) (ctx.cu's qr_tmu_win in
// fp32): W = V^T C with the full product's K partition, mid = T^T W, the
// window's maintenance, C -= V mid with s_tmu_qr_lookahead's kernels when the
// window holds block column k+1.
int s_qr_tmu_win(abft_sctx* c, int64_t k, int scheme, int correct, int64_t cs, int64_t ce,
                 bool encode) {
  const int64_t n = c->n, p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
  int64_t r0, c0, rows, cols;
  s_region(c, k, &r0, &c0, &rows, &cols);
  cs = std::max(cs, c0);
  ce = std::min(ce, c0 + cols);
  if (cs >= ce || rows <= 0) return 0;
  const int64_t cw = ce - cs, cbeg = cs - c0, j0 = cbeg / c->b, ncb = (cw + c->b - 1) / c->b;
  const bool prot = scheme != ABFT_NONE;
  RegionF wreg{c->m + r0 + cs * c->ld, c->ld, rows, cw, c->b};
  const float* V = c->vstore + p + p * c->ld;
  const float* T = c->tstore + k * c->b * c->ld_t;
  float* C = c->m + p + cs * c->ld;
  if (prot && encode) {
    smark(c, SP_ABFT, true);
    ABFT_TRY(blocksum(c->st, wreg, s_sums(c, r0, cs, true)));
    smark(c, SP_ABFT, false);
  }
  int spl = 1, spl2 = 1;
  int64_t need = 0;
  s_gemm_plan(c->sms, w, cols, rows, S_KCHUNK, false, &spl, &need);
  s_gemm_plan(c->sms, w, cols, w, S_KCHUNK, false, &spl2, &need);
  smark(c, SP_TMU, true);
  ABFT_TRY(s_gemm(c, 'T', 'N', w, cw, rows, 1.0f, V, c->ld, C, c->ld, 0.0f, nullptr, 0, c->ww,
                  c->ld_t, nullptr, 0, S_KCHUNK, spl));
  ABFT_TRY(s_gemm(c, 'T', 'N', w, cw, w, 1.0f, T, c->ld_t, c->ww, c->ld_t, 0.0f, nullptr, 0, c->mid,
                  c->ld_t, nullptr, 0, S_KCHUNK, spl2));
  smark(c, SP_TMU, false);
  if (prot) {
    // s_maintain for the window (E_L of V kept per panel, R = mid)
    smark(c, SP_ABFT, true);
    const int64_t nbr = (rows + c->b - 1) / c->b;
    SumOut enc = s_sums(c, r0, cs, scheme == ABFT_FULL);
    double* el = c->el_store + k * c->ld_cs * c->b;
    if (!c->el_ok[k]) {
      RegionF rl{const_cast<float*>(V), c->ld, rows, w, c->b};
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
    ABFT_TRY(widen_matrix(c->st, c->mid, c->ld_t, c->uwd, c->ld_t, w, cw));
    ABFT_TRY(gemm(c->st, 'N', 'N', (int)(2 * nbr), (int)cw, (int)w, -1.0, el, c->ld_cs, c->uwd,
                  c->ld_t, 1.0, enc.cp, c->ld_cs, c->csm + cbeg * c->ld_cs, c->ld_cs, &c->gws));
    if (scheme == ABFT_FULL) {
      RegionF rr{c->mid, c->ld_t, w, cw, c->b};
      SumOut o;
      o.rp = c->er;
      o.rp_ld = c->ld_t;
      ABFT_TRY(blocksum(c->st, rr, o));
      ABFT_TRY(widen_matrix(c->st, V, c->ld, c->lwd, c->ld, rows, w));
      ABFT_TRY(gemm(c->st, 'N', 'N', (int)rows, (int)ncb, (int)w, -1.0, c->lwd, c->ld, c->er,
                    c->ld_t, 1.0, enc.rp, c->ld, c->rsm + j0 * c->ld, c->ld, &c->gws));
    }
    smark(c, SP_ABFT, false);
  }
  const bool fuse = prot && c->fuse_enabled && c->b == 128;
  const bool la = c->lookahead_enabled && pe < n && c->qr_la_sms > 0 && cs == c0;
  const int64_t wa = la ? std::min<int64_t>(c->b, cw) : 0;
  const int res = std::max(8, std::min(c->qr_la_sms, c->sms / 2));
  if (la) {
    smark(c, SP_TMU, true);
    ABFT_TRY(s_gemm(c, 'N', 'N', rows, wa, w, -1.0f, V, c->ld, c->mid, c->ld_t, 1.0f, C, c->ld, C,
                    c->ld));
    smark(c, SP_TMU, false);
    if (prot) {
      smark(c, SP_ABFT, true);
      RegionF ra{C, c->ld, rows, wa, c->b};
      ABFT_TRY(blocksum(c->st, ra, s_sums(c, r0, cs, true)));
      ABFT_TRY(s_verify_sub(c, k, scheme, correct, r0, c0, rows, cols, 0, 1));
      smark(c, SP_ABFT, false);
    }
    CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
    CUDA_TRY(cudaStreamWaitEvent(c->st2, c->ev_a, 0));
    ABFT_TRY(s_qr_panel(c, c->st2, k + 1, res, &c->gws2));
    CUDA_TRY(cudaEventRecord(c->ev_p, c->st2));
  }
  if (cw > wa) {
    const float* midb = c->mid + wa * c->ld_t;
    float* Cb = C + wa * c->ld;
    FusedSums fs;
    if (fuse) fs = s_fused(c, r0, cs + wa);
    smark(c, SP_TMU, true);
    ABFT_TRY(s_gemm(c, 'N', 'N', rows, cw - wa, w, -1.0f, V, c->ld, midb, c->ld_t, 1.0f, Cb, c->ld,
                    Cb, c->ld, fuse ? &fs : nullptr, la ? c->sms - res : 0));
    smark(c, SP_TMU, false);
    if (prot) {
      smark(c, SP_ABFT, true);
      if (!fuse) {
        RegionF rb{Cb, c->ld, rows, cw - wa, c->b};
        ABFT_TRY(blocksum(c->st, rb, s_sums(c, r0, cs + wa, true)));
      }
      ABFT_TRY(s_verify_sub(c, k, scheme, correct, r0, c0, rows, cols, j0 + (wa ? 1 : 0),
                            ncb - (wa ? 1 : 0)));
      smark(c, SP_ABFT, false);
    }
  }
  ABFT_TRY(s_emit_rowblock(c, k, cs, ce));
  if (la) {
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
    c->qr_count = (int)(k + 2);
    ABFT_TRY(s_emit_column(c, k + 1));
    c->pd_ready = k + 1;
  }
  return 0;
}

int s_stream_chunk(const abft_sctx* c) {
  if (c->lu_chunk >= 0) return c->lu_chunk;
  return c->kind == ABFT_LU ? (int)std::max<int64_t>(1, c->nb / 4) : 1;
}

int64_t s_stream_split(const abft_sctx* c) {
  if (c->kind == ABFT_CHOLESKY || s_stream_chunk(c) <= 0 || c->nb < 4) return 0;
  const int64_t s = c->lu_split >= 0 ? c->lu_split : (c->kind == ABFT_LU ? c->nb / 4 : 3);
  return std::max<int64_t>(1, std::min(s, c->nb - 1));
}

int s_lu_stream_chunks(abft_sctx* c, int64_t split, int scheme, const int32_t* schemes,
                       int correct) {
  const int64_t b = c->b, n = c->n;
  auto sch = [&](int64_t k) { return schemes ? schemes[k] : scheme; };
  if (c->kind == ABFT_LU && !c->linv_store)
    ABFT_TRY(salloc(&c->linv_store, c->ld_t * b * c->nb, c->st));
  if (!c->el_store) ABFT_TRY(salloc(&c->el_store, c->ld_cs * b * c->nb, c->st));
  c->pd_ready = -1;
  const bool lu = c->kind == ABFT_LU;
  c->el_ok.assign(c->nb, 0);
  auto run = [&](int64_t k, int64_t cs, int64_t ce) -> int {
    const bool enc = k == 0 || sch(k - 1) == ABFT_NONE;
    if (!lu) return s_qr_tmu_win(c, k, sch(k), correct, cs, ce, enc);
    smark(c, SP_PU, true);
    ABFT_TRY(s_pu_win(c, k, cs, ce));
    smark(c, SP_PU, false);
    return s_lu_tmu_win(c, k, sch(k), correct, cs, ce, enc);
  };
  const int64_t chunk = s_stream_chunk(c), first = std::max<int64_t>(1, chunk / 4);
  for (int64_t q0 = 0, q1 = 0; q0 < split; q0 = q1) {
    q1 = std::min<int64_t>(q0 + (q0 == 0 ? first : chunk), split);
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_in[q1 - 1], 0));
    for (int64_t k = 0; k < q1; ++k) {
      if (k >= q0) {
        if (c->pd_ready != k) {  // else formed by the look-ahead of TMU(k-1)
          smark(c, SP_PD, true);
          ABFT_TRY(s_pd(c, k));
          smark(c, SP_PD, false);
          ABFT_TRY(s_emit_column(c, k));
        }
        c->pd_ready = -1;
        if (lu) {
          const int64_t pe = std::min((k + 1) * b, n);
          ABFT_TRY(copy_matrix(c->st, c->linv, c->ld_t, c->linv_store + k * c->ld_t * b, c->ld_t,
                               b, b));
          // E_L of panel k as s_maintain would take it: the L21 epilogue's, else a pass
          double* el = c->el_store + k * c->ld_cs * b;
          const int64_t nbr = (n - pe + b - 1) / b;
          if (c->el_for == k) {
            ABFT_TRY(copy_matrix(c->st, c->el, c->ld_cs, el, c->ld_cs, 2 * nbr, b));
          } else if (pe < n) {
            RegionF rl{c->m + pe + k * b * c->ld, c->ld, n - pe, b, b};
            SumOut o;
            o.cp = el;
            o.cp_ld = c->ld_cs;
            o.cp_step = 2;
            o.cw = el + 1;
            o.cw_ld = c->ld_cs;
            o.cw_step = 2;
            ABFT_TRY(blocksum(c->st, rl, o));
          }
        }
      }
      ABFT_TRY(run(k, q0 * b, q1 * b));
    }
  }
  const int64_t rch = c->lu_rchunk > 0 ? c->lu_rchunk
                      : (c->lu_rchunk == 0 || lu) ? c->nb
                                                  : std::max<int64_t>(1, c->nb / 8);
  for (int64_t q0 = split; q0 < c->nb; q0 += rch) {
    const int64_t q1 = std::min<int64_t>(q0 + rch, c->nb);
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_in[q1 - 1], 0));
    for (int64_t k = 0; k < split; ++k) ABFT_TRY(run(k, q0 * b, std::min(q1 * b, n)));
  }
  c->sums_valid = sch(split - 1) != ABFT_NONE;
  return 0;
}

int s_iteration(abft_sctx* c, int64_t k, int scheme, const abft_fault* plan, int nplan, int correct,
                bool sync_checks, bool lookahead = false) {
  auto pd = [&]() -> int {
    if (c->pd_ready == k) {  // produced by the previous iteration's look-ahead
      c->pd_ready = -1;
      return 0;
    }
    smark(c, SP_PD, true);
    ABFT_TRY(s_pd(c, k));
    smark(c, SP_PD, false);
    if (sync_checks) ABFT_TRY(s_check_info(c));
    if (c->kind != ABFT_CHOLESKY) ABFT_TRY(s_emit_column(c, k));
    return 0;
  };
  auto pu = [&]() -> int {
    smark(c, SP_PU, true);
    ABFT_TRY(s_pu(c, k));
    smark(c, SP_PU, false);
    if (c->kind == ABFT_CHOLESKY) ABFT_TRY(s_emit_column(c, k));
    ABFT_TRY(s_emit_rowblock(c, k, 0, c->n));
    return 0;
  };
  if (c->kind == ABFT_CHOLESKY) {
    ABFT_TRY(s_wait_in(c, c->st, k));
    ABFT_TRY(s_protected_tmu(c, k, scheme, plan, nplan, correct));
    // (b % 4: the newest panel's K offset must keep the pre-split rows TMA-aligned)
    const bool la = lookahead && c->lookahead_enabled && k >= 1 && k + 1 < c->nb && c->b % 4 == 0;
    if (la && c->chol_cluster) {
      CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
      ABFT_TRY(pd());
      ABFT_TRY(s_chol_lookahead(c, k, c->next_scheme, true));
    } else {
      if (la) ABFT_TRY(s_chol_lookahead(c, k, c->next_scheme));
      ABFT_TRY(pd());
    }
    if (la) CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_p, 0));
    ABFT_TRY(pu());
  } else if (c->kind == ABFT_QR) {
    ABFT_TRY(pd());
    const int64_t pe = std::min((k + 1) * c->b, c->n);
    const bool la = lookahead && c->lookahead_enabled && nplan == 0 && pe < c->n &&
                    k < c->qr_count && c->qr_la_sms > 0;
    if (la)
      ABFT_TRY(s_tmu_qr_lookahead(c, k, scheme, correct));
    else
      ABFT_TRY(s_protected_tmu(c, k, scheme, plan, nplan, correct));
  } else {
    ABFT_TRY(pd());
    ABFT_TRY(pu());
    const int64_t pe = std::min((k + 1) * c->b, c->n);
    if (lookahead && nplan == 0 && pe < c->n && c->lookahead_enabled)
      ABFT_TRY(s_tmu_lu_lookahead(c, k, scheme, correct));
    else
      ABFT_TRY(s_protected_tmu(c, k, scheme, plan, nplan, correct));
  }
  return 0;
}

int s_collect(abft_sctx* c, std::vector<Event>* out) {
  int32_t cnt[2];
  CUDA_TRY(cudaMemcpyAsync(cnt, c->counters, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  if (cnt[0] > c->ev_cap) {
    set_last_error("ABFT event buffer overflow (%d events)", cnt[0]);
    return ABFT_E_OVERFLOW;
  }
  out->resize(cnt[0]);
  if (cnt[0] > 0) CUDA_TRY(cudaMemcpy(out->data(), c->ev, cnt[0] * sizeof(Event), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemsetAsync(c->counters, 0, 2 * sizeof(int32_t), c->st));
  std::stable_sort(out->begin(), out->end(), [](const Event& a, const Event& b) {
    if (a.iter != b.iter) return a.iter < b.iter;
    if (a.bi != b.bi) return a.bi < b.bi;
    if (a.bj != b.bj) return a.bj < b.bj;
    return a.seq < b.seq;
  });
  for (const Event& e : *out)
    if (e.kind < 0) {
      set_last_error("index 0 is out of bounds for axis 0 with size 0");
      return ABFT_E_RANGE;
    }
  return 0;
}

void s_fill(abft_sctx* c, const std::vector<Event>& evs, int64_t k0, abft_report* reports,
            abft_location* locs, int max_locs, int* n_locs) {
  if (reports)
    for (int64_t k = k0; k < c->nb; ++k) memset(&reports[k], 0, sizeof(abft_report));
  int total = 0;
  for (const Event& e : evs) {
    int64_t r0, c0, rows, cols;
    s_region(c, e.iter, &r0, &c0, &rows, &cols);
    if (reports) {
      abft_report& rep = reports[e.iter];
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
  if (n_locs) *n_locs = total;
}

}  // namespace

extern "C" {

ABFT_API int abft_s_destroy(abft_sctx* c);

// A streamed input not yet consumed by abft_s_factorize: entries that touch
// the matrix otherwise copy it now.
static int s_flush_pending_input(abft_sctx* c) {
  if (!c->in_host) return 0;
  const float* a = c->in_host;
  c->in_host = nullptr;
  CUDA_TRY(cudaMemcpy2DAsync(c->m, c->ld * 4, a, c->in_ld * 4, c->n * 4, c->n,
                             cudaMemcpyHostToDevice, c->st));
  return 0;
}

ABFT_API int abft_s_create(abft_sctx** out, int kind, int64_t n, int64_t b, int device) {
  *out = nullptr;
  if (kind < 0 || kind > 2) {
    set_last_error("unknown decomposition kind %d", kind);
    return ABFT_E_INVALID;
  }
  if (n < 1 || !(1 <= b && b <= n)) {
    set_last_error("block size %lld outside [1, %lld]", (long long)b, (long long)n);
    return ABFT_E_DIM;
  }
  if (b > 256) {
    set_last_error("block size %lld > 256 is not supported by the B200 panel kernels", (long long)b);
    return ABFT_E_INVALID;
  }
  SGuard g(device);
  abft_sctx* c = new abft_sctx();
  c->kind = kind;
  c->n = n;
  c->b = b;
  c->nb = (n + b - 1) / b;
  c->ld = s_round_up(n, 16);
  c->device = device;
  c->ld_cs = s_round_even(2 * c->nb);
  c->ld_max = s_round_even(c->nb);
  c->ld_t = s_round_up(b, 4);
  {
    const char* e = getenv("ABFT_NO_FUSE");
    c->fuse_enabled = !(e && e[0] == '1');
    const char* e4 = getenv("ABFT_CHOL_CLUSTER");
    if (e4 && e4[0] == '0') c->chol_cluster = false;
    const char* e5 = getenv("ABFT_LU_COOP");
    if (e5) c->lu_coop = e5[0] == '1';
    const char* e8 = getenv("ABFT_STREAM_CHUNK");
    if (e8) c->lu_chunk = atoi(e8);
    const char* e9 = getenv("ABFT_STREAM_SPLIT");
    if (e9) c->lu_split = atoll(e9);
    const char* e6 = getenv("ABFT_QR_LA_SMS");
    if (e6) c->qr_la_sms = atoi(e6);
  }
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) {
    set_last_error("cudaStreamCreate failed");
    delete c;
    return -1000;
  }
  int rc = 0;
  auto fail = [&](int r) {
    abft_s_destroy(c);
    return r;
  };
  const int64_t ld = c->ld;
  if ((rc = salloc(&c->m, ld * n, c->st))) return fail(rc);
  if ((rc = salloc(&c->gcsw, c->ld_cs * n, c->st))) return fail(rc);
  if ((rc = salloc(&c->csm, c->ld_cs * n, c->st))) return fail(rc);
  if ((rc = salloc(&c->grs, ld * c->nb, c->st))) return fail(rc);
  if ((rc = salloc(&c->rsm, ld * c->nb, c->st))) return fail(rc);
  if ((rc = salloc(&c->gmax, c->ld_max * c->nb, c->st))) return fail(rc);
  if ((rc = salloc(&c->el, c->ld_cs * b, c->st))) return fail(rc);
  if ((rc = salloc(&c->er, c->ld_t * std::max<int64_t>(c->nb, b), c->st))) return fail(rc);
  if ((rc = salloc(&c->lwd, ld * b, c->st))) return fail(rc);
  if (kind == ABFT_CHOLESKY && (rc = salloc(&c->chol_rs, ld * c->nb, c->st))) return fail(rc);
  if (kind == ABFT_QR) {
    if ((rc = salloc(&c->vstore, ld * n, c->st))) return fail(rc);
    if ((rc = salloc(&c->tstore, c->nb * b * c->ld_t, c->st))) return fail(rc);
    if ((rc = salloc(&c->ww, c->ld_t * n, c->st))) return fail(rc);
    if ((rc = salloc(&c->mid, c->ld_t * n, c->st))) return fail(rc);
    if ((rc = salloc(&c->pan64, ld * b, c->st))) return fail(rc);
    if ((rc = salloc(&c->v64, ld * b, c->st))) return fail(rc);
    if ((rc = salloc(&c->t64, c->ld_t * b, c->st))) return fail(rc);
    if ((rc = salloc(&c->gram, c->ld_t * b, c->st))) return fail(rc);
    if ((rc = salloc(&c->qr_q1, ld * b, c->st))) return fail(rc);
    if ((rc = salloc(&c->qr_small, QR_SMALL_BUFS * c->ld_t * b, c->st))) return fail(rc);
    if ((rc = salloc(&c->betas, b, c->st))) return fail(rc);
    c->qr_part_elems = 2 * 160 * (b + 1);
    if ((rc = salloc(&c->qr_part, c->qr_part_elems, c->st))) return fail(rc);
    if ((rc = salloc(&c->qr_rowbuf, 2 * (b + 1) + 128, c->st))) return fail(rc);
    if ((rc = salloc(&c->qr_part2, 160LL * 32 * b, c->st))) return fail(rc);
    if ((rc = salloc(&c->qr_wfin, 32LL * b, c->st))) return fail(rc);
  }
  if ((rc = salloc(&c->uwd, c->ld_t * n, c->st))) return fail(rc);
  if ((rc = salloc(&c->lw, ld * b, c->st))) return fail(rc);
  if ((rc = salloc(&c->uw, c->ld_t * n, c->st))) return fail(rc);
  if ((rc = salloc(&c->linv, c->ld_t * b, c->st))) return fail(rc);
  if ((rc = salloc(&c->uinv, c->ld_t * b, c->st))) return fail(rc);
  if ((rc = salloc(&c->scratch, 4096, c->st))) return fail(rc);
  c->gws.elems = std::min<int64_t>(std::max<int64_t>(8 * ld * b, 1 << 20), int64_t(64) << 20);
  if ((rc = salloc(&c->gws.ptr, c->gws.elems, c->st))) return fail(rc);
  if (kind == ABFT_QR) {
    c->gws2.elems = c->gws.elems;
    if ((rc = salloc(&c->gws2.ptr, c->gws2.elems, c->st))) return fail(rc);
  }
  // split-operand workspace sized once for the deepest s_gemm of the kind
  // (regrowing inside the per-iteration path costs allocator round trips)
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  c->sws_elems = sgemm_workspace_elems((int)n, (int)n, (int)b);
  for (int64_t k = 0; k < c->nb; ++k) {  // the deep-K GEMMs of the kind
    const int64_t p = k * b, pe = std::min(p + b, n);
    int sp;
    int64_t need = 0;
    if (kind == ABFT_CHOLESKY && k > 0) {  // pre-split operands: partials only
      // main-stream updates (all SMs) and the look-ahead's (one SM fewer)
      for (int cap : {c->sms, c->sms - 1, c->sms - (int)((b + 31) / 32)}) {
        int64_t unused;
        s_gemm_plan(cap, n - p, pe - p, p, S_KCHUNK_CHOL, false, &sp, &unused);
        need = std::max(need, sgemm_partial_elems((int)(n - p), (int)(pe - p), sp) + 128);
      }
    } else if (kind == ABFT_QR && pe < n)
      s_gemm_plan(c->sms, pe - p, n - pe, n - p, S_KCHUNK, false, &sp, &need);
    c->sws_elems = std::max(c->sws_elems, need);
  }
  if ((rc = salloc(&c->sws, c->sws_elems, c->st))) return fail(rc);
  if (kind == ABFT_CHOLESKY) {
    c->ldk = (n + 3) / 4 * 4;
    if ((rc = salloc(&c->lsh, c->ldk * n, c->st))) return fail(rc);
    if ((rc = salloc(&c->lsl, c->ldk * n, c->st))) return fail(rc);
  }
  c->ev_cap = 1 << 16;
  if (cudaMalloc(&c->ev, c->ev_cap * sizeof(Event)) != cudaSuccess) return fail(-1000);
  if (cudaMalloc(&c->counters, 4 * sizeof(int32_t)) != cudaSuccess) return fail(-1000);
  cudaMemsetAsync(c->counters, 0, 4 * sizeof(int32_t), c->st);
  c->dirty_cap = 1 << 16;
  if (cudaMalloc(&c->dirty, 2 * c->dirty_cap * sizeof(int32_t)) != cudaSuccess) return fail(-1000);
  if (cudaMalloc(&c->info, 2 * sizeof(int)) != cudaSuccess) return fail(-1000);
  cudaMemsetAsync(c->info, 0, 2 * sizeof(int), c->st);
  if (kind == ABFT_QR) {
    QrPanelWork& q = c->qrw;
    q.q1 = c->qr_q1;
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
  {
    const char* e2 = getenv("ABFT_NO_LOOKAHEAD");
    c->lookahead_enabled = !(e2 && e2[0] == '1');
  }
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(-1000);
  *out = c;
  return 0;
}

ABFT_API int abft_s_destroy(abft_sctx* c) {
  if (!c) return 0;
  SGuard g(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  void* bufs[] = {c->snap_m, c->snap_rs, c->vstore, c->tstore, c->ww, c->mid, c->pan64, c->v64, c->t64, c->gram, c->qr_q1, c->qr_small,
                  c->betas, c->qr_part, c->qr_rowbuf, c->qr_part2, c->qr_wfin,
                  c->chol_rs, c->m,   c->a0,  c->gcsw, c->csm,  c->grs,     c->rsm,   c->gmax,
                  c->el,  c->er,  c->lwd,  c->uwd,  c->lw,      c->uw,    c->linv,
                  c->uinv, c->sws, c->lsh, c->lsl, c->scratch, c->gws.ptr, c->gws2.ptr, c->ev, c->counters, c->dirty,
                  c->dplan, c->dlist, c->info, c->linv_store, c->el_store};
  for (void* p : bufs)
    if (p) cudaFree(p);
  for (auto& pe : c->prof_pending) {
    cudaEventDestroy(pe.second.first);
    cudaEventDestroy(pe.second.second);
  }
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
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
  return 0;
}

ABFT_API void* abft_s_stream(abft_sctx* c) { return reinterpret_cast<void*>(c->st); }
ABFT_API int64_t abft_s_k_done(abft_sctx* c) { return c->k_done; }

ABFT_API int abft_s_keep_input(abft_sctx* c, int keep) {
  c->keep_input = keep != 0;
  return 0;
}

static void s_reset_state(abft_sctx* c) {
  c->el_for = -1;
  c->er_for = -1;
  c->chol_rs_valid = false;
  c->qr_count = 0;
  c->pd_ready = -1;
  c->chol_part = -1;
  c->chol_enc_ahead = false;
  c->k_done = 0;
  c->sums_valid = false;
  c->breakdown_col = -1;
}

ABFT_API int abft_s_set_matrix(abft_sctx* c, const float* a, int64_t lda) {
  SGuard g(c->device);
  c->in_host = nullptr;
  if (lda < c->n) {
    set_last_error("lda < n");
    return ABFT_E_INVALID;
  }
  CUDA_TRY(cudaMemcpy2DAsync(c->m, c->ld * 4, a, lda * 4, c->n * 4, c->n, cudaMemcpyHostToDevice, c->st));
  if (c->keep_input) {
    if (!c->a0) ABFT_TRY(salloc(&c->a0, c->ld * c->n, c->st));
    CUDA_TRY(cudaMemcpyAsync(c->a0, c->m, c->ld * c->n * 4, cudaMemcpyDeviceToDevice, c->st));
  }
  CUDA_TRY(cudaStreamSynchronize(c->st));
  s_reset_state(c);
  return 0;
}

// abft_set_matrix_streamed for the fp32 context.
ABFT_API int abft_s_set_matrix_streamed(abft_sctx* c, const float* a, int64_t lda) {
  if (c->keep_input) return abft_s_set_matrix(c, a, lda);
  SGuard g(c->device);
  if (lda < c->n) {
    set_last_error("lda < n");
    return ABFT_E_INVALID;
  }
  if (c->kind == ABFT_CHOLESKY && !c->rs_tmp) CUDA_TRY(cudaMalloc(&c->rs_tmp, c->ld * sizeof(double)));
  c->in_host = a;
  c->in_ld = lda;
  s_reset_state(c);
  return 0;
}

ABFT_API int abft_s_reset(abft_sctx* c) {
  SGuard g(c->device);
  if (!c->a0) {
    set_last_error("abft_s_reset needs abft_s_keep_input(ctx, 1) before abft_s_set_matrix");
    return ABFT_E_INVALID;
  }
  CUDA_TRY(cudaMemcpyAsync(c->m, c->a0, c->ld * c->n * 4, cudaMemcpyDeviceToDevice, c->st));
  s_reset_state(c);
  return 0;
}

// m <- m m^T + n I (generate_test_matrix's SPD construction, linalg.py:74-75)
ABFT_API int abft_s_make_spd(abft_sctx* c) {
  SGuard g(c->device);
  ABFT_TRY(s_flush_pending_input(c));
  float* T = nullptr;
  ABFT_TRY(salloc(&T, c->ld * c->n, c->st));
  int rc = s_gemm(c, 'N', 'T', c->n, c->n, c->n, 1.0f, c->m, c->ld, c->m, c->ld, 0.0f, nullptr, 0, T,
                  c->ld);
  if (!rc) rc = add_diag(c->st, T, c->ld, c->n, (double)c->n);
  if (!rc) rc = copy_matrix(c->st, T, c->ld, c->m, c->ld, c->n, c->n, 0);
  if (!rc && c->a0) rc = copy_matrix(c->st, T, c->ld, c->a0, c->ld, c->n, c->n, 0);
  cudaStreamSynchronize(c->st);
  cudaFree(T);
  return rc;
}

ABFT_API int abft_s_get_matrix(abft_sctx* c, float* mh, int64_t ldm) {
  SGuard g(c->device);
  ABFT_TRY(s_flush_pending_input(c));
  CUDA_TRY(cudaMemcpy2DAsync(mh, ldm * 4, c->m, c->ld * 4, c->n * 4, c->n, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

ABFT_API int abft_s_iteration(abft_sctx* c, int64_t k, int scheme, const abft_fault* plan, int nplan,
                              int correct, abft_report* rep, abft_location* locs, int max_locs) {
  SGuard g(c->device);
  ABFT_TRY(s_flush_pending_input(c));
  if (k != c->k_done || k < 0 || k >= c->nb) {
    set_last_error("expected iteration %lld, got %lld", (long long)c->k_done, (long long)k);
    return ABFT_E_DIM;
  }
  if (scheme < 0 || scheme > 2) {
    set_last_error("unknown checksum scheme %d", scheme);
    return ABFT_E_INVALID;
  }
  CUDA_TRY(cudaMemsetAsync(c->counters, 0, 2 * sizeof(int32_t), c->st));
  CUDA_TRY(cudaEventRecord(c->e0, c->st));
  if (k == 0) c->want_chol_rs = true;  // a later iteration may ask for FULL
  int rc = s_iteration(c, k, scheme, plan, nplan, correct, true);
  CUDA_TRY(cudaEventRecord(c->e1, c->st));
  c->timed = true;
  if (rc) return rc;
  std::vector<Event> evs;
  ABFT_TRY(s_collect(c, &evs));
  std::vector<abft_report> reps(c->nb);
  int nl = 0;
  s_fill(c, evs, k, reps.data(), locs, max_locs, &nl);
  if (rep) *rep = reps[k];
  c->k_done = k + 1;
  return 0;
}

ABFT_API int abft_s_factorize(abft_sctx* c, int scheme, const int32_t* schemes, const abft_fault* plan,
                              const int64_t* plan_iter, int nplan, int correct, abft_report* reports,
                              abft_location* locs, int max_locs, int* n_locs) {
  SGuard g(c->device);
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
    // streamed input (as abft_factorize): every block column goes out now on
    // st_in; Cholesky iterations wait for their own block, LU / QR for all
    const bool chol = c->kind == ABFT_CHOLESKY;
    for (int64_t j = (int64_t)c->ev_in.size(); j < c->nb; ++j) {
      cudaEvent_t e = nullptr;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->ev_in.push_back(e);
    }
    CUDA_TRY(cudaEventRecord(c->ev_a, c->st));
    CUDA_TRY(cudaStreamWaitEvent(c->st_in, c->ev_a, 0));
    for (int64_t j = 0; j < c->nb; ++j) {
      const int64_t p = j * c->b, w = std::min(c->b, c->n - p);
      const int64_t r0 = chol ? p : 0;
      CUDA_TRY(cudaMemcpy2DAsync(c->m + r0 + p * c->ld, c->ld * 4, c->in_host + r0 + p * c->in_ld,
                                 c->in_ld * 4, (c->n - r0) * 4, w, cudaMemcpyHostToDevice, c->st_in));
      CUDA_TRY(cudaEventRecord(c->ev_in[j], c->st_in));
    }
    c->in_host = nullptr;
    if (chol) {
      c->in_stream = true;
      c->rs_enc.assign(c->nb, 0);
    } else {
      lu_split = k0 == 0 ? s_stream_split(c) : 0;
      if (plan && plan_iter)
        for (int f = 0; f < nplan; ++f)
          if (plan_iter[f] < lu_split) lu_split = 0;
      if (lu_split == 0) CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_in[c->nb - 1], 0));
    }
  }
  if (lu_split > 0) {
    int rc = s_lu_stream_chunks(c, lu_split, scheme, schemes, correct);
    if (rc) {
      cudaEventRecord(c->e1, c->st);
      return rc;
    }
  }
  for (int64_t k = std::max(k0, lu_split); k < c->nb; ++k) {
    const int sch = schemes ? schemes[k] : scheme;
    c->next_scheme = (k + 1 < c->nb) ? (schemes ? schemes[k + 1] : scheme) : ABFT_NONE;
    int f0 = 0, f1 = 0;
    if (plan && plan_iter) {
      while (f0 < nplan && plan_iter[f0] < k) ++f0;
      f1 = f0;
      while (f1 < nplan && plan_iter[f1] == k) ++f1;
    }
    int rc = s_iteration(c, k, sch, plan ? plan + f0 : nullptr, f1 - f0, correct, false, true);
    if (rc) {
      cudaEventRecord(c->e1, c->st);
      c->in_stream = false;
      return rc;
    }
  }
  c->in_stream = false;
  if (c->out_host) {
    CUDA_TRY(cudaEventRecord(c->ev_out, c->st_out));
    CUDA_TRY(cudaStreamWaitEvent(c->st, c->ev_out, 0));
  }
  CUDA_TRY(cudaEventRecord(c->e1, c->st));
  int brk = s_check_info(c);
  if (brk) {
    c->k_done = c->breakdown_col / c->b;
    return brk;
  }
  std::vector<Event> evs;
  ABFT_TRY(s_collect(c, &evs));
  s_fill(c, evs, k0, reports, locs, max_locs, n_locs);
  c->k_done = c->nb;
  return 0;
}

ABFT_API int abft_s_set_input_chunks(abft_sctx* c, int chunk, int64_t split, int right_chunk) {
  if (chunk < -1 || split < -1 || right_chunk < -1) {
    set_last_error("abft_s_set_input_chunks: chunk, split, right_chunk >= -1");
    return ABFT_E_INVALID;
  }
  c->lu_chunk = chunk;
  c->lu_split = split;
  c->lu_rchunk = right_chunk;
  return 0;
}

ABFT_API int abft_s_stream_out(abft_sctx* c, float* host, int64_t ldh) {
  if (host && ldh < c->n) {
    set_last_error("ldh < n");
    return ABFT_E_INVALID;
  }
  c->out_host = host;
  c->out_ld = ldh;
  return 0;
}

ABFT_API int abft_s_last_elapsed_ms(abft_sctx* c, double* ms) {
  SGuard g(c->device);
  *ms = 0.0;
  if (!c->timed) return 0;
  CUDA_TRY(cudaEventSynchronize(c->e1));
  float f = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&f, c->e0, c->e1));
  *ms = f;
  return 0;
}

ABFT_API int abft_s_profile(abft_sctx* c, int enable) {
  c->prof_on = enable != 0;
  for (double& x : c->prof_ms) x = 0.0;
  return 0;
}

ABFT_API int abft_s_profile_read(abft_sctx* c, double* ms) {
  SGuard g(c->device);
  CUDA_TRY(cudaStreamSynchronize(c->st));
  for (auto& pe : c->prof_pending) {
    float f = 0.f;
    cudaEventElapsedTime(&f, pe.second.first, pe.second.second);
    c->prof_ms[pe.first] += f;
    cudaEventDestroy(pe.second.first);
    cudaEventDestroy(pe.second.second);
  }
  c->prof_pending.clear();
  for (int i = 0; i < 4; ++i) ms[i] = c->prof_ms[i];
  return 0;
}

// residual(a, factors) (linalg.py:362-368) with the reconstruction on the
// tcgen05 GEMM (fp32 accuracy) and fp64 Frobenius sums. a0 == NULL: kept input.
ABFT_API int abft_s_residual(abft_sctx* c, const float* a0h, int64_t lda, double* out) {
  SGuard g(c->device);
  ABFT_TRY(s_flush_pending_input(c));
  if (c->k_done < c->nb) {
    set_last_error("factorization incomplete");
    return ABFT_E_INCOMPLETE;
  }
  const int64_t n = c->n, ld = c->ld;
  float *A = nullptr, *L = nullptr, *U = nullptr, *X = nullptr;
  bool own = false;
  int rc = 0;
  if (a0h) {
    rc = salloc(&A, ld * n, c->st);
    own = true;
    if (!rc && cudaMemcpy2DAsync(A, ld * 4, a0h, lda * 4, n * 4, n, cudaMemcpyHostToDevice, c->st) !=
                   cudaSuccess)
      rc = -1000;
  } else if (c->a0) {
    A = c->a0;
  } else {
    set_last_error("no input matrix for the residual");
    return ABFT_E_INVALID;
  }
  if (!rc) rc = salloc(&L, ld * n, c->st);
  if (!rc) rc = salloc(&U, ld * n, c->st);
  if (!rc) rc = salloc(&X, ld * n, c->st);
  if (!rc) {
    if (c->kind == ABFT_LU) {
      rc = copy_matrix(c->st, c->m, ld, L, ld, n, n, 1);
      if (!rc) rc = copy_matrix(c->st, c->m, ld, U, ld, n, n, 2);
      if (!rc) rc = s_gemm(c, 'N', 'N', n, n, n, 1.0f, L, ld, U, ld, 0.0f, nullptr, 0, X, ld);
    } else if (c->kind == ABFT_CHOLESKY) {
      rc = copy_matrix(c->st, c->m, ld, L, ld, n, n, 3);
      if (!rc) rc = s_gemm(c, 'N', 'T', n, n, n, 1.0f, L, ld, L, ld, 0.0f, nullptr, 0, X, ld);
    } else {
      // X = triu(m); for k from last to 0: X[p:n, :] -= V (T (V^T X[p:n, :]))  (linalg.py:351-359)
      rc = copy_matrix(c->st, c->m, ld, X, ld, n, n, 2);
      for (int64_t k = c->qr_count - 1; k >= 0 && !rc; --k) {
        const int64_t p = k * c->b, pe = std::min(p + c->b, n), w = pe - p;
        const float* V = c->vstore + p + p * ld;
        const float* T = c->tstore + k * c->b * c->ld_t;
        float* blk = X + p;
        rc = s_gemm(c, 'T', 'N', w, n, n - p, 1.0f, V, ld, blk, ld, 0.0f, nullptr, 0, c->ww, c->ld_t);
        if (!rc) rc = s_gemm(c, 'N', 'N', w, n, w, 1.0f, T, c->ld_t, c->ww, c->ld_t, 0.0f, nullptr, 0,
                             c->mid, c->ld_t);
        if (!rc) rc = s_gemm(c, 'N', 'N', n - p, n, w, -1.0f, V, ld, c->mid, c->ld_t, 1.0f, blk, ld,
                             blk, ld);
      }
    }
  }
  double* sq = c->scratch + 2048;
  if (!rc) rc = sumsq(c->st, A, ld, n, n, sq, c->scratch);
  if (!rc) rc = sub_matrix(c->st, A, ld, X, ld, n, n);
  if (!rc) rc = sumsq(c->st, X, ld, n, n, sq + 1, c->scratch + 1024);
  double h[2] = {0, 0};
  if (!rc && cudaMemcpyAsync(h, sq, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st) != cudaSuccess)
    rc = -1000;
  cudaStreamSynchronize(c->st);
  for (float* p : {L, U, X})
    if (p) cudaFree(p);
  if (own && A) cudaFree(A);
  if (rc) return rc;
  const double na = sqrt(h[0]), nd = sqrt(h[1]);
  *out = (na == 0.0) ? nd : nd / na;
  return 0;
}

ABFT_API int64_t abft_s_breakdown_column(abft_sctx* c) { return c->breakdown_col; }

// One in-device snapshot slot of the working matrix (and Cholesky's running
// row checksums) for the recompute recovery policy.
ABFT_API int abft_s_snapshot(abft_sctx* c) {
  SGuard g(c->device);
  ABFT_TRY(s_flush_pending_input(c));
  if (!c->snap_m) ABFT_TRY(salloc(&c->snap_m, c->ld * c->n, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->snap_m, c->m, c->ld * c->n * 4, cudaMemcpyDeviceToDevice, c->st));
  if (c->chol_rs) {
    if (!c->snap_rs) ABFT_TRY(salloc(&c->snap_rs, c->ld * c->nb, c->st));
    CUDA_TRY(cudaMemcpyAsync(c->snap_rs, c->chol_rs, c->ld * c->nb * 8, cudaMemcpyDeviceToDevice,
                             c->st));
  }
  c->snap_rs_valid = c->chol_rs_valid;
  c->snap_k = c->k_done;
  c->snap_qr = c->qr_count;
  c->snap_used = true;
  return 0;
}

ABFT_API int abft_s_restore(abft_sctx* c) {
  SGuard g(c->device);
  if (!c->snap_used) {
    set_last_error("empty snapshot slot");
    return ABFT_E_INVALID;
  }
  CUDA_TRY(cudaMemcpyAsync(c->m, c->snap_m, c->ld * c->n * 4, cudaMemcpyDeviceToDevice, c->st));
  if (c->chol_rs && c->snap_rs)
    CUDA_TRY(cudaMemcpyAsync(c->chol_rs, c->snap_rs, c->ld * c->nb * 8, cudaMemcpyDeviceToDevice,
                             c->st));
  c->chol_rs_valid = c->snap_rs_valid && c->snap_rs != nullptr;
  c->k_done = c->snap_k;
  c->qr_count = c->snap_qr;
  c->sums_valid = false;
  c->pd_ready = -1;
  c->chol_part = -1;
  c->chol_enc_ahead = false;
  c->el_for = -1;
  c->er_for = -1;
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return 0;
}

}  // extern "C"
