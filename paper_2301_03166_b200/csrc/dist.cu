// 1-D block-cyclic distributed factorization context.
//
// One process per GPU; rank g of G owns the global column blocks j with
// j mod G == g, stored contiguously (local block l <-> global block l*G + g),
// so the trailing columns of any iteration are a contiguous local suffix and
// every b x b checksum block, its verification and its repair are local to
// one rank. The exchange step is performed by the caller's transport
// (torch.distributed over NCCL; paper_2301_03166_b200/distributed.py) on a
// device buffer `xbuf` between the phases below:
//
//   LU / QR (right-looking, reference linalg.py:230-300, simulator.py:124-167)
//     begin   owner(k): PD of panel k, pack [panel rows p:n | L11^{-1} or T]
//     -- broadcast xbuf from owner(k) --
//     update  every rank: PU (LU) + encode/maintain + trailing update of its
//             local columns with fused block checksums; local max|region|
//     -- all-reduce MAX of the local maxima (only when faults are planned) --
//     finish  inject the plan's locally owned elements, verify/repair local
//             blocks
//   Cholesky (left-looking as the reference, linalg.py:192-229)
//     begin   every rank: partial panel update from its own finished panels,
//             [X | L*rvec | CS] = L_g * [R_g | rvec_g], CS = E_g * R_g
//     -- sum-reduce xbuf to owner(k) --
//     update  owner: encode the panel column, subtract the reduced update,
//             maintained checksums = encoded - reduced checksum products
//     finish  owner: inject/verify, PD + PU of the panel; all: zero the row
//             block m[p:pe, pe:n] of their columns (linalg.py:251-252)
//
// The plan, RNG draws and the event order are host-side and identical on all
// ranks (abft.py:310-333); events are returned in global coordinates.
#include <algorithm>
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

struct DevGuardD {
  int prev = -1;
  explicit DevGuardD(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuardD() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Zero-filled allocation, ordered on the context's (non-blocking) stream: a
// legacy-stream cudaMemset could otherwise land after later work on `st`.
int dalloc0(double** p, int64_t elems, cudaStream_t st) {
  CUDA_TRY(cudaMalloc(p, std::max<int64_t>(elems, 1) * sizeof(double)));
  CUDA_TRY(cudaMemsetAsync(*p, 0, std::max<int64_t>(elems, 1) * sizeof(double), st));
  return 0;
}

}  // namespace

struct abft_dist {
  int kind = 0;
  int64_t n = 0, b = 0, nb = 0, ld = 0;
  int device = 0, rank = 0, world = 1;
  int64_t nbl = 0, ncl = 0;  // local blocks / columns
  cudaStream_t st = nullptr;

  double* m = nullptr;      // n x ncl (ld)
  double* a0 = nullptr;     // kept local input (abft_dist_keep_input)
  bool keep_input = false;
  double* gcsw = nullptr;   // (2nb) x ncl (ld_cs): row 2*gbi plain, 2*gbi+1 weighted
  double* csm = nullptr;    // maintained col sums, region-local
  int64_t ld_cs = 0;
  double* grs = nullptr;    // n x nbl (ld)
  double* rsm = nullptr;    // maintained row sums, region-local (ld)
  double* gmax = nullptr;
  double* fpart = nullptr;  // fused-epilogue per-strip row sums (ld x 4nb, region-local)
  double* fmaxp = nullptr;  // fused-epilogue per-strip max (ld_max x 4nb)   // nb x nbl (ld_max)
  int64_t ld_max = 0;
  double* el = nullptr;     // operand block-row sums (2nb x b, ld_cs)
  double* er = nullptr;     // R * E_R (b x nbl, ld_t)
  int64_t ld_t = 0;
  double* uw = nullptr;     // b x ncl (ld_t)
  double* lw = nullptr;     // n x b (ld)
  double* linv = nullptr;
  double* uinv = nullptr;
  double* bext = nullptr;   // Cholesky: ncl x (b+1), ld_b
  int64_t ld_b = 0;
  double* vstore = nullptr; // QR: every panel's V (n x n, ld)
  double* tstore = nullptr; // QR: every panel's T (nb of b x b, ld_t)
  double* betas = nullptr;
  double* qr_part = nullptr;
  int64_t qr_part_elems = 0;
  double* qr_rowbuf = nullptr;
  double* qr_part2 = nullptr;
  double* qr_wfin = nullptr;
  double* gram = nullptr;
  double* qr_q1 = nullptr;     // n x b: CholeskyQR2 Q of the owner's panel
  double* qr_small = nullptr;  // QR_SMALL_BUFS x (ld_t x b)
  QrPanelWork qrw;
  double* ww = nullptr;     // b x ncl
  double* mid = nullptr;    // b x ncl
  double* dmax = nullptr;   // local max scratch
  GemmWorkspace gws;

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

  int64_t k_done = 0;
  bool sums_valid = false;
  int64_t breakdown_col = -1;
  int qr_count = 0;
  bool fuse_enabled = true;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool timed = false;
  // LU look-ahead across ranks: the owner of panel k+1 factors and packs it
  // in the middle of update(k); the caller broadcasts it on the comm stream
  // (st2) while the trailing update of k still runs on the main stream.
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_free = nullptr, ev_pack = nullptr, ev_comm = nullptr;
  double* la_buf = nullptr;      // set by abft_dist_lookahead for the next update
  int64_t panel_ready = -1;      // panel already factored + packed by the look-ahead
  bool comm_pending = false;     // main stream must wait on ev_comm before the next begin
  bool verified_in_update = false;
  int reserve_sms = 8;           // SMs left to the collective kernels during the big GEMM
  // Cholesky right-looking (default; ABFT_DIST_CHOL=left keeps the reference's
  // left-looking form with its per-iteration sum-reduce)
  bool chol_right = true;
  double* rv = nullptr;          // b x nbl: row-block sums of L over each local block
  int64_t chol_pd_done = -1;     // panel verified + factored by the look-ahead in update(k)
};

namespace {

int owner(const abft_dist* d, int64_t k) { return (int)(k % d->world); }
// number of owned global blocks j <= k
int64_t owned_upto(const abft_dist* d, int64_t k) {
  return k < d->rank ? 0 : (k - d->rank) / d->world + 1;
}
int64_t width(const abft_dist* d, int64_t k) { return std::min(d->b, d->n - k * d->b); }

// LU/QR exchange buffer: panel rows p:n with ld = round_even(n - p), then the
// w x w companion (L11^{-1} for LU, T for QR) at ld_t.
int64_t panel_ld(const abft_dist* d, int64_t k) { return round_even(d->n - k * d->b); }

// Sums of a local, b-aligned region starting at global row r0 and local block column lb.
SumOut sums_local(abft_dist* d, int64_t r0, int64_t lb, bool rows_too) {
  SumOut o;
  const int64_t gbi = r0 / d->b;
  o.cp = d->gcsw + 2 * gbi + lb * d->b * d->ld_cs;
  o.cp_ld = d->ld_cs;
  o.cp_step = 2;
  o.cw = o.cp + 1;
  o.cw_ld = d->ld_cs;
  o.cw_step = 2;
  if (rows_too) {
    o.rp = d->grs + r0 + lb * d->ld;
    o.rp_ld = d->ld;
  }
  o.bm = d->gmax + gbi + lb * d->ld_max;
  o.bm_ld = d->ld_max;
  return o;
}

FusedSums fused_local(abft_dist* d, int64_t r0, int64_t lb) {
  const SumOut o = sums_local(d, r0, lb, true);
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
  f.rpp = d->fpart;
  f.rpp_ld = d->ld;
  f.bmp = d->fmaxp;
  f.bmp_ld = d->ld_max;
  return f;
}

// Local part of the iteration-k region: global rows [r0, r0+rows), local
// columns [lc0, lc0+cols) starting at local block lb0.
struct LocalRegion {
  int64_t r0 = 0, rows = 0, lb0 = 0, lc0 = 0, cols = 0;
  int64_t gr0 = 0, gc0 = 0;  // global region origin (_tmu_region)
};

LocalRegion local_region(const abft_dist* d, int64_t k) {
  LocalRegion L;
  const int64_t p = k * d->b, pe = std::min(p + d->b, d->n);
  if (d->kind == ABFT_CHOLESKY) {
    L.gr0 = p;
    L.gc0 = p;
    if (owner(d, k) == d->rank) {
      L.r0 = p;
      L.rows = d->n - p;
      L.lb0 = k / d->world;
      L.lc0 = L.lb0 * d->b;
      L.cols = pe - p;
    }
    return L;
  }
  L.gr0 = (d->kind == ABFT_LU) ? pe : p;
  L.gc0 = pe;
  L.r0 = L.gr0;
  L.rows = d->n - L.r0;
  L.lb0 = owned_upto(d, k);
  L.lc0 = L.lb0 * d->b;
  L.cols = d->ncl - L.lc0;
  if (pe >= d->n) L.cols = 0;
  if (L.cols < 0) L.cols = 0;
  return L;
}

Maintained maintained(abft_dist* d) {
  Maintained mt;
  mt.cp = d->csm;
  mt.cp_ld = d->ld_cs;
  mt.cp_step = 2;
  mt.cw = d->csm + 1;
  mt.cw_ld = d->ld_cs;
  mt.cw_step = 2;
  mt.rp = d->rsm;
  mt.rp_ld = d->ld;
  return mt;
}

int upload_plan(abft_dist* d, const abft_fault* plan, int nplan) {
  if (nplan > d->dplan_cap) {
    if (d->dplan) cudaFree(d->dplan);
    d->dplan_cap = std::max(nplan, 64);
    CUDA_TRY(cudaMalloc(&d->dplan, d->dplan_cap * sizeof(DevFault)));
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
  CUDA_TRY(cudaMemcpyAsync(d->dplan, h.data(), nplan * sizeof(DevFault), cudaMemcpyHostToDevice,
                           d->st));
  CUDA_TRY(cudaStreamSynchronize(d->st));
  return 0;
}

// Local blocks (region-local bi, bj) touched by the plan's owned elements.
int upload_touched(abft_dist* d, const abft_fault* plan, int nplan, const LocalRegion& R,
                   int* count) {
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
    for (int64_t r = std::max(ft.row, R.r0); r < std::min(std::min(ft.row + er, d->n), R.r0 + R.rows); ++r)
      for (int64_t c = ft.col; c < std::min(ft.col + ec, d->n); ++c) {
        const int64_t jb = c / d->b;
        if ((int)(jb % d->world) != d->rank) continue;
        const int64_t lc = (jb / d->world) * d->b + c % d->b;
        if (lc < R.lc0 || lc >= R.lc0 + R.cols) continue;
        blks.emplace_back((int32_t)((r - R.r0) / d->b), (int32_t)((lc - R.lc0) / d->b));
      }
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
  if (nn > d->dlist_cap) {
    if (d->dlist) cudaFree(d->dlist);
    d->dlist_cap = std::max(nn, 1024);
    CUDA_TRY(cudaMalloc(&d->dlist, d->dlist_cap * sizeof(int32_t)));
  }
  CUDA_TRY(cudaMemcpyAsync(d->dlist, lst.data(), nn * sizeof(int32_t), cudaMemcpyHostToDevice, d->st));
  CUDA_TRY(cudaStreamSynchronize(d->st));
  return 0;
}

// maintain_gemm (abft.py:138-158) for `region -= L @ R` from the operands:
// L is rows x w (ldl), R is w x cols (ldr), both on the device.
// Restricted to the region's local block columns [j0, j0 + ncb) (Rm points at
// the first of them): the maintained sums land at the matching offsets of the
// region-local csm / rsm, so an update split by block columns (look-ahead)
// maintains piece by piece. E_L (the block sums of L) is reused when el_ready.
int maintain_lr_sub(abft_dist* d, const LocalRegion& R, int scheme, const double* L, int64_t ldl,
                    const double* Rm, int64_t ldr, int64_t w, int64_t j0, int64_t ncb,
                    bool el_ready) {
  const int64_t cbeg = j0 * d->b;
  const int64_t cols = std::min(R.cols - cbeg, ncb * d->b);
  if (cols <= 0 || R.rows <= 0) return 0;
  const int64_t nbr = (R.rows + d->b - 1) / d->b, nbc = (cols + d->b - 1) / d->b;
  SumOut enc = sums_local(d, R.r0, R.lb0 + j0, scheme == ABFT_FULL);
  if (!el_ready) {
    Region rl{const_cast<double*>(L), ldl, R.rows, w, d->b};
    SumOut o;
    o.cp = d->el;
    o.cp_ld = d->ld_cs;
    o.cp_step = 2;
    o.cw = d->el + 1;
    o.cw_ld = d->ld_cs;
    o.cw_step = 2;
    ABFT_TRY(blocksum(d->st, rl, o));
  }
  ABFT_TRY(gemm(d->st, 'N', 'N', (int)(2 * nbr), (int)cols, (int)w, -1.0, d->el, d->ld_cs, Rm, ldr,
                1.0, enc.cp, d->ld_cs, d->csm + cbeg * d->ld_cs, d->ld_cs, &d->gws));
  if (scheme == ABFT_FULL) {
    Region rr{const_cast<double*>(Rm), ldr, w, cols, d->b};
    SumOut o;
    o.rp = d->er;
    o.rp_ld = d->ld_t;
    ABFT_TRY(blocksum(d->st, rr, o));
    ABFT_TRY(gemm(d->st, 'N', 'N', (int)R.rows, (int)nbc, (int)w, -1.0, L, ldl, d->er, d->ld_t, 1.0,
                  enc.rp, d->ld, d->rsm + j0 * d->ld, d->ld, &d->gws));
  }
  return 0;
}

int maintain_lr(abft_dist* d, const LocalRegion& R, int scheme, const double* L, int64_t ldl,
                const double* Rm, int64_t ldr, int64_t w) {
  return maintain_lr_sub(d, R, scheme, L, ldl, Rm, ldr, w, 0, (R.cols + d->b - 1) / d->b, false);
}

// ---------------------------------------------------------------------------
// phases
// ---------------------------------------------------------------------------
int begin_lu(abft_dist* d, int64_t k, double* xb) {
  if (owner(d, k) != d->rank) return 0;
  const int64_t n = d->n, p = k * d->b, pe = std::min(p + d->b, n), w = pe - p;
  const int64_t lc = (k / d->world) * d->b, ldp = panel_ld(d, k);
  double* D = d->m + p + lc * d->ld;
  ABFT_TRY(diag_factor_fast(d->st, D, d->ld, (int)w, 0, d->linv, d->ld_t, d->uinv, d->ld_t, d->info, p));
  if (pe < n) {
    // L21 = A21 U11^{-1} straight into the exchange buffer, then back into m
    ABFT_TRY(gemm(d->st, 'N', 'N', (int)(n - pe), (int)w, (int)w, 1.0, D + w, d->ld, d->uinv, d->ld_t,
                  0.0, nullptr, 0, xb + w, ldp, &d->gws));
    ABFT_TRY(copy_matrix(d->st, xb + w, ldp, D + w, d->ld, n - pe, w));
  }
  ABFT_TRY(copy_matrix(d->st, D, d->ld, xb, ldp, w, w));
  ABFT_TRY(copy_matrix(d->st, d->linv, d->ld_t, xb + ldp * w, d->ld_t, w, w));
  return 0;
}

// (the owner's diagonal factorizations run on the cluster kernel: on 8 GPUs
// this chain -- not the trailing update -- bounds the per-iteration time,
// tools/projection.py)
int begin_qr(abft_dist* d, int64_t k, double* xb) {
  if (owner(d, k) != d->rank) return 0;
  const int64_t n = d->n, p = k * d->b, pe = std::min(p + d->b, n), w = pe - p;
  const int64_t lc = (k / d->world) * d->b, ldp = panel_ld(d, k);
  double* D = d->m + p + lc * d->ld;
  ABFT_TRY(fill_matrix(d->st, xb, ldp, n - p, w, 0.0));
  ABFT_TRY(qr_panel_factor(d->st, D, d->ld, n - p, (int)w, xb, ldp, xb + ldp * w, d->ld_t,
                           d->betas, d->qrw));
  return 0;
}

int begin_chol(abft_dist* d, int64_t k, double* xb) {
  const int64_t n = d->n, p = k * d->b, pe = std::min(p + d->b, n), w = pe - p;
  if (k == 0) return 0;
  const int64_t ldp = panel_ld(d, k), nbr = (n - p + d->b - 1) / d->b;
  const int64_t ldc = round_even(2 * nbr);
  double* X = xb;                       // (n-p) x (w+1)
  double* CS = xb + ldp * (w + 1);      // 2nbr x w
  const int64_t pl = owned_upto(d, k - 1) * d->b;  // own finished panels (all full width)
  if (pl == 0) {
    ABFT_TRY(fill_matrix(d->st, X, ldp, n - p, w + 1, 0.0));
    ABFT_TRY(fill_matrix(d->st, CS, ldc, 2 * nbr, w, 0.0));
    return 0;
  }
  // B_ext = [ m[p:pe, 0:pl]^T | rvec ], rvec = block-row-k plain sums of L
  ABFT_TRY(gather_transpose(d->st, d->m + p, 1, d->ld, w, pl, d->bext, d->ld_b));
  ABFT_TRY(gather_transpose(d->st, d->gcsw + 2 * k, 1, d->ld_cs, 1, pl, d->bext + w * d->ld_b,
                            d->ld_b));
  // [X | L rvec] = L_g[p:n, 0:pl] B_ext ; CS = E_g[2k:, 0:pl] B
  ABFT_TRY(gemm(d->st, 'N', 'N', (int)(n - p), (int)(w + 1), (int)pl, 1.0, d->m + p, d->ld, d->bext,
                d->ld_b, 0.0, nullptr, 0, X, ldp, &d->gws));
  ABFT_TRY(gemm(d->st, 'N', 'N', (int)(2 * nbr), (int)w, (int)pl, 1.0, d->gcsw + 2 * k, d->ld_cs,
                d->bext, d->ld_b, 0.0, nullptr, 0, CS, ldc, &d->gws));
  return 0;
}

int local_max(abft_dist* d, const LocalRegion& R, double* out);

// ---------------------------------------------------------------------------
// right-looking Cholesky: panel k is complete when iteration k
// starts (every earlier panel's rank-b update went to all columns as soon as
// that panel was factored), so the protected region of iteration k -- panel
// column k (simulator.py:90-91) -- is verified, factored and broadcast by its
// owner, and every rank applies it to its own trailing columns. The column /
// row checksums of every future panel are encoded once (k = 0) and maintained
// through each rank-b update from the operands (abft.py:138-158 applied one
// panel at a time), so at iteration k they are exactly the reference's
// maintained checksums of the region, summed in another order.
// Exchange of iteration k >= 1: broadcast from owner(k-1) of
//   [L_{k-1} rows p'..n (ldp x w) | block-row checksums of L_{k-1} (ldc x w)].
int64_t chol_right_xe(const abft_dist* d, int64_t k) {
  if (k == 0) return 0;
  const int64_t k1 = k - 1, p1 = k1 * d->b, w = width(d, k1);
  const int64_t nbr = (d->n - p1 + d->b - 1) / d->b;
  return panel_ld(d, k1) * w + round_even(2 * nbr) * w;
}

// RV[q, t] = sum_{c < w_j} L[(j_t b - p1) + c, q] for the rank's blocks j_t >= k
__global__ void rowblock_sums_kernel(const double* L, int64_t ldp, int64_t p1, int w, int64_t n,
                                     int64_t b, int rank, int world, int64_t l0, int nt,
                                     double* RV, int64_t ldrv) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nt * w;
       idx += gridDim.x * blockDim.x) {
    const int q = idx % w, t = idx / w;
    const int64_t jb = ((l0 + t) * world + rank) * b;
    const int64_t wj = (n - jb < b) ? n - jb : b;
    double s = 0.0;
    for (int64_t c = 0; c < wj; ++c) s += L[(jb - p1) + c + (int64_t)q * ldp];
    RV[q + (int64_t)t * ldrv] = s;
  }
}

int begin_chol_right(abft_dist* d, int64_t k, double* xb) {
  const int64_t n = d->n;
  if (k == 0) {
    // encode every local column once: column sums on the global block grid,
    // row sums per local block column, block maxima
    if (d->ncl > 0) {
      Region all{d->m, d->ld, n, d->ncl, d->b};
      ABFT_TRY(blocksum(d->st, all, sums_local(d, 0, 0, true)));
    }
    return 0;
  }
  const int64_t k1 = k - 1;
  if (owner(d, k1) != d->rank) return 0;
  const int64_t p1 = k1 * d->b, w = width(d, k1), ldp = panel_ld(d, k1);
  const int64_t nbr = (n - p1 + d->b - 1) / d->b, ldc = round_even(2 * nbr);
  const int64_t lc = (k1 / d->world) * d->b;
  ABFT_TRY(copy_matrix(d->st, d->m + p1 + lc * d->ld, d->ld, xb, ldp, n - p1, w));
  // block-row checksums of L_{k-1} (chol_pd_pu wrote them on the global grid)
  ABFT_TRY(copy_matrix(d->st, d->gcsw + 2 * k1 + lc * d->ld_cs, d->ld_cs, xb + ldp * w, ldc,
                       2 * nbr, w));
  return 0;
}

// Apply panel k-1 (L = xb) to the rank's local blocks [la, lb) (all global
// indices >= k): the lower-triangular rank-b update of each block column and
// the maintenance of its column / row checksums.
int chol_right_apply(abft_dist* d, int64_t k, const double* xb, int64_t la, int64_t lb) {
  const int64_t n = d->n, b = d->b;
  const int64_t k1 = k - 1, p1 = k1 * b, w = width(d, k1), ldp = panel_ld(d, k1);
  const int64_t nbr = (n - p1 + b - 1) / b, ldc = round_even(2 * nbr);
  const double* L = xb;
  const double* CS = xb + ldp * w;
  if (lb <= la) return 0;
  for (int64_t l = la; l < lb; ++l) {
    const int64_t j = l * d->world + d->rank, jb = j * b, wj = width(d, j), lc = l * b;
    // A[jb:n, j] -= L[jb:n, :] L[jb:jb+wj, :]^T   (rows >= jb: the panel-j region)
    ABFT_TRY(gemm(d->st, 'N', 'T', (int)(n - jb), (int)wj, (int)w, -1.0, L + (jb - p1), ldp,
                  L + (jb - p1), ldp, 1.0, d->m + jb + lc * d->ld, d->ld, d->m + jb + lc * d->ld,
                  d->ld, &d->gws));
    // column sums of panel j's blocks: CS_j -= CS(L) L[jb:jb+wj, :]^T
    const int64_t nbj = d->nb - j;
    ABFT_TRY(gemm(d->st, 'N', 'T', (int)(2 * nbj), (int)wj, (int)w, -1.0, CS + 2 * (j - k1), ldc,
                  L + (jb - p1), ldp, 1.0, d->gcsw + 2 * j + lc * d->ld_cs, d->ld_cs,
                  d->gcsw + 2 * j + lc * d->ld_cs, d->ld_cs, &d->gws));
  }
  // row sums of the future panels: RS[i, l] -= L[i, :] RV[:, l]
  const int nt = (int)(lb - la);
  int blocks = (int)std::min<int64_t>((nt * w + 255) / 256, 1024);
  count_launch();
  rowblock_sums_kernel<<<std::max(blocks, 1), 256, 0, d->st>>>(L, ldp, p1, (int)w, n, b, d->rank,
                                                               d->world, la, nt, d->rv, d->ld_t);
  CUDA_TRY(cudaGetLastError());
  const int64_t r0 = k * b;
  return gemm(d->st, 'N', 'N', (int)(n - r0), nt, (int)w, -1.0, L + (r0 - p1), ldp, d->rv, d->ld_t,
              1.0, d->grs + r0 + la * d->ld, d->ld, d->grs + r0 + la * d->ld, d->ld, &d->gws);
}

// Panel k on its owner, once every update reached it: maintained sums =
// the running ones, recomputed sums (+ block maxima) from one pass.
int chol_right_region(abft_dist* d, int64_t k, int scheme, int nplan) {
  const LocalRegion R = local_region(d, k);
  if (R.rows <= 0 || R.cols <= 0) return 0;
  const bool prot = scheme != ABFT_NONE;
  const int64_t nbr = (R.rows + d->b - 1) / d->b;
  Region reg{d->m + R.r0 + R.lc0 * d->ld, d->ld, R.rows, R.cols, d->b};
  SumOut run = sums_local(d, R.r0, R.lb0, true);
  if (prot) {
    ABFT_TRY(copy_matrix(d->st, run.cp, d->ld_cs, d->csm, d->ld_cs, 2 * nbr, R.cols));
    if (scheme == ABFT_FULL) ABFT_TRY(copy_matrix(d->st, run.rp, d->ld, d->rsm, d->ld, R.rows, 1));
    ABFT_TRY(blocksum(d->st, reg, run));
  } else if (nplan > 0) {
    SumOut o;
    o.bm = run.bm;
    o.bm_ld = run.bm_ld;
    ABFT_TRY(blocksum(d->st, reg, o));
  }
  return 0;
}

int chol_pd_pu_owner(abft_dist* d, int64_t k);
int inject_verify(abft_dist* d, int64_t k, int scheme, const abft_fault* plan, int nplan,
                  int correct, const double* scale);

int update_chol_right(abft_dist* d, int64_t k, int scheme, const double* xb, int nplan,
                      double* max_out) {
  const int64_t l0 = owned_upto(d, k - 1);  // first local block with global index >= k
  if (d->la_buf && owner(d, k) == d->rank && nplan == 0 && k + 1 < d->nb) {
    // cross-rank look-ahead: panel k first, then verified, factored and
    // packed for the broadcast (comm stream) before the rest of the update
    if (k >= 1) ABFT_TRY(chol_right_apply(d, k, xb, l0, l0 + 1));
    ABFT_TRY(chol_right_region(d, k, scheme, 0));
    ABFT_TRY(inject_verify(d, k, scheme, nullptr, 0, 1, nullptr));
    ABFT_TRY(chol_pd_pu_owner(d, k));
    ABFT_TRY(begin_chol_right(d, k + 1, d->la_buf));
    CUDA_TRY(cudaEventRecord(d->ev_pack, d->st));
    CUDA_TRY(cudaStreamWaitEvent(d->st2, d->ev_pack, 0));
    d->panel_ready = k + 1;
    d->chol_pd_done = k;
    d->verified_in_update = true;
    if (k >= 1) ABFT_TRY(chol_right_apply(d, k, xb, l0 + 1, d->nbl));
    return 0;
  }
  if (k >= 1) ABFT_TRY(chol_right_apply(d, k, xb, l0, d->nbl));
  ABFT_TRY(chol_right_region(d, k, scheme, nplan));
  if (nplan > 0 && max_out) ABFT_TRY(local_max(d, local_region(d, k), max_out));
  return 0;
}

int local_max(abft_dist* d, const LocalRegion& R, double* out) {
  const int64_t nbr = (R.rows + d->b - 1) / d->b, nbc = (R.cols + d->b - 1) / d->b;
  if (R.rows <= 0 || R.cols <= 0) {
    CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), d->st));
    return 0;
  }
  return max_reduce(d->st, d->gmax + R.r0 / d->b + R.lb0 * d->ld_max, nbr, nbc, d->ld_max, out);
}

// Verify (and refresh after repairs) local block columns [j0, j0 + ncb) of
// the iteration-k region (events keep region-local block coordinates).
int verify_sub_local(abft_dist* d, int64_t k, int scheme, int correct, const LocalRegion& R,
                     int64_t j0, int64_t ncb) {
  const int64_t cbeg = j0 * d->b;
  const int64_t csub = std::min(R.cols - cbeg, ncb * d->b);
  if (csub <= 0 || R.rows <= 0) return 0;
  Region sub{d->m + R.r0 + (R.lc0 + cbeg) * d->ld, d->ld, R.rows, csub, d->b};
  SumOut rec = sums_local(d, R.r0, R.lb0 + j0, true);
  Maintained mt = maintained(d);
  mt.cp = d->csm + cbeg * d->ld_cs;
  mt.cw = mt.cp + 1;
  mt.rp = d->rsm + j0 * d->ld;
  EventSink sink{d->ev,          d->counters,  d->ev_cap,  d->dirty, d->counters + 1,
                 d->dirty_cap,   (int32_t)k,   (int32_t)j0, d->b};
  ABFT_TRY(verify_blocks(d->st, sub, d->b, scheme, correct, rec, mt, sink));
  ABFT_TRY(blocksum(d->st, sub, rec, d->dirty, d->counters + 1, d->dirty_cap));
  CUDA_TRY(cudaMemsetAsync(d->counters + 1, 0, sizeof(int32_t), d->st));
  return 0;
}

// LU update of iteration k on the owner of panel k+1 (fault-free k): the
// panel's block column is updated and verified first, panel k+1 is factored
// and packed into the look-ahead buffer (ev_pack releases the comm stream),
// then the rest of the trailing matrix is updated on all but reserve_sms SMs.
int update_lu_lookahead(abft_dist* d, int64_t k, int scheme, const double* xb, const LocalRegion& R,
                        double* U12, int64_t w) {
  const int64_t n = d->n, ldp = panel_ld(d, k);
  const bool prot = scheme != ABFT_NONE;
  const double* L21 = xb + w;
  double* A22 = d->m + R.r0 + R.lc0 * d->ld;
  const int64_t wa = std::min<int64_t>(d->b, R.cols);
  ABFT_TRY(gemm(d->st, 'N', 'N', (int)R.rows, (int)wa, (int)w, -1.0, L21, ldp, U12, d->ld, 1.0, A22,
                d->ld, A22, d->ld, &d->gws));
  if (prot) {
    Region ra{A22, d->ld, R.rows, wa, d->b};
    ABFT_TRY(blocksum(d->st, ra, sums_local(d, R.r0, R.lb0, true)));
    ABFT_TRY(verify_sub_local(d, k, scheme, 1, R, 0, 1));
  }
  // panel k+1 (global block k+1 = local block R.lb0 on this rank)
  ABFT_TRY(begin_lu(d, k + 1, d->la_buf));
  CUDA_TRY(cudaEventRecord(d->ev_pack, d->st));
  CUDA_TRY(cudaStreamWaitEvent(d->st2, d->ev_pack, 0));
  d->panel_ready = k + 1;
  if (R.cols > wa) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
    const int cap = std::max(1, sms - d->reserve_sms);
    if (prot && d->fuse_enabled && gemm_can_fuse((int)d->b)) {
      ABFT_TRY(gemm_fused_sums(d->st, 'N', 'N', (int)R.rows, (int)(R.cols - wa), (int)w, -1.0, L21,
                               ldp, U12 + wa * d->ld, d->ld, 1.0, A22 + wa * d->ld, d->ld,
                               A22 + wa * d->ld, d->ld, (int)d->b, fused_local(d, R.r0, R.lb0 + 1),
                               cap));
    } else {
      ABFT_TRY(gemm_reserved(d->st, 'N', 'N', (int)R.rows, (int)(R.cols - wa), (int)w, -1.0, L21, ldp,
                             U12 + wa * d->ld, d->ld, 1.0, A22 + wa * d->ld, d->ld, A22 + wa * d->ld,
                             d->ld, cap));
      if (prot) {
        Region rb{A22 + wa * d->ld, d->ld, R.rows, R.cols - wa, d->b};
        ABFT_TRY(blocksum(d->st, rb, sums_local(d, R.r0, R.lb0 + 1, true)));
      }
    }
    if (prot) ABFT_TRY(verify_sub_local(d, k, scheme, 1, R, 1, (R.cols + d->b - 1) / d->b));
  }
  (void)n;
  d->verified_in_update = true;
  d->sums_valid = prot;
  return 0;
}

// QR update of iteration k on the owner of panel k+1 (fault-free k): the
// first local block column (global block k+1) gets V^T C, T^T W, its
// maintained sums, C -= V mid, and is verified; panel k+1 (Householder +
// V^T V + larft) is then factored and packed into the look-ahead buffer
// (ev_pack releases the comm stream), and only then do the remaining local
// columns run their three GEMMs (the fused one on all but reserve_sms SMs).
int update_qr_lookahead(abft_dist* d, int64_t k, int scheme, const double* xb,
                        const LocalRegion& R, int64_t w) {
  const int64_t n = d->n, p = k * d->b, ldp = panel_ld(d, k);
  const bool prot = scheme != ABFT_NONE;
  const double* V = xb;
  const double* T = xb + ldp * w;
  double* C = d->m + p + R.lc0 * d->ld;
  const int64_t wa = std::min<int64_t>(d->b, R.cols);
  ABFT_TRY(gemm(d->st, 'T', 'N', (int)w, (int)wa, (int)(n - p), 1.0, V, ldp, C, d->ld, 0.0, nullptr,
                0, d->ww, d->ld_t, &d->gws));
  ABFT_TRY(gemm(d->st, 'T', 'N', (int)w, (int)wa, (int)w, 1.0, T, d->ld_t, d->ww, d->ld_t, 0.0,
                nullptr, 0, d->mid, d->ld_t, &d->gws));
  if (prot) ABFT_TRY(maintain_lr_sub(d, R, scheme, V, ldp, d->mid, d->ld_t, w, 0, 1, false));
  ABFT_TRY(gemm(d->st, 'N', 'N', (int)(n - p), (int)wa, (int)w, -1.0, V, ldp, d->mid, d->ld_t, 1.0,
                C, d->ld, C, d->ld, &d->gws));
  if (prot) {
    Region ra{C, d->ld, R.rows, wa, d->b};
    ABFT_TRY(blocksum(d->st, ra, sums_local(d, R.r0, R.lb0, true)));
    ABFT_TRY(verify_sub_local(d, k, scheme, 1, R, 0, 1));
  }
  // panel k+1 (global block k+1 = local block R.lb0 on this rank)
  ABFT_TRY(begin_qr(d, k + 1, d->la_buf));
  CUDA_TRY(cudaEventRecord(d->ev_pack, d->st));
  CUDA_TRY(cudaStreamWaitEvent(d->st2, d->ev_pack, 0));
  d->panel_ready = k + 1;
  if (R.cols > wa) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
    const int cap = std::max(1, sms - d->reserve_sms);
    const int64_t cr = R.cols - wa;
    double* Cr = C + wa * d->ld;
    ABFT_TRY(gemm(d->st, 'T', 'N', (int)w, (int)cr, (int)(n - p), 1.0, V, ldp, Cr, d->ld, 0.0,
                  nullptr, 0, d->ww + wa * d->ld_t, d->ld_t, &d->gws));
    ABFT_TRY(gemm(d->st, 'T', 'N', (int)w, (int)cr, (int)w, 1.0, T, d->ld_t, d->ww + wa * d->ld_t,
                  d->ld_t, 0.0, nullptr, 0, d->mid + wa * d->ld_t, d->ld_t, &d->gws));
    const int64_t nbc = (R.cols + d->b - 1) / d->b;
    if (prot)
      ABFT_TRY(maintain_lr_sub(d, R, scheme, V, ldp, d->mid + wa * d->ld_t, d->ld_t, w, 1, nbc - 1,
                               true));
    if (prot && d->fuse_enabled && gemm_can_fuse((int)d->b)) {
      ABFT_TRY(gemm_fused_sums(d->st, 'N', 'N', (int)(n - p), (int)cr, (int)w, -1.0, V, ldp,
                               d->mid + wa * d->ld_t, d->ld_t, 1.0, Cr, d->ld, Cr, d->ld, (int)d->b,
                               fused_local(d, R.r0, R.lb0 + 1), cap));
    } else {
      ABFT_TRY(gemm_reserved(d->st, 'N', 'N', (int)(n - p), (int)cr, (int)w, -1.0, V, ldp,
                             d->mid + wa * d->ld_t, d->ld_t, 1.0, Cr, d->ld, Cr, d->ld, cap));
      if (prot) {
        Region rb{Cr, d->ld, R.rows, cr, d->b};
        ABFT_TRY(blocksum(d->st, rb, sums_local(d, R.r0, R.lb0 + 1, true)));
      }
    }
    if (prot) ABFT_TRY(verify_sub_local(d, k, scheme, 1, R, 1, nbc));
  }
  d->verified_in_update = true;
  d->sums_valid = prot;
  return 0;
}

int update_lu_qr(abft_dist* d, int64_t k, int scheme, const double* xb, int nplan,
                 double* max_out) {
  const int64_t n = d->n, p = k * d->b, pe = std::min(p + d->b, n), w = pe - p;
  const int64_t ldp = panel_ld(d, k);
  const LocalRegion R = local_region(d, k);
  const bool has = R.rows > 0 && R.cols > 0;
  const bool prot = scheme != ABFT_NONE && has;
  Region reg{d->m + R.r0 + R.lc0 * d->ld, d->ld, R.rows, R.cols, d->b};
  bool fused = false;
  if (d->kind == ABFT_QR) {
    // keep V_k / T_k (residual, qr_t / _qr_vs)
    ABFT_TRY(copy_matrix(d->st, xb, ldp, d->vstore + p + p * d->ld, d->ld, n - p, w));
    ABFT_TRY(copy_matrix(d->st, xb + ldp * w, d->ld_t, d->tstore + k * d->b * d->ld_t, d->ld_t, w, w));
    d->qr_count = (int)(k + 1);
  }
  if (has) {
    if (d->kind == ABFT_LU) {
      double* U12 = d->m + p + R.lc0 * d->ld;
      ABFT_TRY(gemm(d->st, 'N', 'N', (int)w, (int)R.cols, (int)w, 1.0, xb + ldp * w, d->ld_t, U12,
                    d->ld, 0.0, nullptr, 0, d->uw, d->ld_t, &d->gws));
      ABFT_TRY(copy_matrix(d->st, d->uw, d->ld_t, U12, d->ld, w, R.cols));
      if (prot) {
        if (!d->sums_valid) ABFT_TRY(blocksum(d->st, reg, sums_local(d, R.r0, R.lb0, true)));
        ABFT_TRY(maintain_lr(d, R, scheme, xb + w, ldp, U12, d->ld, w));
      }
      const bool la = d->la_buf != nullptr && nplan == 0;
      if (la && owner(d, k + 1) == d->rank)
        return update_lu_lookahead(d, k, scheme, xb, R, U12, w);
      int cap = 0;  // leave SMs to the collective receiving panel k+1 meanwhile
      if (la) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
        cap = std::max(1, sms - d->reserve_sms);
      }
      const bool fuse = prot && d->fuse_enabled && gemm_can_fuse((int)d->b);
      if (fuse) {
        ABFT_TRY(gemm_fused_sums(d->st, 'N', 'N', (int)R.rows, (int)R.cols, (int)w, -1.0, xb + w, ldp,
                                 U12, d->ld, 1.0, reg.ptr, d->ld, reg.ptr, d->ld, (int)d->b,
                                 fused_local(d, R.r0, R.lb0), cap));
        fused = true;
      } else if (cap > 0) {
        ABFT_TRY(gemm_reserved(d->st, 'N', 'N', (int)R.rows, (int)R.cols, (int)w, -1.0, xb + w, ldp,
                               U12, d->ld, 1.0, reg.ptr, d->ld, reg.ptr, d->ld, cap));
      } else {
        ABFT_TRY(gemm(d->st, 'N', 'N', (int)R.rows, (int)R.cols, (int)w, -1.0, xb + w, ldp, U12, d->ld,
                      1.0, reg.ptr, d->ld, reg.ptr, d->ld, &d->gws));
      }
    } else {
      const double* V = xb;
      const double* T = xb + ldp * w;
      double* C = d->m + p + R.lc0 * d->ld;
      if (prot && !d->sums_valid) ABFT_TRY(blocksum(d->st, reg, sums_local(d, R.r0, R.lb0, true)));
      const bool la = d->la_buf != nullptr && nplan == 0;
      if (la && owner(d, k + 1) == d->rank) return update_qr_lookahead(d, k, scheme, xb, R, w);
      int cap = 0;  // leave SMs to the collective receiving panel k+1 meanwhile
      if (la) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
        cap = std::max(1, sms - d->reserve_sms);
      }
      ABFT_TRY(gemm(d->st, 'T', 'N', (int)w, (int)R.cols, (int)(n - p), 1.0, V, ldp, C, d->ld, 0.0,
                    nullptr, 0, d->ww, d->ld_t, &d->gws));
      ABFT_TRY(gemm(d->st, 'T', 'N', (int)w, (int)R.cols, (int)w, 1.0, T, d->ld_t, d->ww, d->ld_t, 0.0,
                    nullptr, 0, d->mid, d->ld_t, &d->gws));
      if (prot) ABFT_TRY(maintain_lr(d, R, scheme, V, ldp, d->mid, d->ld_t, w));
      const bool fuse = prot && d->fuse_enabled && gemm_can_fuse((int)d->b);
      if (fuse) {
        ABFT_TRY(gemm_fused_sums(d->st, 'N', 'N', (int)(n - p), (int)R.cols, (int)w, -1.0, V, ldp,
                                 d->mid, d->ld_t, 1.0, C, d->ld, C, d->ld, (int)d->b,
                                 fused_local(d, R.r0, R.lb0), cap));
        fused = true;
      } else if (cap > 0) {
        ABFT_TRY(gemm_reserved(d->st, 'N', 'N', (int)(n - p), (int)R.cols, (int)w, -1.0, V, ldp,
                               d->mid, d->ld_t, 1.0, C, d->ld, C, d->ld, cap));
      } else {
        ABFT_TRY(gemm(d->st, 'N', 'N', (int)(n - p), (int)R.cols, (int)w, -1.0, V, ldp, d->mid,
                      d->ld_t, 1.0, C, d->ld, C, d->ld, &d->gws));
      }
    }
    if (prot && !fused) {
      ABFT_TRY(blocksum(d->st, reg, sums_local(d, R.r0, R.lb0, true)));
    } else if (!prot && nplan > 0) {
      SumOut o;
      o.bm = d->gmax + R.r0 / d->b + R.lb0 * d->ld_max;
      o.bm_ld = d->ld_max;
      ABFT_TRY(blocksum(d->st, reg, o));
    }
  }
  if (nplan > 0 && max_out) ABFT_TRY(local_max(d, R, max_out));
  return 0;
}

int update_chol(abft_dist* d, int64_t k, int scheme, const double* xb, int nplan,
                double* max_out) {
  const LocalRegion R = local_region(d, k);
  const bool has = R.rows > 0 && R.cols > 0;
  if (has) {
    const int64_t n = d->n, p = k * d->b, w = R.cols;
    const int64_t ldp = panel_ld(d, k), nbr = (n - p + d->b - 1) / d->b, nbc = 1;
    const int64_t ldc = round_even(2 * nbr);
    const bool prot = scheme != ABFT_NONE;
    Region reg{d->m + R.r0 + R.lc0 * d->ld, d->ld, R.rows, R.cols, d->b};
    SumOut enc = sums_local(d, R.r0, R.lb0, true);
    if (prot) {
      // encode the untouched panel column (abft.py:118-135), maintained = encoded - reduced
      ABFT_TRY(blocksum(d->st, reg, enc));
      ABFT_TRY(copy_matrix(d->st, enc.cp, d->ld_cs, d->csm, d->ld_cs, 2 * nbr, w));
      if (scheme == ABFT_FULL) ABFT_TRY(copy_matrix(d->st, enc.rp, d->ld, d->rsm, d->ld, R.rows, nbc));
      if (k > 0) {
        ABFT_TRY(sub_matrix(d->st, xb + ldp * (w + 1), ldc, d->csm, d->ld_cs, 2 * nbr, w));
        if (scheme == ABFT_FULL) ABFT_TRY(sub_matrix(d->st, xb + ldp * w, ldp, d->rsm, d->ld, R.rows, 1));
      }
    }
    if (k > 0) ABFT_TRY(sub_matrix(d->st, xb, ldp, reg.ptr, d->ld, R.rows, w));  // P -= L L^T
    if (prot) {
      ABFT_TRY(blocksum(d->st, reg, enc));
    } else if (nplan > 0) {
      SumOut o;
      o.bm = enc.bm;
      o.bm_ld = enc.bm_ld;
      ABFT_TRY(blocksum(d->st, reg, o));
    }
  }
  if (nplan > 0 && max_out) ABFT_TRY(local_max(d, R, max_out));
  return 0;
}

int inject_verify(abft_dist* d, int64_t k, int scheme, const abft_fault* plan, int nplan,
                  int correct, const double* scale) {
  const LocalRegion R = local_region(d, k);
  const bool has = R.rows > 0 && R.cols > 0;
  const bool prot = scheme != ABFT_NONE && has;
  Region reg{d->m + R.r0 + R.lc0 * d->ld, d->ld, R.rows, R.cols, d->b};
  if (nplan > 0) {
    for (int f = 0; f < nplan; ++f)
      if (plan[f].row < 0 || plan[f].row >= d->n || plan[f].col < 0 || plan[f].col >= d->n) {
        set_last_error("fault at (%lld, %lld) outside matrix", (long long)plan[f].row,
                       (long long)plan[f].col);
        return ABFT_E_RANGE;
      }
  }
  if (nplan > 0 && has) {
    ABFT_TRY(upload_plan(d, plan, nplan));
    ABFT_TRY(inject_mapped(d->st, d->m, d->ld, d->n, d->dplan, nplan, scale, d->world, d->rank,
                           d->b));
    if (prot) {
      int cnt = 0;
      ABFT_TRY(upload_touched(d, plan, nplan, R, &cnt));
      if (cnt > 0)
        ABFT_TRY(blocksum(d->st, reg, sums_local(d, R.r0, R.lb0, true), d->dlist, nullptr, cnt));
    }
  }
  if (d->verified_in_update) {  // look-ahead owner: verified block column by block column
    d->verified_in_update = false;
    return 0;
  }
  if (prot) {
    EventSink sink{d->ev, d->counters, d->ev_cap, d->dirty, d->counters + 1, d->dirty_cap,
                   (int32_t)k};
    ABFT_TRY(verify_blocks(d->st, reg, d->b, scheme, correct, sums_local(d, R.r0, R.lb0, true),
                           maintained(d), sink));
    ABFT_TRY(blocksum(d->st, reg, sums_local(d, R.r0, R.lb0, true), d->dirty, d->counters + 1,
                      d->dirty_cap));
    CUDA_TRY(cudaMemsetAsync(d->counters + 1, 0, sizeof(int32_t), d->st));
  }
  d->sums_valid = prot;
  return 0;
}

// Cholesky PD + PU of panel k (owner) after verification; every rank zeroes
// its columns of the row block m[p:pe, pe:n] (linalg.py:228-229, :251-252).
int chol_pd_pu_owner(abft_dist* d, int64_t k) {
  const int64_t n = d->n, p = k * d->b, pe = std::min(p + d->b, n), w = pe - p;
  if (owner(d, k) != d->rank) return 0;
  const int64_t lc = (k / d->world) * d->b;
  double* D = d->m + p + lc * d->ld;
  ABFT_TRY(diag_factor_fast(d->st, D, d->ld, (int)w, 1, d->linv, d->ld_t, nullptr, 0, d->info, p));
  if (pe < n) {
    ABFT_TRY(gemm(d->st, 'N', 'T', (int)(n - pe), (int)w, (int)w, 1.0, D + w, d->ld, d->linv,
                  d->ld_t, 0.0, nullptr, 0, d->lw, d->ld, &d->gws));
    ABFT_TRY(copy_matrix(d->st, d->lw, d->ld, D + w, d->ld, n - pe, w));
  }
  // block-row checksums of the finished L panel (operand sums of later maintenance)
  Region reg{D, d->ld, n - p, w, d->b};
  SumOut o = sums_local(d, p, k / d->world, false);
  o.bm = nullptr;
  return blocksum(d->st, reg, o);
}

int chol_pd_pu(abft_dist* d, int64_t k) {
  const int64_t n = d->n, p = k * d->b, pe = std::min(p + d->b, n), w = pe - p;
  if (d->chol_pd_done == k) {
    d->chol_pd_done = -1;  // factored by the look-ahead in update(k)
  } else {
    ABFT_TRY(chol_pd_pu_owner(d, k));
  }
  const int64_t tc0 = owned_upto(d, k) * d->b;
  if (pe < n && d->ncl > tc0) ABFT_TRY(fill_matrix(d->st, d->m + p + tc0 * d->ld, d->ld, w, d->ncl - tc0, 0.0));
  return 0;
}

int check_info(abft_dist* d) {
  int h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, d->info, sizeof(int), cudaMemcpyDeviceToHost, d->st));
  CUDA_TRY(cudaStreamSynchronize(d->st));
  if (h != 0) {
    d->breakdown_col = h - 1;
    if (d->kind == ABFT_CHOLESKY)
      set_last_error("non-positive pivot at column %lld", (long long)d->breakdown_col);
    else
      set_last_error("zero pivot at column %lld", (long long)d->breakdown_col);
    CUDA_TRY(cudaMemsetAsync(d->info, 0, sizeof(int), d->st));
    return ABFT_E_BREAKDOWN;
  }
  return 0;
}

int check_k(abft_dist* d, int64_t k, int scheme) {
  if (k < 0 || k >= d->nb) {
    set_last_error("iteration %lld out of range for %lld blocks", (long long)k, (long long)d->nb);
    return ABFT_E_DIM;
  }
  if (scheme < 0 || scheme > 2) {
    set_last_error("unknown checksum scheme %d", scheme);
    return ABFT_E_INVALID;
  }
  return 0;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

ABFT_API int abft_dist_destroy(abft_dist* d);

ABFT_API int abft_dist_create(abft_dist** out, int kind, int64_t n, int64_t b, int device, int rank,
                              int world) {
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
  if (world < 1 || rank < 0 || rank >= world) {
    set_last_error("rank %d outside world of %d", rank, world);
    return ABFT_E_INVALID;
  }
  DevGuardD g(device);
  abft_dist* d = new abft_dist();
  d->kind = kind;
  d->n = n;
  d->b = b;
  d->nb = (n + b - 1) / b;
  d->ld = round_up(n, 16);
  d->device = device;
  d->rank = rank;
  d->world = world;
  d->nbl = d->nb > rank ? (d->nb - 1 - rank) / world + 1 : 0;
  d->ncl = 0;
  for (int64_t l = 0; l < d->nbl; ++l) d->ncl += width(d, l * world + rank);
  d->ld_cs = round_even(2 * d->nb);
  d->ld_max = round_even(d->nb);
  d->ld_t = round_even(b);
  d->ld_b = round_even(std::max<int64_t>(d->ncl, 1));
  {
    const char* e = getenv("ABFT_NO_FUSE");
    d->fuse_enabled = !(e && e[0] == '1');
  }
  int rc = 0;
  auto fail = [&](int r) {
    abft_dist_destroy(d);
    return r;
  };
  if (cudaStreamCreateWithFlags(&d->st, cudaStreamNonBlocking) != cudaSuccess) {
    set_last_error("cudaStreamCreate failed");
    delete d;
    return -1000;
  }
  const int64_t ncl = std::max<int64_t>(d->ncl, 1), nbl = std::max<int64_t>(d->nbl, 1), ld = d->ld;
  if ((rc = dalloc0(&d->m, ld * ncl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->gcsw, d->ld_cs * ncl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->csm, d->ld_cs * ncl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->grs, ld * nbl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->rsm, ld * nbl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->gmax, d->ld_max * nbl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->fpart, ld * 4 * nbl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->fmaxp, d->ld_max * 4 * nbl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->el, d->ld_cs * b, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->er, d->ld_t * std::max<int64_t>(nbl, b), d->st))) return fail(rc);
  if ((rc = dalloc0(&d->uw, d->ld_t * ncl, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->lw, ld * b, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->linv, d->ld_t * b, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->uinv, d->ld_t * b, d->st))) return fail(rc);
  if ((rc = dalloc0(&d->dmax, 2, d->st))) return fail(rc);
  if (kind == ABFT_CHOLESKY && (rc = dalloc0(&d->bext, d->ld_b * (b + 1), d->st))) return fail(rc);
  if (kind == ABFT_CHOLESKY && (rc = dalloc0(&d->rv, d->ld_t * nbl, d->st))) return fail(rc);
  if (kind == ABFT_QR) {
    if ((rc = dalloc0(&d->vstore, ld * n, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->tstore, d->nb * b * d->ld_t, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->betas, b, d->st))) return fail(rc);
    d->qr_part_elems = 2 * 160 * (b + 1);
    if ((rc = dalloc0(&d->qr_part, d->qr_part_elems, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->qr_rowbuf, 2 * (b + 1) + 128, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->qr_part2, 160LL * 32 * b, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->qr_wfin, 32LL * b, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->gram, d->ld_t * b, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->qr_q1, ld * b, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->qr_small, QR_SMALL_BUFS * d->ld_t * b, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->ww, d->ld_t * ncl, d->st))) return fail(rc);
    if ((rc = dalloc0(&d->mid, d->ld_t * ncl, d->st))) return fail(rc);
  }
  d->gws.elems = std::min<int64_t>(std::max<int64_t>(8 * ld * b, 1 << 20), int64_t(64) << 20);
  if ((rc = dalloc0(&d->gws.ptr, d->gws.elems, d->st))) return fail(rc);
  d->ev_cap = 1 << 16;
  if (cudaMalloc(&d->ev, d->ev_cap * sizeof(Event)) != cudaSuccess) return fail(-1000);
  if (cudaMalloc(&d->counters, 4 * sizeof(int32_t)) != cudaSuccess) return fail(-1000);
  cudaMemset(d->counters, 0, 4 * sizeof(int32_t));
  d->dirty_cap = 1 << 16;
  if (cudaMalloc(&d->dirty, 2 * d->dirty_cap * sizeof(int32_t)) != cudaSuccess) return fail(-1000);
  if (cudaMalloc(&d->info, 2 * sizeof(int)) != cudaSuccess) return fail(-1000);
  cudaMemset(d->info, 0, 2 * sizeof(int));
  if (kind == ABFT_QR) {
    QrPanelWork& q = d->qrw;
    q.q1 = d->qr_q1;
    q.ldq = ld;
    q.small = d->qr_small;
    q.lds = d->ld_t;
    q.info = d->info + 1;
    q.gws = &d->gws;
    q.part = d->qr_part;
    q.part_elems = d->qr_part_elems;
    q.rowbuf = d->qr_rowbuf;
    q.part2 = d->qr_part2;
    q.wfin = d->qr_wfin;
    q.gram = d->gram;
    q.ldg = d->ld_t;
  }
  cudaEventCreate(&d->e0);
  cudaEventCreate(&d->e1);
  cudaStreamCreateWithFlags(&d->st2, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&d->ev_free, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&d->ev_pack, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&d->ev_comm, cudaEventDisableTiming);
  {
    const char* ec = getenv("ABFT_DIST_CHOL");
    d->chol_right = !(ec && (ec[0] == 'l' || ec[0] == 'L'));
  }
  {
    const char* e = getenv("ABFT_DIST_RESERVE_SMS");
    if (e) d->reserve_sms = std::max(0, atoi(e));
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(-1000);
  *out = d;
  return 0;
}

ABFT_API int abft_dist_destroy(abft_dist* d) {
  if (!d) return 0;
  DevGuardD g(d->device);
  if (d->st) cudaStreamSynchronize(d->st);
  double* bufs[] = {d->fpart,  d->fmaxp,
                    d->m,      d->a0,     d->gcsw,   d->csm,    d->grs,       d->rsm,      d->gmax,
                    d->el,     d->er,     d->uw,     d->lw,        d->linv,     d->uinv,
                    d->bext,   d->rv,     d->vstore, d->tstore, d->betas,     d->qr_part,  d->qr_rowbuf,
                    d->qr_part2, d->qr_wfin, d->gram, d->qr_q1, d->qr_small, d->ww,       d->mid,      d->dmax,
                    d->gws.ptr};
  for (double* p : bufs)
    if (p) cudaFree(p);
  if (d->ev) cudaFree(d->ev);
  if (d->counters) cudaFree(d->counters);
  if (d->dirty) cudaFree(d->dirty);
  if (d->dplan) cudaFree(d->dplan);
  if (d->dlist) cudaFree(d->dlist);
  if (d->info) cudaFree(d->info);
  if (d->e0) cudaEventDestroy(d->e0);
  if (d->e1) cudaEventDestroy(d->e1);
  if (d->st2) {
    cudaStreamSynchronize(d->st2);
    cudaStreamDestroy(d->st2);
  }
  for (cudaEvent_t e : {d->ev_free, d->ev_pack, d->ev_comm})
    if (e) cudaEventDestroy(e);
  if (d->st) cudaStreamDestroy(d->st);
  delete d;
  return 0;
}

ABFT_API int64_t abft_dist_local_cols(abft_dist* d) { return d->ncl; }

ABFT_API void* abft_dist_stream(abft_dist* d) { return reinterpret_cast<void*>(d->st); }

ABFT_API int64_t abft_dist_xbuf_elems(abft_dist* d, int64_t k) {
  if (k < 0 || k >= d->nb) return 0;
  const int64_t p = k * d->b, w = width(d, k), ldp = panel_ld(d, k);
  if (d->kind == ABFT_CHOLESKY) {
    if (d->chol_right) return chol_right_xe(d, k);
    if (k == 0) return 0;
    const int64_t nbr = (d->n - p + d->b - 1) / d->b;
    return ldp * (w + 1) + round_even(2 * nbr) * w;
  }
  if (p + w >= d->n && d->kind == ABFT_LU) return 0;  // last LU panel: nothing to send
  return ldp * w + d->ld_t * w;
}

ABFT_API int abft_dist_set_matrix(abft_dist* d, const double* a, int64_t lda) {
  DevGuardD g(d->device);
  if (lda < d->n) {
    set_last_error("lda < n");
    return ABFT_E_INVALID;
  }
  for (int64_t l = 0; l < d->nbl; ++l) {
    const int64_t j = l * d->world + d->rank;
    CUDA_TRY(cudaMemcpy2DAsync(d->m + l * d->b * d->ld, d->ld * 8, a + j * d->b * lda, lda * 8,
                               d->n * 8, width(d, j), cudaMemcpyHostToDevice, d->st));
  }
  if (d->keep_input) {
    if (!d->a0) ABFT_TRY(dalloc0(&d->a0, d->ld * std::max<int64_t>(d->ncl, 1), d->st));
    CUDA_TRY(cudaMemcpyAsync(d->a0, d->m, d->ld * d->ncl * 8, cudaMemcpyDeviceToDevice, d->st));
  }
  CUDA_TRY(cudaStreamSynchronize(d->st));
  d->k_done = 0;
  d->sums_valid = false;
  d->qr_count = 0;
  d->breakdown_col = -1;
  d->panel_ready = -1;
  d->comm_pending = false;
  d->la_buf = nullptr;
  d->verified_in_update = false;
  d->chol_pd_done = -1;
  return 0;
}

ABFT_API int abft_dist_keep_input(abft_dist* d, int keep) {
  d->keep_input = keep != 0;
  return 0;
}

// Restore the local columns from the kept input (a new factorization without
// a host round trip); asynchronous on the context stream.
ABFT_API int abft_dist_reset(abft_dist* d) {
  DevGuardD g(d->device);
  if (!d->a0) {
    set_last_error("abft_dist_reset needs abft_dist_keep_input(d, 1) before abft_dist_set_matrix");
    return ABFT_E_INVALID;
  }
  CUDA_TRY(cudaMemcpyAsync(d->m, d->a0, d->ld * d->ncl * 8, cudaMemcpyDeviceToDevice, d->st));
  d->k_done = 0;
  d->sums_valid = false;
  d->qr_count = 0;
  d->breakdown_col = -1;
  d->panel_ready = -1;
  d->comm_pending = false;
  d->la_buf = nullptr;
  d->verified_in_update = false;
  d->chol_pd_done = -1;
  return 0;
}

// The rank's own column blocks (n x local_cols, ldl), already scattered.
ABFT_API int abft_dist_set_local(abft_dist* d, const double* local, int64_t ldl) {
  DevGuardD g(d->device);
  if (ldl < d->n) {
    set_last_error("ldl < n");
    return ABFT_E_INVALID;
  }
  if (d->ncl > 0)
    CUDA_TRY(cudaMemcpy2DAsync(d->m, d->ld * 8, local, ldl * 8, d->n * 8, d->ncl,
                               cudaMemcpyHostToDevice, d->st));
  if (d->keep_input) {
    if (!d->a0) ABFT_TRY(dalloc0(&d->a0, d->ld * std::max<int64_t>(d->ncl, 1), d->st));
    CUDA_TRY(cudaMemcpyAsync(d->a0, d->m, d->ld * d->ncl * 8, cudaMemcpyDeviceToDevice, d->st));
  }
  CUDA_TRY(cudaStreamSynchronize(d->st));
  d->k_done = 0;
  d->sums_valid = false;
  d->qr_count = 0;
  d->breakdown_col = -1;
  d->panel_ready = -1;
  d->comm_pending = false;
  d->la_buf = nullptr;
  d->verified_in_update = false;
  d->chol_pd_done = -1;
  return 0;
}

ABFT_API int abft_dist_get_matrix(abft_dist* d, double* out, int64_t ldo) {
  DevGuardD g(d->device);
  if (d->ncl > 0)
    CUDA_TRY(cudaMemcpy2DAsync(out, ldo * 8, d->m, d->ld * 8, d->n * 8, d->ncl,
                               cudaMemcpyDeviceToHost, d->st));
  CUDA_TRY(cudaStreamSynchronize(d->st));
  return 0;
}

ABFT_API int abft_dist_begin(abft_dist* d, int64_t k, int scheme, double* xbuf) {
  DevGuardD g(d->device);
  ABFT_TRY(check_k(d, k, scheme));
  if (k != d->k_done) {
    set_last_error("expected iteration %lld, got %lld", (long long)d->k_done, (long long)k);
    return ABFT_E_DIM;
  }
  if (k == 0) {
    CUDA_TRY(cudaMemsetAsync(d->counters, 0, 2 * sizeof(int32_t), d->st));
    CUDA_TRY(cudaEventRecord(d->e0, d->st));
    d->timed = false;
  }
  if (d->comm_pending) {  // the look-ahead broadcast of this panel ran on the comm stream
    CUDA_TRY(cudaStreamWaitEvent(d->st, d->ev_comm, 0));
    d->comm_pending = false;
  }
  if ((d->kind != ABFT_CHOLESKY || d->chol_right) && d->panel_ready == k) {  // packed by the look-ahead
    d->panel_ready = -1;
    return 0;
  }
  if (d->kind == ABFT_LU) {
    // the last LU panel is factored in place; nothing is exchanged
    const int64_t p = k * d->b, pe = std::min(p + d->b, d->n);
    if (pe >= d->n) {
      if (owner(d, k) == d->rank) {
        const int64_t lc = (k / d->world) * d->b;
        ABFT_TRY(diag_factor_fast(d->st, d->m + p + lc * d->ld, d->ld, (int)(pe - p), 0, d->linv,
                             d->ld_t, d->uinv, d->ld_t, d->info, p));
      }
      return 0;
    }
    return begin_lu(d, k, xbuf);
  }
  if (d->kind == ABFT_QR) return begin_qr(d, k, xbuf);
  if (d->chol_right) return begin_chol_right(d, k, xbuf);
  return begin_chol(d, k, xbuf);
}

// The exchange step of iteration k, between abft_dist_begin and
// abft_dist_update: 0 none, 1 broadcast from *root, 2 sum-reduce to *root
// (left-looking Cholesky); abft_dist_xbuf_elems(k) doubles of the buffer.
ABFT_API int abft_dist_exchange(abft_dist* d, int64_t k, int* root) {
  *root = 0;
  if (k < 0 || k >= d->nb || abft_dist_xbuf_elems(d, k) == 0) return 0;
  if (d->kind == ABFT_CHOLESKY) {
    if (d->chol_right) {
      *root = owner(d, k - 1);
      return 1;
    }
    *root = owner(d, k);
    return 2;
  }
  *root = owner(d, k);
  return 1;
}

ABFT_API int abft_dist_update(abft_dist* d, int64_t k, int scheme, const double* xbuf, int nplan,
                              double* local_max) {
  DevGuardD g(d->device);
  ABFT_TRY(check_k(d, k, scheme));
  if (d->kind == ABFT_CHOLESKY && !d->chol_right) return update_chol(d, k, scheme, xbuf, nplan, local_max);
  if (d->kind == ABFT_CHOLESKY) {
    if (d->la_buf) {
      CUDA_TRY(cudaEventRecord(d->ev_free, d->st));
      CUDA_TRY(cudaStreamWaitEvent(d->st2, d->ev_free, 0));
    }
    const int rc = update_chol_right(d, k, scheme, xbuf, nplan, local_max);
    d->la_buf = nullptr;
    return rc;
  }
  if (d->kind == ABFT_LU && std::min((k + 1) * d->b, d->n) >= d->n) {
    d->la_buf = nullptr;
    if (nplan > 0 && local_max) CUDA_TRY(cudaMemsetAsync(local_max, 0, sizeof(double), d->st));
    return 0;
  }
  if (d->la_buf) {
    // the comm stream may overwrite the look-ahead buffer only after every
    // earlier reader on the main stream (update(k-1)) is done
    CUDA_TRY(cudaEventRecord(d->ev_free, d->st));
    CUDA_TRY(cudaStreamWaitEvent(d->st2, d->ev_free, 0));
  }
  const int rc = update_lu_qr(d, k, scheme, xbuf, nplan, local_max);
  d->la_buf = nullptr;
  return rc;
}

// LU / QR look-ahead for the next abft_dist_update(k): the owner of panel k+1
// factors it mid-update into `xnext` (abft_dist_xbuf_elems(k+1) doubles);
// the caller then broadcasts `xnext` from rank (k+1) mod G on the comm stream
// (abft_dist_comm_stream) and calls abft_dist_comm_done; begin(k+1) makes the
// main stream wait for that broadcast.
ABFT_API int abft_dist_lookahead(abft_dist* d, int64_t k, double* xnext) {
  if ((d->kind == ABFT_CHOLESKY && !d->chol_right) || k + 1 >= d->nb ||
      abft_dist_xbuf_elems(d, k + 1) == 0) {
    set_last_error("no look-ahead panel after iteration %lld", (long long)k);
    return ABFT_E_INVALID;
  }
  d->la_buf = xnext;
  return 0;
}

ABFT_API void* abft_dist_comm_stream(abft_dist* d) { return reinterpret_cast<void*>(d->st2); }

ABFT_API int abft_dist_comm_done(abft_dist* d) {
  DevGuardD g(d->device);
  CUDA_TRY(cudaEventRecord(d->ev_comm, d->st2));
  d->comm_pending = true;
  return 0;
}

ABFT_API int abft_dist_finish(abft_dist* d, int64_t k, int scheme, const abft_fault* plan, int nplan,
                              int correct, const double* scale) {
  DevGuardD g(d->device);
  ABFT_TRY(check_k(d, k, scheme));
  ABFT_TRY(inject_verify(d, k, scheme, plan, nplan, correct, scale));
  if (d->kind == ABFT_CHOLESKY) ABFT_TRY(chol_pd_pu(d, k));
  d->k_done = k + 1;
  if (d->k_done == d->nb) {
    CUDA_TRY(cudaEventRecord(d->e1, d->st));
    d->timed = true;
  }
  return 0;
}

// Synchronize, check for a numeric breakdown and return every ABFT event
// since the last call in global coordinates (row/col of the element or block
// corner, block_row/block_col on the global region-local grid, iteration in
// `iters`), unsorted; the host merges ranks and orders them like the
// reference (iteration, block row, block column, column).
ABFT_API int abft_dist_events(abft_dist* d, abft_location* locs, int64_t* iters, int max_locs,
                              int* n_out) {
  DevGuardD g(d->device);
  *n_out = 0;
  ABFT_TRY(check_info(d));
  int32_t cnt[2];
  CUDA_TRY(cudaMemcpyAsync(cnt, d->counters, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, d->st));
  CUDA_TRY(cudaStreamSynchronize(d->st));
  if (cnt[0] > d->ev_cap) {
    set_last_error("ABFT event buffer overflow (%d events)", cnt[0]);
    return ABFT_E_OVERFLOW;
  }
  std::vector<Event> evs(cnt[0]);
  if (cnt[0] > 0)
    CUDA_TRY(cudaMemcpy(evs.data(), d->ev, cnt[0] * sizeof(Event), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemsetAsync(d->counters, 0, 2 * sizeof(int32_t), d->st));
  *n_out = (int)evs.size();
  for (size_t i = 0; i < evs.size(); ++i) {
    const Event& e = evs[i];
    if (e.kind < 0) {
      set_last_error("index 0 is out of bounds for axis 0 with size 0");
      return ABFT_E_RANGE;
    }
    if ((int)i >= max_locs) continue;
    const LocalRegion R = local_region(d, e.iter);
    const int64_t jg = (R.lb0 + e.bj) * d->world + d->rank;  // global block column
    abft_location& L = locs[i];
    L.row = R.r0 + e.row;
    L.col = jg * d->b + (e.col - (int64_t)e.bj * d->b);
    L.kind = e.kind;
    L.flag = e.flag;
    L.detected_kind = e.detected_kind;
    L.corrected = e.corrected;
    L.uncorrectable = e.uncorrectable;
    L.block_row = e.bi;
    L.block_col = (int32_t)(jg - R.gc0 / d->b);
    L.seq = e.seq;
    if (iters) iters[i] = e.iter;
  }
  return 0;
}

ABFT_API int64_t abft_dist_k_done(abft_dist* d) { return d->k_done; }

ABFT_API int abft_dist_get_qr_panel(abft_dist* d, int64_t k, double* V, int64_t ldv, double* T,
                                    int64_t ldt) {
  DevGuardD g(d->device);
  if (d->kind != ABFT_QR || k < 0 || k >= d->qr_count) {
    set_last_error("no QR panel %lld", (long long)k);
    return ABFT_E_INVALID;
  }
  const int64_t p = k * d->b, w = width(d, k);
  if (V)
    CUDA_TRY(cudaMemcpy2DAsync(V, ldv * 8, d->vstore + p + p * d->ld, d->ld * 8, (d->n - p) * 8, w,
                               cudaMemcpyDeviceToHost, d->st));
  if (T)
    CUDA_TRY(cudaMemcpy2DAsync(T, ldt * 8, d->tstore + k * d->b * d->ld_t, d->ld_t * 8, w * 8, w,
                               cudaMemcpyDeviceToHost, d->st));
  CUDA_TRY(cudaStreamSynchronize(d->st));
  return 0;
}

ABFT_API int abft_dist_elapsed_ms(abft_dist* d, double* ms) {
  DevGuardD g(d->device);
  *ms = 0.0;
  if (!d->timed) return 0;
  CUDA_TRY(cudaEventSynchronize(d->e1));
  float f = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&f, d->e0, d->e1));
  *ms = f;
  return 0;
}

}  // extern "C"
