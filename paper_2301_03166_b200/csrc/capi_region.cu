// Region-level ABFT on host arrays, executed on the current device:
// encode / maintain_gemm / verify_correct / inject_faults
// (/root/reference/pkg/src/slackwise/abft.py:118-307). These back the drop-in
// versions of the reference's module-level ABFT functions, which operate on
// caller-owned numpy arrays (pkg/tests/test_abft.py).
#include <algorithm>
#include <vector>

#include "abft_b200.h"
#include "abft_kernels.cuh"
#include "gemm.cuh"

using namespace abft;

namespace {

inline int64_t round_even(int64_t x) { return (x + 1) / 2 * 2; }

// RAII device buffer
struct DBuf {
  double* p = nullptr;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  int alloc(int64_t elems) {
    CUDA_TRY(cudaMalloc(&p, std::max<int64_t>(elems, 1) * sizeof(double)));
    return 0;
  }
};

int upload(DBuf& d, const double* h, int64_t ldh, int64_t rows, int64_t cols, int64_t ldd) {
  ABFT_TRY(d.alloc(ldd * std::max<int64_t>(cols, 1)));
  if (rows > 0 && cols > 0)
    CUDA_TRY(cudaMemcpy2D(d.p, ldd * 8, h, ldh * 8, rows * 8, cols, cudaMemcpyHostToDevice));
  return 0;
}

int download(const DBuf& d, int64_t ldd, double* h, int64_t ldh, int64_t rows, int64_t cols) {
  if (rows > 0 && cols > 0)
    CUDA_TRY(cudaMemcpy2D(h, ldh * 8, d.p, ldd * 8, rows * 8, cols, cudaMemcpyDeviceToHost));
  return 0;
}

}  // namespace

extern "C" {

ABFT_API int abft_region_encode(const double* m, int64_t ldm, int64_t rows, int64_t cols,
                                int64_t b, int scheme, double* col_plain, double* col_weighted,
                                double* row_plain, double* row_weighted) {
  if (scheme == ABFT_NONE) {
    set_last_error("cannot encode with scheme 'none'");
    return ABFT_E_INVALID;
  }
  if (rows <= 0 || cols <= 0) return 0;
  const int64_t nbr = (rows + b - 1) / b, nbc = (cols + b - 1) / b;
  const int64_t ld = round_even(rows);
  DBuf dm, cp, cw, rp, rw;
  ABFT_TRY(upload(dm, m, ldm, rows, cols, ld));
  ABFT_TRY(cp.alloc(nbr * cols));
  ABFT_TRY(cw.alloc(nbr * cols));
  ABFT_TRY(rp.alloc(rows * nbc));
  ABFT_TRY(rw.alloc(rows * nbc));
  Region reg{dm.p, ld, rows, cols, b};
  SumOut o;
  o.cp = cp.p;
  o.cp_ld = nbr;
  o.cp_step = 1;
  o.cw = cw.p;
  o.cw_ld = nbr;
  o.cw_step = 1;
  if (scheme == ABFT_FULL) {
    o.rp = rp.p;
    o.rp_ld = rows;
    o.rw = rw.p;
    o.rw_ld = rows;
  }
  ABFT_TRY(blocksum(nullptr, reg, o));
  CUDA_TRY(cudaDeviceSynchronize());
  ABFT_TRY(download(cp, nbr, col_plain, nbr, nbr, cols));
  ABFT_TRY(download(cw, nbr, col_weighted, nbr, nbr, cols));
  if (scheme == ABFT_FULL) {
    ABFT_TRY(download(rp, rows, row_plain, rows, rows, nbc));
    ABFT_TRY(download(rw, rows, row_weighted, rows, rows, nbc));
  }
  return 0;
}

// cs -= operand products (maintain_gemm): col sums from (1^T L_i) R and
// (w^T L_i) R; FULL row sums from L (R 1_j) and L (R w_j).
ABFT_API int abft_region_maintain(int64_t rows, int64_t cols, int64_t kdim, int64_t b, int scheme,
                                  const double* left, int64_t ldl, const double* right,
                                  int64_t ldr, double* col_plain, double* col_weighted,
                                  double* row_plain, double* row_weighted) {
  if (rows <= 0 || cols <= 0) return 0;
  const int64_t nbr = (rows + b - 1) / b, nbc = (cols + b - 1) / b;
  const int64_t ldL = round_even(rows), ldR = round_even(kdim);
  DBuf dL, dR, el, cs, er, erw, rs;
  ABFT_TRY(upload(dL, left, ldl, rows, kdim, ldL));
  ABFT_TRY(upload(dR, right, ldr, kdim, cols, ldR));
  // interleaved operand sums (2nbr x kdim) and checksums (2nbr x cols)
  const int64_t ldc = round_even(2 * nbr);
  ABFT_TRY(el.alloc(ldc * std::max<int64_t>(kdim, 1)));
  ABFT_TRY(cs.alloc(ldc * cols));
  std::vector<double> h(ldc * cols);
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t i = 0; i < nbr; ++i) {
      h[2 * i + c * ldc] = col_plain[i + c * nbr];
      h[2 * i + 1 + c * ldc] = col_weighted[i + c * nbr];
    }
  CUDA_TRY(cudaMemcpy(cs.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  if (kdim > 0) {
    Region rl{dL.p, ldL, rows, kdim, b};
    SumOut o;
    o.cp = el.p;
    o.cp_ld = ldc;
    o.cp_step = 2;
    o.cw = el.p + 1;
    o.cw_ld = ldc;
    o.cw_step = 2;
    ABFT_TRY(blocksum(nullptr, rl, o));
  }
  GemmWorkspace ws;
  ABFT_TRY(gemm(nullptr, 'N', 'N', (int)(2 * nbr), (int)cols, (int)kdim, -1.0, el.p, ldc, dR.p, ldR,
                1.0, cs.p, ldc, cs.p, ldc, &ws, 1));
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(h.data(), cs.p, h.size() * 8, cudaMemcpyDeviceToHost));
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t i = 0; i < nbr; ++i) {
      col_plain[i + c * nbr] = h[2 * i + c * ldc];
      col_weighted[i + c * nbr] = h[2 * i + 1 + c * ldc];
    }
  if (scheme == ABFT_FULL) {
    // R E_R: per block column plain and weighted row sums of R (kdim x nbc each)
    const int64_t ldk = round_even(std::max<int64_t>(kdim, 1));
    ABFT_TRY(er.alloc(ldk * nbc));
    ABFT_TRY(erw.alloc(ldk * nbc));
    if (kdim > 0) {
      Region rr{dR.p, ldR, kdim, cols, b};
      SumOut o;
      o.rp = er.p;
      o.rp_ld = ldk;
      o.rw = erw.p;
      o.rw_ld = ldk;
      ABFT_TRY(blocksum(nullptr, rr, o));
    }
    const int64_t ldrs = round_even(rows);
    ABFT_TRY(rs.alloc(ldrs * nbc));
    DBuf rsw;
    ABFT_TRY(rsw.alloc(ldrs * nbc));
    CUDA_TRY(cudaMemcpy2D(rs.p, ldrs * 8, row_plain, rows * 8, rows * 8, nbc, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy2D(rsw.p, ldrs * 8, row_weighted, rows * 8, rows * 8, nbc,
                          cudaMemcpyHostToDevice));
    ABFT_TRY(gemm(nullptr, 'N', 'N', (int)rows, (int)nbc, (int)kdim, -1.0, dL.p, ldL, er.p, ldk,
                  1.0, rs.p, ldrs, rs.p, ldrs, &ws, 1));
    ABFT_TRY(gemm(nullptr, 'N', 'N', (int)rows, (int)nbc, (int)kdim, -1.0, dL.p, ldL, erw.p, ldk,
                  1.0, rsw.p, ldrs, rsw.p, ldrs, &ws, 1));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy2D(row_plain, rows * 8, rs.p, ldrs * 8, rows * 8, nbc, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy2D(row_weighted, rows * 8, rsw.p, ldrs * 8, rows * 8, nbc,
                          cudaMemcpyDeviceToHost));
  }
  return 0;
}

ABFT_API int abft_region_verify(double* m, int64_t ldm, int64_t rows, int64_t cols, int64_t b,
                                int scheme, int correct, int64_t r0, int64_t c0,
                                const double* col_plain, const double* col_weighted,
                                const double* row_plain, abft_report* rep, abft_location* locs,
                                int max_locs) {
  if (rep) memset(rep, 0, sizeof(*rep));
  if (rows <= 0 || cols <= 0) return 0;
  if (scheme == ABFT_NONE) {
    set_last_error("cannot verify with scheme 'none'");
    return ABFT_E_INVALID;
  }
  const int64_t nbr = (rows + b - 1) / b, nbc = (cols + b - 1) / b;
  const int64_t ld = round_even(rows);
  DBuf dm, rcp, rcw, rrp, rbm, mcp, mcw, mrp;
  ABFT_TRY(upload(dm, m, ldm, rows, cols, ld));
  ABFT_TRY(rcp.alloc(nbr * cols));
  ABFT_TRY(rcw.alloc(nbr * cols));
  ABFT_TRY(rrp.alloc(rows * nbc));
  ABFT_TRY(rbm.alloc(nbr * nbc));
  ABFT_TRY(upload(mcp, col_plain, nbr, nbr, cols, nbr));
  ABFT_TRY(upload(mcw, col_weighted, nbr, nbr, cols, nbr));
  if (scheme == ABFT_FULL) ABFT_TRY(upload(mrp, row_plain, rows, rows, nbc, rows));
  Region reg{dm.p, ld, rows, cols, b};
  SumOut rec;
  rec.cp = rcp.p;
  rec.cp_ld = nbr;
  rec.cw = rcw.p;
  rec.cw_ld = nbr;
  rec.rp = rrp.p;
  rec.rp_ld = rows;
  rec.bm = rbm.p;
  rec.bm_ld = nbr;
  ABFT_TRY(blocksum(nullptr, reg, rec));
  Maintained mt;
  mt.cp = mcp.p;
  mt.cp_ld = nbr;
  mt.cp_step = 1;
  mt.cw = mcw.p;
  mt.cw_ld = nbr;
  mt.cw_step = 1;
  mt.rp = scheme == ABFT_FULL ? mrp.p : nullptr;
  mt.rp_ld = rows;
  Event* ev = nullptr;
  int32_t* cnt = nullptr;
  const int cap = 1 << 16;
  CUDA_TRY(cudaMalloc(&ev, cap * sizeof(Event)));
  CUDA_TRY(cudaMalloc(&cnt, 2 * sizeof(int32_t)));
  CUDA_TRY(cudaMemset(cnt, 0, 2 * sizeof(int32_t)));
  EventSink sink{ev, cnt, cap, nullptr, nullptr, 0, 0, 0, b};
  int rc = verify_blocks(nullptr, reg, b, scheme, correct, rec, mt, sink);
  int32_t h = 0;
  std::vector<Event> evs;
  if (!rc && cudaDeviceSynchronize() == cudaSuccess &&
      cudaMemcpy(&h, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost) == cudaSuccess) {
    if (h > cap) {
      set_last_error("event buffer overflow");
      rc = ABFT_E_OVERFLOW;
    } else {
      evs.resize(h);
      if (h > 0 && cudaMemcpy(evs.data(), ev, h * sizeof(Event), cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = -1000;
    }
  } else if (!rc) {
    set_last_error("verify failed: %s", cudaGetErrorString(cudaGetLastError()));
    rc = -1000;
  }
  cudaFree(ev);
  cudaFree(cnt);
  if (rc) return rc;
  std::sort(evs.begin(), evs.end(), [](const Event& a, const Event& bb) {
    if (a.bi != bb.bi) return a.bi < bb.bi;
    if (a.bj != bb.bj) return a.bj < bb.bj;
    return a.seq < bb.seq;
  });
  if (rep) rep->n_locations = (int32_t)evs.size();
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
      locs[i].row = e.row + r0;
      locs[i].col = e.col + c0;
      locs[i].kind = e.kind;
      locs[i].flag = e.flag;
      locs[i].detected_kind = e.detected_kind;
      locs[i].corrected = e.corrected;
      locs[i].uncorrectable = e.uncorrectable;
      locs[i].block_row = e.bi;
      locs[i].block_col = e.bj;
      locs[i].seq = e.seq;
    }
  }
  if (correct) ABFT_TRY(download(dm, ld, m, ldm, rows, cols));
  return 0;
}

ABFT_API int abft_inject(double* m, int64_t ldm, int64_t n_rows, int64_t n_cols,
                         const abft_fault* plan, int nplan, double scale) {
  if (nplan <= 0) return 0;
  for (int f = 0; f < nplan; ++f) {
    if (!(0 <= plan[f].row && plan[f].row < n_rows && 0 <= plan[f].col && plan[f].col < n_cols)) {
      set_last_error("fault at (%lld, %lld) outside matrix", (long long)plan[f].row,
                     (long long)plan[f].col);
      return ABFT_E_RANGE;
    }
  }
  const int64_t ld = round_even(n_rows);
  DBuf dm;
  ABFT_TRY(upload(dm, m, ldm, n_rows, n_cols, ld));
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
  DevFault* dp = nullptr;
  CUDA_TRY(cudaMalloc(&dp, nplan * sizeof(DevFault)));
  CUDA_TRY(cudaMemcpy(dp, h.data(), nplan * sizeof(DevFault), cudaMemcpyHostToDevice));
  int rc = inject(nullptr, dm.p, ld, n_rows, n_cols, dp, nplan, nullptr, 0, 0, 0, scale);
  if (!rc && cudaDeviceSynchronize() != cudaSuccess) rc = -1000;
  cudaFree(dp);
  if (rc) return rc;
  return download(dm, ld, m, ldm, n_rows, n_cols);
}

}  // extern "C"
