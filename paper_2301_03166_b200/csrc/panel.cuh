#pragma once
#include "common.cuh"

namespace abft {

// Diagonal-block factorization (w <= 256) + triangular inverses on one CTA.
// mode 0 = LU (no pivoting): Linv = L^{-1} (unit lower), Uinv = U^{-1}.
// mode 1 = Cholesky: Linv = L^{-1}; strict upper of D zeroed. Uinv ignored.
// mode 2 = LU of D - diag(s) with s_c = -sign(pivot candidate) (sgn out):
// the modified LU of the Householder reconstruction (qr_panel.cu).
// *info_dev = 1 + (col_base + local column) of the first breakdown; left
// untouched (0) if none, and never overwritten once set.
int diag_factor(cudaStream_t st, double* D, int64_t ld, int w, int mode, double* Linv, int64_t ldl,
                double* Uinv, int64_t ldu, int* info_dev, int64_t col_base, double* sgn = nullptr);
int diag_factor(cudaStream_t st, float* D, int64_t ld, int w, int mode, float* Linv, int64_t ldl,
                float* Uinv, int64_t ldu, int* info_dev, int64_t col_base, float* sgn = nullptr);

// Householder panel (nk x w) in place: R above/on the diagonal, zeros below;
// V (nk x w, unit diagonal, zeros above) and betas (tau) out. part: >= 2*148*(w+1)
// doubles, rowbuf: >= 2*(w+1) doubles of device scratch.
// part2: >= 148*32*w doubles, wfin: >= 32*w doubles (shared-memory sub-panel
// kernel); null selects the whole-panel kernel. gate: if non-null the kernel
// does nothing unless *gate != 0 (fallback of qr_panel_factor).
int qr_panel(cudaStream_t st, double* P, int64_t ld, int64_t nk, int w, double* V, int64_t ldv,
             double* betas, double* part, int64_t part_elems, double* rowbuf, double* part2 = nullptr,
             double* wfin = nullptr, const int* gate = nullptr);

// T factor (w x w upper) from Gm = V^T V and betas (gate as for qr_panel).
int larft(cudaStream_t st, const double* Gm, int64_t ldg, const double* betas, int w, double* T,
          int64_t ldt, const int* gate = nullptr);

// diag_factor on a thread-block cluster of ceil(w/32) CTAs (small_factor.cu):
// same contract, the inverses from the same launch; needs that many free SMs
// at once (side streams next to a persistent GEMM keep diag_factor).
// ABFT_NO_CLUSTER_FACTOR=1 routes it to diag_factor.
int diag_factor_fast(cudaStream_t st, double* D, int64_t ld, int w, int mode, double* Linv,
                     int64_t ldl, double* Uinv, int64_t ldu, int* info_dev, int64_t col_base,
                     double* sgn = nullptr);
int diag_factor_fast(cudaStream_t st, float* D, int64_t ld, int w, int mode, float* Linv,
                     int64_t ldl, float* Uinv, int64_t ldu, int* info_dev, int64_t col_base,
                     float* sgn = nullptr);

// L^{-1} of the lower triangle of the w x w block D (unit: unit diagonal);
// skipped if *info_dev != 0.
int tri_inverse_lower(cudaStream_t st, const double* D, int64_t ld, int w, bool unit, double* Linv,
                      int64_t ldl, const int* info_dev);

// LU with partial pivoting of the m x w panel P in place (LAPACK dgetf2
// semantics: ipiv[j] = panel-local row swapped with row j; L unit lower
// below, U on/above the diagonal), lu_pivot.cu. part: >= 2 (G+1)(w+2)
// doubles (G <= #SMs). info: 1 + col_base + column of an exactly singular
// (or non-finite) pivot.
int lu_panel_pivot(cudaStream_t st, double* P, int64_t ld, int64_t m, int w, int32_t* ipiv,
                   double* part, int64_t part_elems, int* info, int64_t col_base);
// Row interchanges ipiv[0..w) at rows k0.. applied to columns [c0, c0+ncols)
// (LAPACK dlaswp, in order; reverse: last first, i.e. P^T).
int laswp(cudaStream_t st, double* A, int64_t ld, int64_t c0, int64_t ncols, int64_t k0, int w,
          const int32_t* ipiv, bool reverse = false);

struct GemmWorkspace;

// Workspace of qr_panel_factor.
struct QrPanelWork {
  double* q1 = nullptr;     // >= m x w, leading dim ldq (the CholeskyQR2 Q)
  int64_t ldq = 0;
  double* small = nullptr;  // QR_SMALL_BUFS buffers of lds x w each
  int64_t lds = 0;
  int* info = nullptr;      // 1 device int: 0 = fast path valid, else exact fallback ran
  GemmWorkspace* gws = nullptr;
  // exact fallback (cooperative Householder panel + V^T V + larft)
  double* part = nullptr;
  int64_t part_elems = 0;
  double* rowbuf = nullptr;
  double* part2 = nullptr;
  double* wfin = nullptr;
  double* gram = nullptr;
  int64_t ldg = 0;
};
constexpr int QR_SMALL_BUFS = 12;

// The Householder panel of linalg.py:260-300 (R in place with zeros below, V
// unit lower trapezoidal, T upper, betas = diag T): CholeskyQR2 + Householder
// reconstruction on the tensor cores, with the cooperative per-column panel
// (qr_panel + larft) as the exact fallback when the Gram matrix is not safely
// positive definite (see qr_panel.cu). max_ctas caps every GEMM launch (the
// look-ahead runs it beside the trailing update). ABFT_QR_PANEL=coop forces
// the cooperative panel.
int qr_panel_factor(cudaStream_t st, double* P, int64_t ld, int64_t m, int w, double* V,
                    int64_t ldv, double* T, int64_t ldt, double* betas, const QrPanelWork& ws,
                    int max_ctas = 0);

}  // namespace abft
