#pragma once
#include "common.cuh"

namespace abft {

// Diagonal-block factorization (w <= 256) + triangular inverses on one CTA.
// mode 0 = LU (no pivoting): Linv = L^{-1} (unit lower), Uinv = U^{-1}.
// mode 1 = Cholesky: Linv = L^{-1}; strict upper of D zeroed. Uinv ignored.
// *info_dev = 1 + (col_base + local column) of the first breakdown; left
// untouched (0) if none, and never overwritten once set.
int diag_factor(cudaStream_t st, double* D, int64_t ld, int w, int mode, double* Linv, int64_t ldl,
                double* Uinv, int64_t ldu, int* info_dev, int64_t col_base);
int diag_factor(cudaStream_t st, float* D, int64_t ld, int w, int mode, float* Linv, int64_t ldl,
                float* Uinv, int64_t ldu, int* info_dev, int64_t col_base);

// Householder panel (nk x w) in place: R above/on the diagonal, zeros below;
// V (nk x w, unit diagonal, zeros above) and betas (tau) out. part: >= 2*148*(w+1)
// doubles, rowbuf: >= 2*(w+1) doubles of device scratch.
// part2: >= 148*32*w doubles, wfin: >= 32*w doubles (shared-memory sub-panel
// kernel); null selects the whole-panel kernel.
int qr_panel(cudaStream_t st, double* P, int64_t ld, int64_t nk, int w, double* V, int64_t ldv,
             double* betas, double* part, int64_t part_elems, double* rowbuf, double* part2 = nullptr,
             double* wfin = nullptr);

// T factor (w x w upper) from Gm = V^T V and betas.
int larft(cudaStream_t st, const double* Gm, int64_t ldg, const double* betas, int w, double* T,
          int64_t ldt);

}  // namespace abft
