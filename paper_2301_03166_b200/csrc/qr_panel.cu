// Householder panel on the tensor cores (K5 QR panel, fast path).
//
// The reference factors the (n-p) x b panel column by column
// (/root/reference/pkg/src/slackwise/linalg.py:260-300): reflector j from
// x = panel[j:, j] with alpha = -copysign(||x||, x0 or 1), v scaled to v0 = 1,
// tau_j = beta v0^2; the rest of the panel gets H_j; T by the forward
// columnwise recurrence. On a B200 that loop is one grid-wide reduction per
// column. Here the same factorization comes out of GEMMs:
//
//   1. CholeskyQR2 (all tall work on the DMMA GEMM):
//        G1 = A^T A,  R1 = chol(G1),  Q1 = A R1^{-1}
//        G2 = Q1^T Q1, R2 = chol(G2), R = R2 R1, Q = Q1 R2^{-1}
//      (Q orthonormal to O(eps) when cond(A) << eps^{-1/2}, Yamamoto et al.)
//   2. Householder reconstruction (Ballard et al., "Reconstructing
//      Householder vectors from tall-skinny QR"): the unpivoted LU
//        Q - S = Y U   with s_j = -sign(pivot candidate) (|u_jj| >= 1)
//      gives V = Y (unit lower trapezoidal), T = -U S Y1^{-T}, and
//      R_hh = S R. With s_j = -sign(.) the reflectors are those of the
//      reference's sign rule (tau_j in [1, 2], R_jj = alpha), so V, T and R
//      equal the reference's up to rounding.
//   The bottom of V is one GEMM: V2 = Q1[w:] (U R2)^{-1}.
//
// Every step is asynchronous. Safety is decided on the device: the Cholesky
// breakdown test (diag_factor mode 1) or an orthogonality test on G2
// (w * max|G2 - I| >= 1/2, i.e. Q1 too far from orthonormal for one more
// pass to restore it) sets ws.info, the fast path then leaves the panel
// untouched, and the cooperative per-column panel + V^T V + larft run in its
// place (they return immediately when the fast path succeeded). Rank-deficient
// or zero columns (the reference's normx == 0 branches, :273-276) always take
// the exact fallback.
#include "gemm.cuh"
#include "panel.cuh"

namespace abft {

namespace {

constexpr int ORTHO_BAD = 1 << 24;

// info := ORTHO_BAD unless w * max|G - I| < 1/2 (all finite): one element
// per thread, any offender flags the panel (no reduction needed)
__global__ void __launch_bounds__(256) ortho_check_kernel(const double* G, int64_t ldg, int w,
                                                          int* info) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= w * w) return;
  const int i = idx % w, j = idx / w;
  const double v = G[i + (int64_t)j * ldg] - (i == j ? 1.0 : 0.0);
  if (!(fabs(v) * w < 0.5)) atomicCAS(info, 0, ORTHO_BAD);  // also catches NaN
}

// From the in-place modified LU X = Y \ U (strict lower Y, upper U) and s:
//   V[0:w, :] = unit lower Y with zeros above,  U = upper(X),
//   W = -S Y^{-T}  (W[i, j] = -s_i Yinv[j, i])  so that T = U W.
__global__ void recon_prep_kernel(const double* X, int64_t ldx, const double* Yinv,
                                  int64_t ldy, const double* sgn, int w, double* V, int64_t ldv,
                                  double* U, double* W, int64_t lds) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < w * w;
       idx += gridDim.x * blockDim.x) {
    const int i = idx % w, j = idx / w;
    const double x = X[i + (int64_t)j * ldx];
    V[i + (int64_t)j * ldv] = i > j ? x : (i == j ? 1.0 : 0.0);
    U[i + (int64_t)j * lds] = i <= j ? x : 0.0;
    W[i + (int64_t)j * lds] = -sgn[i] * Yinv[j + (int64_t)i * ldy];
  }
}

// betas = diag(T); if the fast path is valid (*info == 0): the panel becomes
// R_hh = S R on and above the diagonal and zeros below (linalg.py:289-290).
__global__ void recon_finish_kernel(const double* T, int64_t ldt, const double* R, int64_t ldr,
                                    const double* sgn, int w, int64_t m, double* betas, double* P,
                                    int64_t ld, const int* info) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid < w) betas[tid] = T[tid + tid * ldt];
  if (*info != 0) return;
  const int64_t total = m * w;
  for (int64_t idx = tid; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % m;
    const int j = (int)(idx / m);
    P[i + j * ld] = (i <= j) ? sgn[i] * R[i + (int64_t)j * ldr] : 0.0;
  }
}

// G = V^T V (w x w) for the fallback's larft, gated on *info != 0 (plain
// shared-memory tiles: it only runs for degenerate panels).
__global__ void __launch_bounds__(256) gram_gated_kernel(const double* V, int64_t ldv, int64_t m,
                                                         int w, double* G, int64_t ldg,
                                                         const int* info) {
  if (*info == 0) return;
  __shared__ double a[32][33], b[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 4 outputs
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t r0 = 0; r0 < m; r0 += 32) {
    for (int q = ty; q < 32; q += 8) {
      const int64_t r = r0 + tx;
      a[q][tx] = (r < m && i0 + q < w) ? V[r + (int64_t)(i0 + q) * ldv] : 0.0;
      b[q][tx] = (r < m && j0 + q < w) ? V[r + (int64_t)(j0 + q) * ldv] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int ii = ty + 8 * t;
      double s = 0.0;
      for (int l = 0; l < 32; ++l) s = fma(a[ii][l], b[tx][l], s);
      acc[t] += s;
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int ii = i0 + ty + 8 * t, jj = j0 + tx;
    if (ii < w && jj < w) G[ii + (int64_t)jj * ldg] = acc[t];
  }
}

bool coop_forced() {
  static const int v = [] {
    const char* e = getenv("ABFT_QR_PANEL");
    return (e && (e[0] == 'c' || e[0] == 'C')) ? 1 : 0;
  }();
  return v == 1;
}

int coop_panel(cudaStream_t st, double* P, int64_t ld, int64_t m, int w, double* V, int64_t ldv,
               double* T, int64_t ldt, double* betas, const QrPanelWork& ws, const int* gate) {
  ABFT_TRY(qr_panel(st, P, ld, m, w, V, ldv, betas, ws.part, ws.part_elems, ws.rowbuf, ws.part2,
                    ws.wfin, gate));
  if (gate) {
    count_launch();
    gram_gated_kernel<<<dim3((w + 31) / 32, (w + 31) / 32), 256, 0, st>>>(V, ldv, m, w, ws.gram,
                                                                         ws.ldg, gate);
    CUDA_TRY(cudaGetLastError());
  } else {
    ABFT_TRY(gemm(st, 'T', 'N', w, w, (int)m, 1.0, V, ldv, V, ldv, 0.0, nullptr, 0, ws.gram,
                  ws.ldg, ws.gws));
  }
  return larft(st, ws.gram, ws.ldg, betas, w, T, ldt, gate);
}

}  // namespace

int qr_panel_factor(cudaStream_t st, double* P, int64_t ld, int64_t m, int w, double* V,
                    int64_t ldv, double* T, int64_t ldt, double* betas, const QrPanelWork& ws,
                    int max_ctas) {
  if (w <= 0 || m <= 0) return 0;
  if (coop_forced() || !ws.q1 || !ws.small || !ws.info) {
    return coop_panel(st, P, ld, m, w, V, ldv, T, ldt, betas, ws, nullptr);
  }
  const int64_t s = ws.lds;
  double* G1 = ws.small + 0 * s * w;    // G1, then L1 in place
  double* L1i = ws.small + 1 * s * w;   // L1^{-1} = R1^{-T}
  double* G2 = ws.small + 2 * s * w;    // G2, then L2 in place
  double* L2i = ws.small + 3 * s * w;   // L2^{-1} = R2^{-T}
  double* X = ws.small + 4 * s * w;     // Q_top, then Y \ U in place
  double* Yi = ws.small + 5 * s * w;    // Y^{-1}
  double* Ui = ws.small + 6 * s * w;    // U^{-1}
  double* Mt = ws.small + 7 * s * w;    // R2^{-1} U^{-1}
  double* U = ws.small + 8 * s * w;     // upper(X)
  double* W = ws.small + 9 * s * w;     // -S Y^{-T}
  double* R = ws.small + 10 * s * w;    // R2 R1
  double* sg = ws.small + 11 * s * w;   // s (w)
  double* Q1 = ws.q1;
  const int64_t lq = ws.ldq;
  GemmWorkspace* g = ws.gws;
  const int mi = (int)m;
  CUDA_TRY(cudaMemsetAsync(ws.info, 0, sizeof(int), st));
  // the multi-CTA diagonal-block kernel needs ceil(w/32) co-resident SMs
  // (cooperative launch, anywhere on the chip): beside the look-ahead's
  // persistent GEMM it runs on the panel's reserved SMs
  auto dfac = [&](double* D, int mode, double* Li, double* Ui, double* sg) {
    return (max_ctas > 0 && max_ctas < (w + 31) / 32)
               ? diag_factor(st, D, s, w, mode, Li, s, Ui, s, ws.info, 0, sg)
               : diag_factor_fast(st, D, s, w, mode, Li, s, Ui, s, ws.info, 0, sg);
  };
  // CholeskyQR, pass 1
  ABFT_TRY(gemm_capped(st, 'T', 'N', w, w, mi, 1.0, P, ld, P, ld, 0.0, nullptr, 0, G1, s, g,
                       max_ctas));
  ABFT_TRY(dfac(G1, 1, L1i, nullptr, nullptr));
  ABFT_TRY(gemm_capped(st, 'N', 'T', mi, w, w, 1.0, P, ld, L1i, s, 0.0, nullptr, 0, Q1, lq, g,
                       max_ctas));
  // pass 2
  ABFT_TRY(gemm_capped(st, 'T', 'N', w, w, mi, 1.0, Q1, lq, Q1, lq, 0.0, nullptr, 0, G2, s, g,
                       max_ctas));
  count_launch();
  ortho_check_kernel<<<(w * w + 255) / 256, 256, 0, st>>>(G2, s, w, ws.info);
  CUDA_TRY(cudaGetLastError());
  ABFT_TRY(dfac(G2, 1, L2i, nullptr, nullptr));
  // R = R2 R1 = L2^T L1^T
  ABFT_TRY(gemm_capped(st, 'T', 'T', w, w, w, 1.0, G2, s, G1, s, 0.0, nullptr, 0, R, s, g,
                       max_ctas));
  // reconstruction: X = Q_top = Q1[0:w] R2^{-1}; Q_top - S = Y U
  ABFT_TRY(gemm_capped(st, 'N', 'T', w, w, w, 1.0, Q1, lq, L2i, s, 0.0, nullptr, 0, X, s, g,
                       max_ctas));
  ABFT_TRY(dfac(X, 2, Yi, Ui, sg));
  // V[w:m] = Q1[w:m] R2^{-1} U^{-1}
  ABFT_TRY(gemm_capped(st, 'T', 'N', w, w, w, 1.0, L2i, s, Ui, s, 0.0, nullptr, 0, Mt, s, g,
                       max_ctas));
  if (m > w)
    ABFT_TRY(gemm_capped(st, 'N', 'N', mi - w, w, w, 1.0, Q1 + w, lq, Mt, s, 0.0, nullptr, 0,
                         V + w, ldv, g, max_ctas));
  count_launch();
  recon_prep_kernel<<<std::max(1, std::min(64, (w * w + 255) / 256)), 256, 0, st>>>(
      X, s, Yi, s, sg, w, V, ldv, U, W, s);
  CUDA_TRY(cudaGetLastError());
  // T = -U S Y^{-T}
  ABFT_TRY(gemm_capped(st, 'N', 'N', w, w, w, 1.0, U, s, W, s, 0.0, nullptr, 0, T, ldt, g,
                       max_ctas));
  {
    const int64_t total = m * w;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
    if (max_ctas > 0) blocks = std::min(blocks, max_ctas * 8);
    count_launch();
    recon_finish_kernel<<<std::max(blocks, (w + 255) / 256), 256, 0, st>>>(
        T, ldt, R, s, sg, w, m, betas, P, ld, ws.info);
    CUDA_TRY(cudaGetLastError());
  }
  // exact fallback, a no-op unless the fast path flagged the panel
  return coop_panel(st, P, ld, m, w, V, ldv, T, ldt, betas, ws, ws.info);
}

}  // namespace abft
