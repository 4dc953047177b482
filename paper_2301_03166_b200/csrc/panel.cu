// Panel kernels (K5/K6): diagonal-block factorization + triangular inverses.
//
// The reference's panel decompositions are Python column loops
// (/root/reference/pkg/src/slackwise/linalg.py):
//   LU  unpivoted dgetf2 on the nk x b panel   :230-238
//   Chol Crout dpotf2 on the b x b block       :219-229
// and its panel updates solve against the diagonal block with LAPACK dgesv
//   Chol L21 = A21 L11^{-T}                     :246-252
//   LU   U12 = L11^{-1} A12                     :253-257
// B200 restatement: the w x w diagonal block is factored by ONE CTA with
// 32-column sub-panels staged in shared memory (the block is L2-resident),
// and the same CTA forms the triangular inverses. Everything tall-skinny
// (L21 = A21 U11^{-1}, L21 = A21 L11^{-T}, U12 = L11^{-1} A12) then runs as a
// DMMA GEMM over all SMs (gemm.cu), so the panel is GEMM-bound, not a
// per-column loop. Breakdown detection follows the reference exactly: LU
// pivot == 0 or non-finite (:234), Cholesky pivot <= 0 or non-finite (:223).
#include "panel.cuh"

#include <cooperative_groups.h>

namespace abft {

namespace {

constexpr int DT = 512;   // threads of the diagonal kernel
constexpr int NBK = 32;   // sub-panel width
constexpr int PLD = 257;  // smem leading dim of the staged sub-panel (w <= 256)
constexpr int DIAG_SMEM = (NBK * PLD + 224 * 33) * 8 + 64;   // bytes for fp64 (fp32 uses half)
constexpr int INV_SMEM = (256 * 33 + 32 * 257) * 8;

// Accessor for a (possibly transposed) column-major matrix.
template <typename T>
struct Acc {
  T* p;
  int64_t ld;
  bool t;
  ABFT_DEVINL T& at(int r, int c) const { return t ? p[c + r * ld] : p[r + c * ld]; }
};

// mode 0: LU without pivoting (L unit lower \ U upper in place),
//         Linv = L^{-1}, Uinv = U^{-1} (formed by tri_inverse_kernel).
// mode 1: Cholesky, L lower in place with the strict upper part zeroed.
// mode 2: LU of D - S with S = diag(s), s_c = -sign(pivot candidate) chosen
//         column by column (|pivot| >= 1, no breakdown): the modified LU of
//         the Householder reconstruction (qr_panel.cu); s written to sgn.
// info: 1 + global column of the first breakdown (atomicCAS, first wins).
// 512 threads viewed as 16 warps x 32 lanes: lanes walk rows, warps walk
// columns (no integer division in the inner loops); the trailing update of
// each 32-column sub-panel is register-blocked (7 rows x 2 columns / thread).
template <typename T>
__global__ void __launch_bounds__(DT, 1)
    diag_factor_kernel(T* D, int64_t ld, int w, int mode, T* Linv, int64_t ldl,
                       T* Uinv, int64_t ldu, int* info, int64_t col_base, T* sgn) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T* sm = reinterpret_cast<T*>(sm_raw);
  T* Ps = sm;                 // [NBK][PLD]  Ps[c*PLD + r]
  T* Rs = sm + NBK * PLD;     // [224][33]   Rs[c*33 + i]
  __shared__ int s_bad;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  if (tid == 0) s_bad = 0;
  __syncthreads();

  for (int jb = 0; jb < w; jb += NBK) {
    const int jw = min(NBK, w - jb);
    const int rem = w - jb;
    for (int c = ty; c < jw; c += DT / 32)
      for (int r = tx; r < rem; r += 32) Ps[c * PLD + r] = D[(jb + r) + (int64_t)(jb + c) * ld];
    __syncthreads();
    if (mode != 1) {
      // LU: the sub-panel lives in registers, one row per thread; per pivot
      // the owner of row c publishes it (double-buffered) and ONE barrier
      // separates the pivots (the shared-memory form needed three)
      T a[NBK];
      const bool own = tid < rem;
#pragma unroll
      for (int c = 0; c < NBK; ++c) a[c] = (own && c < jw) ? Ps[c * PLD + tid] : T(0);
      T* prow = Rs;  // [2][NBK] pivot rows (Rs is free during the panel phase)
      bool badf = false;
#pragma unroll
      for (int c = 0; c < NBK; ++c) {
        if (c < jw && !badf) {  // uniform across the CTA
          T* pr = prow + (c & 1) * NBK;
          if (tid == c) {
#pragma unroll
            for (int cc = c; cc < NBK; ++cc) pr[cc] = a[cc];
          }
          __syncthreads();
          T piv = pr[c];
          if (mode == 2) {
            // s = -sign(x) (x = -0.0 counts as +, as copysign(., x0 or 1) in linalg.py:278)
            const T sv = (piv < T(0)) ? T(1) : T(-1);
            piv -= sv;
            if (tid == c) a[c] = piv;
            if (tid == 0 && sgn) sgn[jb + c] = sv;
          }
          if (piv == T(0) || !isfinite(piv)) {
            badf = true;
            if (tid == 0) {
              s_bad = jb + c + 1;
              atomicCAS(info, 0, (int)(col_base + jb + c + 1));
            }
          } else if (own && tid > c) {
            const T l = a[c] / piv;
            a[c] = l;
#pragma unroll
            for (int cc = c + 1; cc < NBK; ++cc) a[cc] = fma(-l, pr[cc], a[cc]);
          }
        }
      }
      if (own && !badf) {
#pragma unroll
        for (int c = 0; c < NBK; ++c)
          if (c < jw) Ps[c * PLD + tid] = a[c];
      }
    }
    for (int c = 0; c < jw && mode == 1; ++c) {
      const T piv = Ps[c * PLD + c];
      const bool bad = (mode == 0) ? (piv == 0.0 || !isfinite(piv)) : (!(piv > 0.0) || !isfinite(piv));
      if (bad) {
        if (tid == 0) {
          s_bad = jb + c + 1;
          atomicCAS(info, 0, (int)(col_base + jb + c + 1));
        }
        break;  // uniform: every thread saw the same pivot
      }
      __syncthreads();
      if (mode == 0) {
        for (int r = c + 1 + tid; r < rem; r += DT) Ps[c * PLD + r] /= piv;
        __syncthreads();
        for (int cc = c + 1 + ty; cc < jw; cc += DT / 32) {
          const T u = Ps[cc * PLD + c];
          for (int r = c + 1 + tx; r < rem; r += 32) Ps[cc * PLD + r] -= Ps[c * PLD + r] * u;
        }
      } else {
        const T d = sqrt(piv);
        for (int r = c + tid; r < rem; r += DT) Ps[c * PLD + r] = (r == c) ? d : Ps[c * PLD + r] / d;
        __syncthreads();
        for (int cc = c + 1 + ty; cc < jw; cc += DT / 32) {
          const T u = Ps[c * PLD + cc];
          for (int r = cc + tx; r < rem; r += 32) Ps[cc * PLD + r] -= Ps[c * PLD + r] * u;
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (s_bad) return;
    for (int c = ty; c < jw; c += DT / 32)
      for (int r = tx; r < rem; r += 32)
        if (mode != 1 || r >= c) D[(jb + r) + (int64_t)(jb + c) * ld] = Ps[c * PLD + r];
    __syncthreads();
    const int ncols = w - jb - jw;
    if (ncols <= 0) continue;
    const T* Rop;  // right operand of the trailing update: R[l][c] = Rop[c*ldr + l]
    int ldr;
    if (mode != 1) {
      // U row block: R = L11^{-1} D[jb:jb+jw, jb+jw:w] (unit lower), one column per thread
      for (int c = ty; c < ncols; c += DT / 32)
        for (int i = tx; i < jw; i += 32) Rs[c * 33 + i] = D[(jb + i) + (int64_t)(jb + jw + c) * ld];
      __syncthreads();
      for (int c = tid; c < ncols; c += DT) {
        for (int i = 1; i < jw; ++i) {
          T x = Rs[c * 33 + i];
          for (int l = 0; l < i; ++l) x -= Ps[l * PLD + i] * Rs[c * 33 + l];
          Rs[c * 33 + i] = x;
        }
      }
      __syncthreads();
      for (int c = ty; c < ncols; c += DT / 32)
        for (int i = tx; i < jw; i += 32) D[(jb + i) + (int64_t)(jb + jw + c) * ld] = Rs[c * 33 + i];
      Rop = Rs;
      ldr = 33;
    } else {
      // Cholesky: R[l][c] = L21[c][l] = Ps[l*PLD + jw + c]  -> stage transposed in Rs
      for (int c = ty; c < ncols; c += DT / 32)
        for (int i = tx; i < jw; i += 32) Rs[c * 33 + i] = Ps[i * PLD + jw + c];
      __syncthreads();
      Rop = Rs;
      ldr = 33;
    }
    // trailing update D[jb+jw+r, jb+jw+c] -= sum_l P21[r][l] * R[l][c]
    const int nr = rem - jw;
    for (int c0 = 2 * ty; c0 < ncols; c0 += DT / 16) {
      T acc[7][2];
#pragma unroll
      for (int i = 0; i < 7; ++i) acc[i][0] = acc[i][1] = 0.0;
      const bool c1ok = c0 + 1 < ncols;
      for (int l = 0; l < jw; ++l) {
        const T r0v = Rop[c0 * ldr + l];
        const T r1v = c1ok ? Rop[(c0 + 1) * ldr + l] : 0.0;
#pragma unroll
        for (int i = 0; i < 7; ++i) {
          const int r = tx + 32 * i;
          const T pv = (r < nr) ? Ps[l * PLD + jw + r] : 0.0;
          acc[i][0] = fma(pv, r0v, acc[i][0]);
          acc[i][1] = fma(pv, r1v, acc[i][1]);
        }
      }
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        const int r = tx + 32 * i;
        if (r >= nr) continue;
        if (mode != 1 || r >= c0) D[(jb + jw + r) + (int64_t)(jb + jw + c0) * ld] -= acc[i][0];
        if (c1ok && (mode != 1 || r >= c0 + 1))
          D[(jb + jw + r) + (int64_t)(jb + jw + c0 + 1) * ld] -= acc[i][1];
      }
    }
    __syncthreads();
  }
  if (mode == 1) {
    for (int c = ty; c < w; c += DT / 32)
      for (int r = tx; r < c; r += 32) D[r + (int64_t)c * ld] = 0.0;
  }
}

// Triangular inverses, one CTA per 32-column block of the result:
// blockIdx.y = 0: X = L^{-1} (unit lower for LU, non-unit for Cholesky),
// blockIdx.y = 1: X = U^{-1}, computed as ((U^T)^{-1})^T through transposed
// accessors. Column block jb of X solves L X[:, jb] = E[:, jb] by block
// forward substitution: T = E - L[r0.., c0..r0] X[c0..r0, :] from shared
// memory (register-blocked), then a right-looking 32x32 solve in parallel.
template <typename T>
__global__ void __launch_bounds__(DT)
    tri_inverse_kernel(const T* D, int64_t ld, int w, int unit_l, T* Linv,
                       int64_t ldl, T* Uinv, int64_t ldu, const int* info) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T* sm = reinterpret_cast<T*>(sm_raw);
  if (*info != 0) return;  // factorization broke down: nothing to invert
  const bool upper = blockIdx.y == 1;
  if (upper && !Uinv) return;
  const Acc<T> L{const_cast<T*>(D), ld, upper};
  const Acc<T> X{upper ? Uinv : Linv, upper ? ldu : ldl, upper};
  const bool unit = upper ? false : (unit_l != 0);
  const int jb = blockIdx.x;
  const int c0 = jb * NBK;
  if (c0 >= w) return;
  const int cw = min(NBK, w - c0);
  T* Xs = sm;                // [w][33]: Xs[r*33 + c] = X(r, c0 + c), rows r >= c0
  T* Ls = sm + 256 * 33;     // [32][257]: Ls[r*257 + l] = L(r0 + r, c0 + l)
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  // rows above the diagonal block are zero
  for (int r = ty; r < c0; r += DT / 32)
    if (tx < cw) X.at(r, c0 + tx) = 0.0;
  for (int r0 = c0; r0 < w; r0 += NBK) {
    const int rh = min(NBK, w - r0);
    const int lw = r0 + rh - c0;
    for (int r = ty; r < rh; r += DT / 32)
      for (int l = tx; l < lw; l += 32)
        Ls[r * 257 + l] = (c0 + l <= r0 + r) ? L.at(r0 + r, c0 + l) : 0.0;
    __syncthreads();
    // T = E - L(r0.., c0..r0) X(c0..r0, :): thread (row ty*2+{0,1}, col tx)
    for (int rr = 2 * ty; rr < rh; rr += DT / 16) {
      T a0 = (r0 + rr == c0 + tx) ? 1.0 : 0.0;
      T a1 = (r0 + rr + 1 == c0 + tx) ? 1.0 : 0.0;
      if (tx < cw) {
        for (int l = 0; l < r0 - c0; ++l) {
          const T xv = Xs[l * 33 + tx];
          a0 -= Ls[rr * 257 + l] * xv;
          if (rr + 1 < rh) a1 -= Ls[(rr + 1) * 257 + l] * xv;
        }
        Xs[(r0 - c0 + rr) * 33 + tx] = a0;
        if (rr + 1 < rh) Xs[(r0 - c0 + rr + 1) * 33 + tx] = a1;
      }
    }
    __syncthreads();
    // L(r0..,r0..) Y = T, right-looking: row i final, eliminate it below
    for (int i = 0; i < rh; ++i) {
      if (!unit) {
        if (tid < cw) Xs[(r0 - c0 + i) * 33 + tid] /= Ls[i * 257 + (r0 + i - c0)];
        __syncthreads();
      }
      for (int idx = tid; idx < (rh - i - 1) * 32; idx += DT) {
        const int r = i + 1 + (idx >> 5), c = idx & 31;
        if (c < cw)
          Xs[(r0 - c0 + r) * 33 + c] -= Ls[r * 257 + (r0 + i - c0)] * Xs[(r0 - c0 + i) * 33 + c];
      }
      __syncthreads();
    }
  }
  for (int r = c0 + ty; r < w; r += DT / 32)
    if (tx < cw) X.at(r, c0 + tx) = Xs[(r - c0) * 33 + tx];
}

}  // namespace

template <typename T>
static int diag_factor_t(cudaStream_t st, T* D, int64_t ld, int w, int mode, T* Linv, int64_t ldl,
                         T* Uinv, int64_t ldu, int* info_dev, int64_t col_base, T* sgn) {
  if (w <= 0) return 0;
  if (w > 256) {
    set_last_error("diag_factor: block width %d > 256 (host-level blocking required)", w);
    return -1;
  }
  const int dsm = DIAG_SMEM / 8 * (int)sizeof(T) + 64;
  const int ism = INV_SMEM / 8 * (int)sizeof(T);
  ABFT_TRY(ensure_smem_attr((const void*)diag_factor_kernel<T>, dsm));
  count_launch();
  diag_factor_kernel<T><<<1, DT, dsm, st>>>(D, ld, w, mode, Linv, ldl, Uinv, ldu, info_dev,
                                            col_base, sgn);
  CUDA_TRY(cudaGetLastError());
  if (Linv || Uinv) {
    ABFT_TRY(ensure_smem_attr((const void*)tri_inverse_kernel<T>, ism));
    dim3 grid((w + NBK - 1) / NBK, Uinv ? 2 : 1);
    count_launch();
    tri_inverse_kernel<T><<<grid, DT, ism, st>>>(D, ld, w, mode != 1 ? 1 : 0, Linv, ldl, Uinv,
                                                 ldu, info_dev);
    CUDA_TRY(cudaGetLastError());
  }
  return 0;
}

int tri_inverse_lower(cudaStream_t st, const double* D, int64_t ld, int w, bool unit, double* Linv,
                      int64_t ldl, const int* info_dev) {
  if (w <= 0) return 0;
  const int ism = INV_SMEM;
  ABFT_TRY(ensure_smem_attr((const void*)tri_inverse_kernel<double>, ism));
  count_launch();
  tri_inverse_kernel<double><<<dim3((w + NBK - 1) / NBK, 1), DT, ism, st>>>(
      D, ld, w, unit ? 1 : 0, Linv, ldl, nullptr, 0, info_dev);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int diag_factor(cudaStream_t st, double* D, int64_t ld, int w, int mode, double* Linv, int64_t ldl,
                double* Uinv, int64_t ldu, int* info_dev, int64_t col_base, double* sgn) {
  return diag_factor_t(st, D, ld, w, mode, Linv, ldl, Uinv, ldu, info_dev, col_base, sgn);
}
int diag_factor(cudaStream_t st, float* D, int64_t ld, int w, int mode, float* Linv, int64_t ldl,
                float* Uinv, int64_t ldu, int* info_dev, int64_t col_base, float* sgn) {
  return diag_factor_t(st, D, ld, w, mode, Linv, ldl, Uinv, ldu, info_dev, col_base, sgn);
}

// ===========================================================================
// QR panel (K5 geqr2 + larft)
// ===========================================================================
// Householder panel factorization with the reference's LAPACK sign
// convention (linalg.py:260-300): alpha = -copysign(||x||, x0 or 1),
// v scaled so v0 = 1, tau = beta * v0^2, R on/above the diagonal and zeros
// below, V kept separately.
//
// One cooperative kernel over the whole panel with ONE grid-wide reduction
// per column: each CTA owns a contiguous row slab and contributes, in one
// pass, the partial sum of squares of x[1:] and the partial dot products
// x[1:] . P[1:, c] for every trailing panel column c. After the grid sync
// every CTA reduces the partials in a fixed order (deterministic), recovers
// alpha/beta and w[c] = dots[c] + v0 * P[j, c] (v differs from x only in its
// first entry), and applies the reflector to its own rows. The owner of row j
// publishes row j through the partial buffer, so no second sync is needed.
namespace {

constexpr int QT = 256;

__global__ void __launch_bounds__(QT)
    qr_panel_kernel(double* P, int64_t ld, int64_t nk, int w, double* V, int64_t ldv,
                    double* betas, double* part, double* rowbuf, const int* gate) {
  if (gate && *gate == 0) return;  // uniform over the grid: before any grid.sync
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double qsm[];
  double* wv = qsm;        // [w]
  double* rowj = qsm + w;  // [w]
  const int G = gridDim.x, gi = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rpc = (nk + G - 1) / G;
  const int64_t r_lo = min(nk, gi * rpc), r_hi = min(nk, r_lo + rpc);
  const int W1 = w + 1;

  for (int j = 0; j < w; ++j) {
    double* buf = part + (int64_t)(j & 1) * G * W1;
    double* rb = rowbuf + (j & 1) * W1;
    // ---- phase A: partials over own rows i > j ----
    const int64_t i0 = max(r_lo, (int64_t)j + 1);
    for (int c = j + warp; c < w; c += QT / 32) {
      double s = 0.0;
      for (int64_t i = i0 + lane; i < r_hi; i += 32) s = fma(P[i + j * ld], P[i + c * ld], s);
      s = warp_sum(s);
      if (lane == 0) buf[(int64_t)gi * W1 + (c - j)] = s;
    }
    if (j >= r_lo && j < r_hi) {
      for (int c = j + tid; c < w; c += QT) rb[c - j] = P[j + c * ld];
    }
    grid.sync();
    // ---- phase B: reduce (fixed order), reflector, update own rows ----
    for (int c = j + tid; c < w; c += QT) {
      double s = 0.0;
      for (int g2 = 0; g2 < G; ++g2) s += buf[(int64_t)g2 * W1 + (c - j)];
      wv[c] = s;
      rowj[c] = rb[c - j];
    }
    __syncthreads();
    const double s1 = wv[j];
    const double x0 = rowj[j];
    const double normx = sqrt(s1 + x0 * x0);
    const bool own_j = (j >= r_lo && j < r_hi);
    if (normx == 0.0) {
      if (tid == 0 && gi == 0) betas[j] = 0.0;
      for (int64_t i = r_lo + tid; i < r_hi; i += QT)
        if (i >= j) V[i + j * ldv] = (i == j) ? 1.0 : 0.0;
      __syncthreads();
      continue;
    }
    const double alpha = -copysign(normx, x0 != 0.0 ? x0 : 1.0);
    const double v0 = x0 - alpha;
    const double vn2 = s1 + v0 * v0;
    if (vn2 == 0.0) {
      if (tid == 0 && gi == 0) betas[j] = 0.0;
      if (own_j && tid == 0) P[j + j * ld] = alpha;
      for (int64_t i = r_lo + tid; i < r_hi; i += QT)
        if (i >= j) V[i + j * ldv] = (i == j) ? 1.0 : 0.0;
      __syncthreads();
      continue;
    }
    const double beta = 2.0 / vn2;
    __syncthreads();
    for (int c = j + 1 + tid; c < w; c += QT) wv[c] = wv[c] + v0 * rowj[c];
    __syncthreads();
    // rest -= beta * outer(v, w)  (linalg.py:287-288)
    const int64_t nrows = r_hi - max(r_lo, (int64_t)j);
    const int64_t rbeg = max(r_lo, (int64_t)j);
    const int ncols = w - j - 1;
    for (int64_t idx = tid; idx < nrows * ncols; idx += QT) {
      const int64_t i = rbeg + idx % nrows;
      const int c = j + 1 + (int)(idx / nrows);
      const double vi = (i == j) ? v0 : P[i + j * ld];
      P[i + c * ld] -= beta * (vi * wv[c]);
    }
    __syncthreads();
    for (int64_t i = rbeg + tid; i < r_hi; i += QT) {
      if (i == j) {
        P[j + j * ld] = alpha;
        V[j + j * ldv] = v0 / v0;
      } else {
        V[i + j * ldv] = P[i + j * ld] / v0;
        P[i + j * ld] = 0.0;
      }
    }
    if (tid == 0 && gi == 0) betas[j] = beta * v0 * v0;
    __syncthreads();
  }
}

// T (w x w, upper) from betas and Gm = V^T V (upper part used), forward
// columnwise dlarft (linalg.py:294-298) in blocked form:
//   diagonal 32x32 blocks by the column recurrence, then
//   T[0:j0, jb] = -T[0:j0, 0:j0] * (Gm[0:j0, jb] * T[jb, jb]).
__global__ void __launch_bounds__(512)
    larft_kernel(const double* Gm, int64_t ldg, const double* betas, int w, double* T,
                 int64_t ldt, const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double lsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nblk = (w + 31) / 32;
  // zero T
  for (int64_t idx = tid; idx < (int64_t)w * w; idx += blockDim.x)
    T[(idx % w) + (idx / w) * ldt] = 0.0;
  __syncthreads();
  // diagonal blocks: one warp per block (lane = row within block), the
  // block of Gm and the T block staged in shared memory
  for (int bk = warp; bk < nblk; bk += blockDim.x / 32) {
    const int j0 = bk * 32, jw = min(32, w - j0);
    double* Gs = lsm + (int64_t)bk * 2 * 32 * 33;  // Gs[r*33 + c] = Gm(j0 + r, j0 + c)
    double* Ts = Gs + 32 * 33;                     // Ts[r*33 + c] = T(j0 + r, j0 + c)
    for (int c = 0; c < 32; ++c) {
      Gs[lane * 33 + c] = (lane < jw && c < jw) ? Gm[(j0 + lane) + (int64_t)(j0 + c) * ldg] : 0.0;
      Ts[lane * 33 + c] = 0.0;
    }
    __syncwarp();
    for (int jj = 0; jj < jw; ++jj) {
      const double bj = betas[j0 + jj];
      if (lane < jj) {
        double s = 0.0;
        for (int l = lane; l < jj; ++l) s = fma(Ts[lane * 33 + l], Gs[l * 33 + jj], s);
        Ts[lane * 33 + jj] = -bj * s;
      }
      if (lane == 0) Ts[jj * 33 + jj] = bj;
      __syncwarp();
    }
    if (lane < jw)
      for (int c = lane; c < jw; ++c) T[(j0 + lane) + (int64_t)(j0 + c) * ldt] = Ts[lane * 33 + c];
  }
  __syncthreads();
  double* Ys = lsm;  // [j0][32]
  for (int bk = 1; bk < nblk; ++bk) {
    const int j0 = bk * 32, jw = min(32, w - j0);
    for (int idx = tid; idx < j0 * jw; idx += blockDim.x) {
      const int i = idx % j0, c = idx / j0;
      double s = 0.0;
      for (int l = 0; l <= c; ++l) s += Gm[i + (j0 + l) * ldg] * T[(j0 + l) + (j0 + c) * ldt];
      Ys[i + c * j0] = s;
    }
    __syncthreads();
    for (int idx = tid; idx < j0 * jw; idx += blockDim.x) {
      const int i = idx % j0, c = idx / j0;
      double s = 0.0;
      for (int l = i; l < j0; ++l) s += T[i + l * ldt] * Ys[l + c * j0];
      T[i + (j0 + c) * ldt] = -s;
    }
    __syncthreads();
  }
}


// Householder panel v2: 32-column sub-panels resident in shared memory.
// Every CTA owns a slab of <= QR_RMAX panel rows; for each sub-panel it keeps
// the slab of P and V in shared memory, and each column costs ONE grid-wide
// reduction of <= 32 values: the norm^2 of x[1:], the dots x[1:] . P[1:, c]
// with the remaining sub-panel columns, and the dots V[1:, l] . x[1:] with the
// sub-panel's previous reflectors (for its T). After the sub-panel, the
// remaining panel columns receive the block reflector I - V_s T_s V_s^T
// (two more grid syncs: reduce-scatter of V_s^T C, then gather).
constexpr int QR_RMAX = 256;   // max rows per CTA
constexpr int QR_RS = QR_RMAX + 1;
constexpr int QR_SMEM = (3 * 32 * QR_RS + 32 * 33 + 4 * 32) * 8;

__global__ void __launch_bounds__(QT, 1)
    qr_panel2_kernel(double* P, int64_t ld, int64_t nk, int w, double* V, int64_t ldv,
                     double* betas, double* part, double* rowbuf, double* part2, double* wfin,
                     const int* gate) {
  if (gate && *gate == 0) return;  // uniform over the grid: before any grid.sync
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double qs[];
  double* Ps = qs;                  // [32][QR_RS]  sub-panel slab, Ps[c*QR_RS + i]
  double* Vs = Ps + 32 * QR_RS;     // [32][QR_RS]
  double* Ws = Vs + 32 * QR_RS;     // [32][QR_RS]  W' = T_s^T V_s^T C, Ws[l*QR_RS + c]
  double* Ts = Ws + 32 * QR_RS;     // [32][33]     T_s (upper)
  double* red = Ts + 32 * 33;       // [32] reduced values
  double* rowj = red + 32;          // [32] row j of the sub-panel
  double* vrow = rowj + 32;         // [32] row j of V_s
  double* tcol = vrow + 32;         // [32] V_s^T v_j
  const int G = gridDim.x, gi = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rpc = (nk + G - 1) / G;
  const int64_t r_lo = min(nk, gi * rpc), r_hi = min(nk, r_lo + rpc);
  const int nr = (int)(r_hi - r_lo);

  for (int cs = 0; cs < w; cs += 32) {
    const int cw = min(32, w - cs);
    // ---- load the slab, zero V_s and T_s ----
    for (int idx = tid; idx < cw * nr; idx += QT) {
      const int c = idx / nr, i = idx % nr;
      Ps[c * QR_RS + i] = P[(r_lo + i) + (int64_t)(cs + c) * ld];
      Vs[c * QR_RS + i] = 0.0;
    }
    for (int idx = tid; idx < 32 * 33; idx += QT) Ts[idx] = 0.0;
    __syncthreads();
    for (int jj = 0; jj < cw; ++jj) {
      const int64_t j = cs + jj;  // panel row/col of the pivot
      double* buf = part + (int64_t)(j & 1) * G * 32;
      double* rb = rowbuf + (j & 1) * 64;
      // ---- phase A: partial reductions over own rows i > j ----
      const int i0 = (int)max((int64_t)0, j + 1 - r_lo);
      const int nv = cw;  // [0]: |x|^2, [1, cw-jj): dots with columns jj+1.., [cw-jj, cw): V dots
      for (int v = warp; v < nv; v += QT / 32) {
        double acc = 0.0;
        if (v == 0) {
          for (int i = i0 + lane; i < nr; i += 32) {
            const double x = Ps[jj * QR_RS + i];
            acc = fma(x, x, acc);
          }
        } else if (v < cw - jj) {
          const int c = jj + v;
          for (int i = i0 + lane; i < nr; i += 32) acc = fma(Ps[jj * QR_RS + i], Ps[c * QR_RS + i], acc);
        } else {
          const int l = v - (cw - jj);
          for (int i = i0 + lane; i < nr; i += 32) acc = fma(Vs[l * QR_RS + i], Ps[jj * QR_RS + i], acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) buf[(int64_t)gi * 32 + v] = acc;
      }
      if (j >= r_lo && j < r_hi) {
        const int il = (int)(j - r_lo);
        for (int c = tid; c < 32; c += QT) {
          rb[c] = (c >= jj && c < cw) ? Ps[c * QR_RS + il] : 0.0;
          rb[32 + c] = (c < jj) ? Vs[c * QR_RS + il] : 0.0;
        }
      }
      grid.sync();
      // ---- phase B: fixed-order reduction over the G partials (all threads:
      //      value = tid % 32, CTA subset = tid / 32; loads issued in parallel),
      //      reflector, update own rows ----
      {
        const int v = tid & 31, grp = tid >> 5;
        double acc = 0.0;
        if (v < nv) {
          double t[19];  // G <= 152 (148 SMs)
#pragma unroll
          for (int q2 = 0; q2 < 19; ++q2) {
            const int g2 = grp + 8 * q2;
            t[q2] = (g2 < G) ? buf[(int64_t)g2 * 32 + v] : 0.0;
          }
#pragma unroll
          for (int q2 = 0; q2 < 19; ++q2) acc += t[q2];
        }
        Ws[grp * 32 + v] = acc;  // Ws is free during the column loop
        __syncthreads();
        if (tid < nv) {
          double s = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < 8; ++q2) s += Ws[q2 * 32 + tid];
          red[tid] = s;
        }
      }
      if (tid < 32) {
        rowj[tid] = rb[tid];
        vrow[tid] = rb[32 + tid];
      }
      __syncthreads();
      const double s1 = red[0];
      const double x0 = rowj[jj];
      const double normx = sqrt(s1 + x0 * x0);
      double alpha = 0.0, v0 = 1.0, beta = 0.0;
      bool reflect = false;
      if (normx != 0.0) {
        alpha = -copysign(normx, x0 != 0.0 ? x0 : 1.0);
        v0 = x0 - alpha;
        const double vn2 = s1 + v0 * v0;
        if (vn2 != 0.0) {
          beta = 2.0 / vn2;
          reflect = true;
        }
      }
      const bool own_j = (j >= r_lo && j < r_hi);
      const int il_j = (int)(j - r_lo);
      if (!reflect) {
        // reference: normx == 0 -> betas 0, v = e_j; vn2 == 0 -> also panel[j, j] = alpha
        if (tid == 0 && gi == 0) betas[j] = 0.0;
        if (own_j && tid == 0) {
          Vs[jj * QR_RS + il_j] = 1.0;
          if (normx != 0.0) Ps[jj * QR_RS + il_j] = alpha;
        }
        __syncthreads();
        continue;  // T_s column jj stays zero (tau = 0)
      }
      const double tau = beta * v0 * v0;
      // w[c] = dots[c] + v0 * P[j, c]  for c in (jj, cw)
      if (tid > jj && tid < cw) red[tid - jj] = red[tid - jj] + v0 * rowj[tid];
      // T_s recurrence: t[l] = V_s[:, l]^T v_j = V_s[j, l] + (sum_{i>j} V_s[i, l] x_i) / v0
      if (tid < jj) tcol[tid] = vrow[tid] + red[(cw - jj) + tid] / v0;
      __syncthreads();
      if (tid < jj) {
        double acc = 0.0;
        for (int m = tid; m < jj; ++m) acc += Ts[tid * 33 + m] * tcol[m];
        Ts[tid * 33 + jj] = -tau * acc;
      }
      if (tid == 0) Ts[jj * 33 + jj] = tau;
      // rest -= beta * outer(v, w) over own rows i >= j
      const int ib = (int)max((int64_t)0, j - r_lo);
      const int ncc = cw - jj - 1;
      // warp per column, lanes over rows (no per-element div/mod)
      for (int cq = warp; cq < ncc; cq += QT / 32) {
        const int c = jj + 1 + cq;
        const double bw = red[c - jj];
        for (int i = ib + lane; i < nr; i += 32) {
          const double vi = (r_lo + i == j) ? v0 : Ps[jj * QR_RS + i];
          Ps[c * QR_RS + i] -= beta * (vi * bw);
        }
      }
      __syncthreads();
      for (int i = ib + tid; i < nr; i += QT) {
        if (r_lo + i == j) {
          Ps[jj * QR_RS + i] = alpha;
          Vs[jj * QR_RS + i] = v0 / v0;
        } else {
          Vs[jj * QR_RS + i] = Ps[jj * QR_RS + i] / v0;
          Ps[jj * QR_RS + i] = 0.0;
        }
      }
      if (tid == 0 && gi == 0) betas[j] = tau;
      __syncthreads();
    }
    // ---- write the sub-panel and its V back ----
    for (int idx = tid; idx < cw * nr; idx += QT) {
      const int c = idx / nr, i = idx % nr;
      P[(r_lo + i) + (int64_t)(cs + c) * ld] = Ps[c * QR_RS + i];
      V[(r_lo + i) + (int64_t)(cs + c) * ldv] = Vs[c * QR_RS + i];
    }
    const int ce = cs + cw;
    const int rem = w - ce;
    if (rem <= 0) break;
    // ---- block reflector on the remaining panel columns: C -= V_s T_s^T (V_s^T C) ----
    // C is processed in 32-column chunks staged in shared memory (Ws), so every
    // dot product runs out of shared memory.
    const int ib = (int)max((int64_t)0, (int64_t)cs - r_lo);  // V_s is zero above row cs
    for (int cc0 = 0; cc0 < rem; cc0 += 32) {
      const int ccw = min(32, rem - cc0);
      for (int c = warp; c < ccw; c += QT / 32)
        for (int i = ib + lane; i < nr; i += 32)
          Ws[c * QR_RS + i] = P[(r_lo + i) + (int64_t)(ce + cc0 + c) * ld];
      __syncthreads();
      for (int idx = tid; idx < cw * ccw; idx += QT) {
        const int l = idx / ccw, c = idx % ccw;
        double acc = 0.0;
        for (int i = ib; i < nr; ++i) acc = fma(Vs[l * QR_RS + i], Ws[c * QR_RS + i], acc);
        part2[((int64_t)gi * 32 + l) * rem + cc0 + c] = acc;
      }
      __syncthreads();
    }
    grid.sync();
    // reduce-scatter: CTA gi reduces a slice of the cw x rem entries (warp per entry)
    const int tot = cw * rem;
    const int per = (tot + G - 1) / G;
    for (int e = gi * per + warp; e < min(tot, (gi + 1) * per); e += QT / 32) {
      double acc = 0.0;
      for (int g2 = lane; g2 < G; g2 += 32) acc += part2[(int64_t)g2 * 32 * rem + e];
      acc = warp_sum(acc);
      if (lane == 0) wfin[e] = acc;
    }
    grid.sync();
    // W' = T_s^T W into Ps (the sub-panel slab is already written back)
    for (int idx = tid; idx < cw * rem; idx += QT) Ws[(idx / rem) * QR_RS + idx % rem] = wfin[idx];
    __syncthreads();
    for (int idx = tid; idx < cw * rem; idx += QT) {
      const int l = idx / rem, c = idx % rem;
      double acc = 0.0;
      for (int m = 0; m <= l; ++m) acc = fma(Ts[m * 33 + l], Ws[m * QR_RS + c], acc);
      Ps[l * QR_RS + c] = acc;
    }
    __syncthreads();
    // C(own rows) -= V_s W', chunk by chunk through shared memory
    for (int cc0 = 0; cc0 < rem; cc0 += 32) {
      const int ccw = min(32, rem - cc0);
      for (int c = warp; c < ccw; c += QT / 32)
        for (int i = ib + lane; i < nr; i += 32) {
          double acc = 0.0;
          for (int l = 0; l < cw; ++l) acc = fma(Vs[l * QR_RS + i], Ps[l * QR_RS + cc0 + c], acc);
          P[(r_lo + i) + (int64_t)(ce + cc0 + c) * ld] -= acc;
        }
    }
    grid.sync();  // the next sub-panel's slab load reads other CTAs' rows? no: own rows only,
                  // but wfin / part2 are reused by the next block update
  }
}

}  // namespace

int qr_panel(cudaStream_t st, double* P, int64_t ld, int64_t nk, int w, double* V, int64_t ldv,
             double* betas, double* part, int64_t part_elems, double* rowbuf, double* part2,
             double* wfin, const int* gate) {
  if (w <= 0 || nk <= 0) return 0;
  if (part2 && wfin) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // rows per CTA target (ABFT_QR_ROWS, default 64): more rows per CTA
    // means fewer CTAs in each per-column grid barrier and reduction
    static const int rows_t = [] {
      const char* e = getenv("ABFT_QR_ROWS");
      const int v = e ? atoi(e) : 0;
      return v >= 16 && v <= QR_RMAX ? v : 64;
    }();
    int G = (int)((nk + rows_t - 1) / rows_t);
    if (G > sms) G = sms;
    if (G > 152) G = 152;  // the per-column reduction reads 19 x 8 partials
    if ((nk + G - 1) / G <= QR_RMAX && 2LL * G * 32 <= part_elems) {
      ABFT_TRY(ensure_smem_attr((const void*)qr_panel2_kernel, QR_SMEM));
      void* args[] = {&P, &ld, &nk, &w, &V, &ldv, &betas, &part, &rowbuf, &part2, &wfin, &gate};
      count_launch();
      CUDA_TRY(cudaLaunchCooperativeKernel((void*)qr_panel2_kernel, dim3(G), dim3(QT), args,
                                           (size_t)QR_SMEM, st));
      return 0;
    }
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int G = (int)((nk + 63) / 64);
  if (G > sms) G = sms;
  const int64_t need = 2LL * G * (w + 1);
  if (need > part_elems) {
    G = (int)(part_elems / (2LL * (w + 1)));
    if (G < 1) {
      set_last_error("qr_panel: partial buffer too small");
      return -1;
    }
  }
  size_t smem = 2 * (size_t)w * sizeof(double);
  int max_per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_per_sm, qr_panel_kernel, QT, smem));
  if (max_per_sm < 1) {
    set_last_error("qr_panel: kernel cannot be resident");
    return -1;
  }
  void* args[] = {&P, &ld, &nk, &w, &V, &ldv, &betas, &part, &rowbuf, &gate};
  count_launch();
  CUDA_TRY(cudaLaunchCooperativeKernel((void*)qr_panel_kernel, dim3(G), dim3(QT), args, smem, st));
  return 0;
}

int larft(cudaStream_t st, const double* Gm, int64_t ldg, const double* betas, int w, double* T,
          int64_t ldt, const int* gate) {
  if (w <= 0) return 0;
  const size_t nblk = (size_t)(w + 31) / 32;
  size_t smem = std::max((size_t)w * 32, nblk * 2 * 32 * 33) * sizeof(double);
  if (smem > 200 * 1024) {
    set_last_error("larft: panel width %d too large", w);
    return -1;
  }
  ABFT_TRY(ensure_smem_attr((const void*)larft_kernel, 200 * 1024));
  count_launch();
  larft_kernel<<<1, 512, smem, st>>>(Gm, ldg, betas, w, T, ldt, gate);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace abft
