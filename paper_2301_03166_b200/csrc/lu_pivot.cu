// LU with partial pivoting (option, BASELINE config C2).
//
// The reference factors LU without pivoting (linalg.py:230-238); its inputs
// are row-diagonally dominant (linalg.py:63-78), where partial pivoting picks
// the diagonal and changes nothing. For general inputs the drop-in offers
// LAPACK dgetrf semantics (P A = L U, ipiv as LAPACK's, 0-based): the tall
// panel is factored with partial pivoting by ONE cooperative kernel, one
// grid-wide barrier per column:
//
//   phase A (every CTA, its slab of panel rows): local argmax of |P[i, j]|
//            over rows i >= j (ties to the smallest row, as idamax), the
//            candidate row's full panel row published in the CTA's partial
//            slot; the owner of row j publishes row j;
//   -- grid.sync --
//   phase B (every CTA): fixed-order reduction of the G candidates -> pivot
//            row r and its values u; the owners of rows j and r swap them
//            (whole panel rows, the L part of earlier columns included);
//            every CTA scales its rows below j by 1/u_j and applies the
//            rank-1 update to the panel's remaining columns.
//
// laswp applies the panel's interchanges to the columns outside the panel
// (LAPACK dlaswp: in order; the reconstruction applies them in reverse).
#include <cooperative_groups.h>

#include "panel.cuh"

namespace abft {

namespace {

constexpr int PT = 256;  // threads per CTA (>= the grid size: phase B reads one candidate per thread)
constexpr int LU_RMAX = 512;  // rows per CTA slab (multipliers staged in shared memory)

// warp argmax of (value, row): ties to the smallest row
ABFT_DEVINL void argmax_warp(double& bv, int64_t& bi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) {
      bv = ov;
      bi = oi;
    }
  }
}

__global__ void __launch_bounds__(PT)
    lu_panel_pivot_kernel(double* P, int64_t ld, int64_t m, int w, int32_t* ipiv, double* part,
                          int* info, int64_t col_base) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, gi = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rpc = (m + G - 1) / G;
  const int64_t r_lo = min(m, gi * rpc), r_hi = min(m, r_lo + rpc);
  // partial slot of CTA g for column parity q: [val, idx, row values (w)]
  const int64_t slot = 2 + w;
  __shared__ double s_val[PT / 32];
  __shared__ int64_t s_idx[PT / 32];
  __shared__ double s_u[256];
  __shared__ double s_rowj[256];
  __shared__ double s_l[LU_RMAX];
  __shared__ int64_t s_grp[PT / 32];
  __shared__ int64_t s_piv;
  __shared__ int s_win;
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  for (int j = 0; j < w; ++j) {
    double* buf = part + (int64_t)(j & 1) * (G + 1) * slot;
    // ---- phase A: local argmax over own rows >= j (NaN counts as +inf so a
    //      NaN column reaches the breakdown test; ties to the smallest row) ----
    double bv = -1.0;
    int64_t bi = -1;
    for (int64_t i = max(r_lo, (int64_t)j) + tid; i < r_hi; i += PT) {
      const double x = fabs(P[i + (int64_t)j * ld]);
      const double v = (x != x) ? INFINITY : x;
      if (v > bv) {  // rows visit in increasing order: the first max is kept
        bv = v;
        bi = i;
      }
    }
    argmax_warp(bv, bi);
    if (lane == 0) {
      s_val[warp] = bv;
      s_idx[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double v = -1.0;
      int64_t ix = -1;
      for (int q = 0; q < PT / 32; ++q)
        if (s_idx[q] >= 0 && (ix < 0 || s_val[q] > v || (s_val[q] == v && s_idx[q] < ix))) {
          v = s_val[q];
          ix = s_idx[q];
        }
      buf[(int64_t)gi * slot + 0] = v;
      buf[(int64_t)gi * slot + 1] = (double)ix;
      s_piv = ix;
    }
    __syncthreads();
    if (s_piv >= 0)
      for (int c = tid; c < w; c += PT) buf[(int64_t)gi * slot + 2 + c] = P[s_piv + (int64_t)c * ld];
    if (j >= r_lo && j < r_hi)  // row j (its old values) in the extra slot G
      for (int c = tid; c < w; c += PT) buf[(int64_t)G * slot + 2 + c] = P[j + (int64_t)c * ld];
    grid.sync();
    // ---- phase B: the pivot (block-parallel fixed-order argmax over the G
    //      candidates), the interchange, the rank-1 update ----
    {
      double v = -1.0;
      int64_t ix = -1;
      if (tid < G) {
        ix = (int64_t)buf[(int64_t)tid * slot + 1];
        v = ix >= 0 ? buf[(int64_t)tid * slot + 0] : -1.0;
      }
      // argmax over (value, candidate row): ties to the smallest row
      int64_t g = ix >= 0 ? tid : -1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, ix, o);
        const int64_t og = __shfl_xor_sync(0xffffffffu, g, o);
        if (oi >= 0 && (ix < 0 || ov > v || (ov == v && oi < ix))) {
          v = ov;
          ix = oi;
          g = og;
        }
      }
      if (lane == 0) {
        s_val[warp] = v;
        s_idx[warp] = ix;
        s_grp[warp] = g;
      }
      __syncthreads();
      if (tid == 0) {
        double bv2 = -1.0;
        int64_t bx = -1, bg = -1;
        for (int q = 0; q < PT / 32; ++q)
          if (s_idx[q] >= 0 && (bx < 0 || s_val[q] > bv2 || (s_val[q] == bv2 && s_idx[q] < bx))) {
            bv2 = s_val[q];
            bx = s_idx[q];
            bg = s_grp[q];
          }
        s_piv = bx < 0 ? j : bx;
        s_win = (int)bg;
      }
      __syncthreads();
      const int wg = s_win;
      for (int c = tid; c < w; c += PT) {
        s_u[c] = wg < 0 ? 0.0 : buf[(int64_t)wg * slot + 2 + c];
        s_rowj[c] = buf[(int64_t)G * slot + 2 + c];
      }
      __syncthreads();
      if (tid == 0) {
        const double piv = s_u[j];
        if (!(piv != 0.0) || !isfinite(piv)) {
          s_bad = 1;
          if (gi == 0) {
            atomicCAS(info, 0, (int)(col_base + j + 1));
            // the columns after the breakdown are not factored: no interchanges
            // (laswp still runs on them; stale ipiv entries sent it out of bounds)
            for (int jj = j + 1; jj < w; ++jj) ipiv[jj] = (int32_t)jj;
          }
        }
        if (gi == 0) ipiv[j] = (int32_t)s_piv;
      }
      __syncthreads();
    }
    if (s_bad) return;  // uniform across the grid: every CTA saw the same pivot
    const int64_t r = s_piv;
    const double piv = s_u[j];
    if (r != j) {
      if (j >= r_lo && j < r_hi)
        for (int c = tid; c < w; c += PT) P[j + (int64_t)c * ld] = s_u[c];
      if (r >= r_lo && r < r_hi)
        for (int c = tid; c < w; c += PT) P[r + (int64_t)c * ld] = s_rowj[c];
    }
    __syncthreads();
    // rows below j in this slab: l = x / piv (multipliers staged in shared
    // memory), then rest -= l * u with warps over columns and lanes over rows
    // (independent coalesced read-modify-writes: no serial latency chain)
    const int64_t ib = max(r_lo, (int64_t)j + 1);
    const int nr = (int)max((int64_t)0, r_hi - ib);
    const double rp = 1.0 / piv;
    for (int t = tid; t < nr; t += PT) {
      const int64_t i = ib + t;
      const double l = P[i + (int64_t)j * ld] * rp;
      P[i + (int64_t)j * ld] = l;
      s_l[t] = l;
    }
    __syncthreads();
    for (int c = j + 1 + warp; c < w; c += PT / 32) {
      const double u = s_u[c];
      double* col = P + (int64_t)c * ld + ib;
      for (int t = lane; t < nr; t += 32) col[t] = fma(-s_l[t], u, col[t]);
    }
    // the next column's phase A reads only this CTA's rows: no barrier needed
    // beyond the block-level one below (s_u / s_rowj are rewritten next column)
    __syncthreads();
  }
}

// A[k0 + j, c] <-> A[k0 + ipiv[j], c] for j in order (reverse: last first),
// columns [c0, c0 + ncols): one thread per column.
__global__ void laswp_kernel(double* A, int64_t ld, int64_t c0, int64_t ncols, int64_t k0, int w,
                             const int32_t* ipiv, int reverse) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols;
       c += (int64_t)gridDim.x * blockDim.x) {
    double* col = A + (c0 + c) * ld + k0;
    for (int t = 0; t < w; ++t) {
      const int j = reverse ? w - 1 - t : t;
      const int64_t r = ipiv[j];
      if (r != j) {
        const double x = col[j];
        col[j] = col[r];
        col[r] = x;
      }
    }
  }
}

}  // namespace

int lu_panel_pivot(cudaStream_t st, double* P, int64_t ld, int64_t m, int w, int32_t* ipiv,
                   double* part, int64_t part_elems, int* info, int64_t col_base) {
  if (w <= 0 || m <= 0) return 0;
  if (w > 256) {
    set_last_error("lu_panel_pivot: panel width %d > 256", w);
    return -1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int G = (int)std::min<int64_t>((m + 63) / 64, sms);
  while (G > 1 && 2LL * (G + 1) * (2 + w) > part_elems) --G;
  if (2LL * (G + 1) * (2 + w) > part_elems || (m + G - 1) / G > LU_RMAX) {
    set_last_error("lu_panel_pivot: panel of %lld rows too tall for %d CTAs", (long long)m, G);
    return -1;
  }
  void* args[] = {&P, &ld, &m, &w, &ipiv, &part, &info, &col_base};
  count_launch();
  CUDA_TRY(cudaLaunchCooperativeKernel((void*)lu_panel_pivot_kernel, dim3(G), dim3(PT), args, 0, st));
  return 0;
}

int laswp(cudaStream_t st, double* A, int64_t ld, int64_t c0, int64_t ncols, int64_t k0, int w,
          const int32_t* ipiv, bool reverse) {
  if (ncols <= 0 || w <= 0) return 0;
  const int blocks = (int)std::min<int64_t>((ncols + 127) / 128, 1184);
  count_launch();
  laswp_kernel<<<blocks, 128, 0, st>>>(A, ld, c0, ncols, k0, w, ipiv, reverse ? 1 : 0);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace abft
