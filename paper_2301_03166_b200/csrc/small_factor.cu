// Multi-CTA diagonal-block factorization (K5 PD, fast path).
//
// Same contract as diag_factor (panel.cuh): the w x w block D is factored in
// place -- LU unpivoted (linalg.py:230-238, mode 0), Cholesky (linalg.py:
// 219-229, mode 1) or the sign-shifted LU of the Householder reconstruction
// (mode 2, qr_panel.cu) -- and the triangular inverses L^{-1} (and U^{-1})
// come out of the same launch. diag_factor runs all of it on one CTA (a
// 32-column sub-panel loop: ~0.47 ms at w = 256 with its inverses); here CTA
// r of nb = ceil(w/32) co-resident CTAs (cooperative launch) owns block
// column r in its shared memory and the blocked right-looking algorithm runs
// across them:
//
//   step j:  CTA j factors its 32 x 32 diagonal block with one warp (rows in
//            registers, pivot row through shared memory, warp-level syncs),
//            inverts it (right-looking substitution), solves the rows below
//            against the inverse and publishes the block column and the
//            inverse blocks through global memory (L2);
//            grid barrier (an L2 counter);
//            CTA r > j pulls the panel from L2 and updates its block column
//            (LU: U_jr = L_jj^{-1} A_jr, A_ir -= L_ij U_jr; Cholesky:
//            A_ir -= L_ij L_rj^T); CTA r <= j advances block column r of
//            X = L^{-1} by the same elimination applied to the identity, so
//            the inverse costs no extra phase.
//   LU then forms U^{-1} by block back substitution over the final U columns.
//
// Round-2 history: the first version was a thread-block cluster pulling the
// panel over DSMEM (seven readers on one CTA's shared-memory port, ~21 B/cycle)
// with a register-resident 256-row pivot loop (~1000 cycles per pivot); the
// warp-level diagonal block, the L2 exchange and the cooperative launch (no
// GPC co-location, so it also runs beside a persistent GEMM that leaves a few
// SMs free) took w = 256 LU from 590 to 214 us (tools/probe/cf_trace.cu).
//
// w is padded to 32 nb with the identity (a block-diagonal extension that
// changes no pivot of the real block). Breakdown follows the reference: LU
// pivot == 0 or non-finite, Cholesky pivot <= 0 or non-finite; info gets
// 1 + (col_base + column) of the first one and nothing else is written.
#include <atomic>
#include <mutex>

#include "panel.cuh"

namespace abft {

namespace {


#ifdef CF_TRACE
__device__ long long g_cf_trace[8][64];
__device__ long long g_cf_clk[4];
#define CF_MARK(slot)                                                         \
  do {                                                                        \
    if (threadIdx.x == 0 && (slot) < 64) {                                    \
      long long t_;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      g_cf_trace[blockIdx.x][(slot)] = t_;                            \
    }                                                                         \
  } while (0)
#else
#define CF_MARK(slot) \
  do {                \
  } while (0)
#endif

constexpr int CF_T = 256;    // threads per CTA (8 warps)
constexpr int CF_MAXB = 8;   // CTAs (block columns) per launch: w <= 256
constexpr int TS = 33;       // stride of the 32 x 32 tiles

// Grid barrier of the nb co-resident CTAs (cooperative launch): sync[0]
// counts arrivals (monotonic; the host zeroes the slot before the launch),
// sync[1] carries the breakdown flag. Release/acquire through the L2.
ABFT_DEVINL void grid_barrier(int* sync, int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(sync, 1);
    int v;
    do {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(sync) : "memory");
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

ABFT_DEVINL int read_flag(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Out[i, c] -= sum_l A[i + l*lda] * B[l*TS + c] for rows i in [r0, r1)
// (r1 - r0 <= 224), c < 32. A may live in another CTA's shared memory.
template <typename T>
ABFT_DEVINL void tile_update(T* Out, int ldo, int r0, int r1, const T* A, int lda, const T* B) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  T acc[7][4];
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[q][e] = T(0);
#pragma unroll 4
  for (int l = 0; l < 32; ++l) {
    T b[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) b[e] = B[l * TS + ty * 4 + e];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const int i = r0 + tx + 32 * q;
      const T a = (i < r1) ? A[i + l * lda] : T(0);
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[q][e] = fma(a, b[e], acc[q][e]);
    }
  }
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const int i = r0 + tx + 32 * q;
    if (i < r1) {
#pragma unroll
      for (int e = 0; e < 4; ++e) Out[i + (ty * 4 + e) * ldo] -= acc[q][e];
    }
  }
}

// Dst[r0:r1, 0:32] (column stride ldd) = block column starting at global
// column c0 of the w x w matrix G (ld), rows r0..r1 (r1 - r0 <= 256), with
// the identity padding beyond w. Warp = 4 columns, lane = rows; all loads
// are issued before the stores (one L2 round trip).
template <typename T>
ABFT_DEVINL void global_block_column(T* Dst, int ldd, const T* G, int64_t ld, int w, int c0, int r0,
                                     int r1) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  T v[4][8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int gc = c0 + ty + 8 * q;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int i = r0 + tx + 32 * e;
      v[q][e] = (i < r1 && i < w && gc < w) ? __ldcg(G + i + (int64_t)gc * ld) : (i == gc ? T(1) : T(0));
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int i = r0 + tx + 32 * e;
      if (i < r1) Dst[i + (ty + 8 * q) * ldd] = v[q][e];
    }
}

// Tile (col-major, stride TS) = the 32 x 32 diagonal block at (c0, c0) of G
// (identity padding beyond w).
template <typename T>
ABFT_DEVINL void global_tile(T* Tile, const T* G, int64_t ld, int w, int c0) {
  for (int idx = threadIdx.x; idx < 32 * 32; idx += CF_T) {
    const int i = idx & 31, c = idx >> 5;
    Tile[i + c * TS] = (c0 + i < w && c0 + c < w) ? __ldcg(G + (c0 + i) + (int64_t)(c0 + c) * ld)
                                                  : (i == c ? T(1) : T(0));
  }
}

// Y[32j : 32j+32, :] = Tm (col-major, stride TS) * Y[32j : 32j+32, :]; the
// result also lands in B (row-major tile B[l*TS + c]) for the following
// rank-32 update. Ends with a barrier.
template <typename T>
ABFT_DEVINL void tile_tri_apply(T* Y, int ldy, int j, const T* Tm, T* B) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  T o[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll 8
  for (int l = 0; l < 32; ++l) {
    const T t = Tm[tx + l * TS];
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = fma(t, Y[(32 * j + l) + (ty * 4 + e) * ldy], o[e]);
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    Y[(32 * j + tx) + (ty * 4 + e) * ldy] = o[e];
    B[tx * TS + ty * 4 + e] = o[e];
  }
  __syncthreads();
}

// Inverse of the 32 x 32 diagonal block of a column block (rows 32j..), one
// warp, lane = result column. Right-looking substitution: as soon as x_k is
// final every pending partial sum takes its term (independent FMAs), so the
// dependent chain per step is one multiply + one FMA; the diagonal's
// reciprocals are formed up front (one division per lane, in parallel).
// lower: L^{-1} (unit: LU's L), else U^{-1} (upper, non-unit).
template <typename T>
__device__ __noinline__ void tile_inverse(const T* C, int ldc, int j, bool lower, bool unit, T* Out) {
  const int lane = threadIdx.x & 31;
  const T* Dg = C + 32 * j;
  const T rd_own = unit ? T(1) : T(1) / Dg[lane + lane * ldc];
  T x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? T(1) : T(0);
  if (lower) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const T rk = __shfl_sync(0xffffffffu, rd_own, k);
      x[k] *= rk;
#pragma unroll
      for (int i = k + 1; i < 32; ++i) x[i] = fma(-Dg[i + k * ldc], x[k], x[i]);
    }
  } else {
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      const T rk = __shfl_sync(0xffffffffu, rd_own, k);
      x[k] *= rk;
#pragma unroll
      for (int i = 0; i < k; ++i) x[i] = fma(-Dg[i + k * ldc], x[k], x[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) Out[i + lane * TS] = x[i];
}

// Factor the 32 x 32 diagonal block at rows c0.. of the block column (Cs,
// column stride Wp) in place, by ONE warp: lane t holds row t in registers.
// Per pivot: the pivot row (LU) or pivot column (Cholesky) goes through
// shared memory (pr, double-buffered: one __syncwarp per pivot), every lane
// forms one reciprocal, and rows above the pivot get a zero multiplier so
// the rank-1 update is unconditional (no selects); the breakdown test is
// tracked without branches (nothing is written back after a breakdown).
// MODE 0 LU, 2 sign-shifted LU (s -> sgn), 1 Cholesky (lower part
// meaningful). Returns the local column of the first breakdown or -1.
template <int MODE, typename T>
__device__ __noinline__ int diag_block_factor(T* Cs, int Wp, int c0, T* pr, T* sgn, int w) {
  const int t = threadIdx.x & 31;
  T* D = Cs + c0;
  T a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = D[t + c * Wp];
  int badc = -1;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    T* p = pr + (c & 1) * 32;
    if (MODE == 1) {
      if (t >= c) p[t] = a[c];  // column c of the diagonal block
      __syncwarp();
      const T piv = p[c];
      const bool brk = !(piv > T(0)) || !isfinite(piv);
      badc = (badc < 0 && brk) ? c : badc;
      const T d = sqrt(piv);
      const T rd = T(1) / d;
      const T l = (t > c) ? a[c] * rd : T(0);  // l_{t,c}
      a[c] = (t > c) ? l : (t == c ? d : a[c]);
#pragma unroll
      for (int cc = c + 1; cc < 32; ++cc) a[cc] = fma(-l, p[cc] * rd, a[cc]);  // l_{cc,c} = p[cc]/d
    } else {
      if (t == c) {
#pragma unroll
        for (int cc = c; cc < 32; ++cc) p[cc] = a[cc];  // pivot row
      }
      __syncwarp();
      T piv = p[c];
      if (MODE == 2) {
        // s = -sign(x), x = -0.0 counted as + (copysign(., x0 or 1), linalg.py:278)
        const T sv = (piv < T(0)) ? T(1) : T(-1);
        piv -= sv;
        if (t == c) a[c] = piv;
        if (t == 0 && sgn && c0 + c < w) sgn[c0 + c] = sv;
      }
      const bool brk = (piv == T(0)) || !isfinite(piv);
      badc = (badc < 0 && brk) ? c : badc;
      const T rp = T(1) / piv;
      const T l = (t > c) ? a[c] * rp : T(0);
      if (t > c) a[c] = l;
#pragma unroll
      for (int cc = c + 1; cc < 32; ++cc) a[cc] = fma(-l, p[cc], a[cc]);
    }
  }
  if (badc < 0) {
#pragma unroll
    for (int c = 0; c < 32; ++c) D[t + c * Wp] = a[c];
  }
  __syncwarp();
  return badc;
}

// Out[i, c] = sum_l Out[i, l] * B(l, c), B(l, c) = B[l*bl + c*bc], rows
// [r0, r1) (r1 - r0 <= 224): the panel solve L21 = A21 U11^{-1} (LU) or
// A21 L11^{-T} (Cholesky) against the inverted diagonal block.
template <typename T>
ABFT_DEVINL void tile_mul_inplace(T* Out, int ldo, int r0, int r1, const T* B, int bl, int bc) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  T acc[7][4];
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[q][e] = T(0);
#pragma unroll 4
  for (int l = 0; l < 32; ++l) {
    T b[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) b[e] = B[l * bl + (ty * 4 + e) * bc];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const int i = r0 + tx + 32 * q;
      const T a = (i < r1) ? Out[i + l * ldo] : T(0);
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[q][e] = fma(a, b[e], acc[q][e]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const int i = r0 + tx + 32 * q;
    if (i < r1) {
#pragma unroll
      for (int e = 0; e < 4; ++e) Out[i + (ty * 4 + e) * ldo] = acc[q][e];
    }
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(CF_T, 1)
    coop_factor_kernel(T* D, int64_t ld, int w, int mode, T* Linv, int64_t ldl, T* Uinv,
                          int64_t ldu, int* info, int64_t col_base, T* sgn, int* sync) {
  extern __shared__ __align__(16) unsigned char cf_raw[];
  const int nb = (int)gridDim.x;
  const int r = (int)blockIdx.x;
  int gen = 0;
  const int Wp = 32 * nb;  // padded order = column stride of Cs / Xs
  T* Cs = reinterpret_cast<T*>(cf_raw);  // block column r of the matrix
  T* Xs = Cs + 32 * Wp;                  // block column r of L^{-1}, then of U^{-1}
  T* Ps = Xs + 32 * Wp;                  // local copy of the step's panel
  T* Li = Ps + 32 * Wp;                  // L_rr^{-1} (col-major, stride TS)
  T* Ui = Li + 32 * TS;                  // U_rr^{-1}
  T* Lj = Ui + 32 * TS;                  // copy of the step's L_jj^{-1}
  T* Bt = Lj + 32 * TS;                  // right operand of the rank-32 update
  T* pr = Bt + 32 * TS;                  // [2][32] pivot rows
  int* s_bad = reinterpret_cast<int*>(pr + 64);
  const int tid = threadIdx.x, ty = tid >> 5;
  const bool lu = mode != 1;
  const int c0 = 32 * r;

  // load the block column (identity padding), X = I on block r
  // (warp per column, lane over rows: no integer division in these loops)
  for (int c = ty; c < 32; c += CF_T / 32)
    for (int i = tid & 31; i < Wp; i += 32) {
      const int gc = c0 + c;
      Cs[i + c * Wp] = (i < w && gc < w) ? D[i + (int64_t)gc * ld] : (i == gc ? T(1) : T(0));
      Xs[i + c * Wp] = (i == gc) ? T(1) : T(0);
    }
  if (tid == 0) *s_bad = 0;
  __syncthreads();

  bool bad = false;
  CF_MARK(0);
  for (int j = 0; j < nb && !bad; ++j) {
    if (r == j) {
      // ---- factor block column j: the diagonal block by one warp, its
      //      inverses by two, then the rows below against the inverse ----
      if (ty == 0) {
        const int badc = mode == 0   ? diag_block_factor<0>(Cs, Wp, c0, pr, sgn, w)
                         : mode == 1 ? diag_block_factor<1>(Cs, Wp, c0, pr, sgn, w)
                                     : diag_block_factor<2>(Cs, Wp, c0, pr, sgn, w);
        if (badc >= 0 && (tid & 31) == 0) {
          *s_bad = 1;
          if (c0 + badc < w) atomicCAS(info, 0, (int)(col_base + c0 + badc + 1));
        }
      }
      __syncthreads();
      CF_MARK(44 + 2 * j);
      if (*s_bad == 0) {
        if (ty == 0) tile_inverse(Cs, Wp, j, true, lu, Li);
        if (ty == 1 && lu) tile_inverse(Cs, Wp, j, false, false, Ui);
        __syncthreads();
        CF_MARK(45 + 2 * j);
        if (c0 + 32 < Wp) {
          if (lu)
            tile_mul_inplace(Cs, Wp, c0 + 32, Wp, Ui, 1, TS);   // L21 = A21 U11^{-1}
          else
            tile_mul_inplace(Cs, Wp, c0 + 32, Wp, Li, TS, 1);   // L21 = A21 L11^{-T}
        }
        // publish the final block column (rows >= 32j) and the diagonal
        // block's inverses through global memory (L2): the other CTAs read
        // them from there after the grid barrier (a DSMEM pull would put
        // seven readers on this CTA's shared-memory port)
        for (int c = ty; c < 32; c += CF_T / 32)
          for (int i = c0 + (tid & 31); i < Wp; i += 32)
            if (i < w && c0 + c < w) D[i + (int64_t)(c0 + c) * ld] = Cs[i + c * Wp];
        for (int idx = tid; idx < 32 * 32; idx += CF_T) {
          const int i = idx & 31, c = idx >> 5;
          if (c0 + i < w && c0 + c < w) {
            Linv[(c0 + i) + (int64_t)(c0 + c) * ldl] = Li[i + c * TS];
            if (lu) Uinv[(c0 + i) + (int64_t)(c0 + c) * ldu] = Ui[i + c * TS];
          }
        }
      }
      __syncthreads();
      CF_MARK(1 + 4 * j);
    }
    if (r == j && *s_bad && tid == 0) atomicExch(sync + 1, 1);
    grid_barrier(sync, ++gen * nb);  // panel j, its inverses and its flag are visible
    CF_MARK(2 + 4 * j);
    if (read_flag(sync + 1)) {
      bad = true;
      break;
    }
    const T* Pj = Cs;
    if (r != j) {
      global_block_column(Ps, Wp, D, ld, w, 32 * j, 32 * j, Wp);
      global_tile(Lj, Linv, ldl, w, 32 * j);
      Pj = Ps;
    } else {
      for (int idx = tid; idx < 32 * TS; idx += CF_T) Lj[idx] = Li[idx];
    }
    __syncthreads();
    CF_MARK(3 + 4 * j);
    if (r > j) {
      if (lu) {
        tile_tri_apply(Cs, Wp, j, Lj, Bt);  // U_jr
        tile_update(Cs, Wp, 32 * j + 32, Wp, Pj, Wp, Bt);
      } else {
        for (int idx = tid; idx < 32 * 32; idx += CF_T) {
          const int l = idx >> 5, cc = idx & 31;
          Bt[l * TS + cc] = Pj[(c0 + cc) + l * Wp];  // L_rj^T
        }
        __syncthreads();
        tile_update(Cs, Wp, c0, Wp, Pj, Wp, Bt);
      }
    } else {
      tile_tri_apply(Xs, Wp, j, Lj, Bt);
      if (32 * j + 32 < Wp) tile_update(Xs, Wp, 32 * j + 32, Wp, Pj, Wp, Bt);
    }
    __syncthreads();
    CF_MARK(4 + 4 * j);
  }
  CF_MARK(40);
  grid_barrier(sync, ++gen * nb);  // every block column final
  CF_MARK(41);
  if (!bad) {
    // factor out (Cholesky: lower part, zeros above)
    for (int c = ty; c < 32 && c0 + c < w; c += CF_T / 32)
      for (int i = tid & 31; i < w; i += 32) {
        const int gc = c0 + c;
        D[i + (int64_t)gc * ld] = (lu || i >= gc) ? Cs[i + c * Wp] : T(0);
        Linv[i + (int64_t)gc * ldl] = (i >= c0) ? Xs[i + c * Wp] : T(0);
      }
    if (lu && Uinv) {
      // U^{-1}, block column r: Y = E_r, then for j = r..0:
      //   Y_jr = U_jj^{-1} Y_jr,  Y_ir -= U_ij Y_jr (i < j)  (U_ij: block
      //   column j of the final factor, read back from D)
      grid_barrier(sync, ++gen * nb);  // every CTA's block column is in D
      for (int c = ty; c < 32; c += CF_T / 32)
        for (int i = tid & 31; i < Wp; i += 32) Xs[i + c * Wp] = (i == c0 + c) ? T(1) : T(0);
      __syncthreads();
      for (int j = r; j >= 0; --j) {
        const T* Uj = Cs;
        if (j != r) {
          global_tile(Lj, Uinv, ldu, w, 32 * j);
          if (j > 0) global_block_column(Ps, Wp, D, ld, w, 32 * j, 0, 32 * j);
          Uj = Ps;
        } else {
          for (int idx = tid; idx < 32 * TS; idx += CF_T) Lj[idx] = Ui[idx];
        }
        __syncthreads();
        tile_tri_apply(Xs, Wp, j, Lj, Bt);
        if (j > 0) tile_update(Xs, Wp, 0, 32 * j, Uj, Wp, Bt);
        __syncthreads();
      }
      for (int c = ty; c < 32 && c0 + c < w; c += CF_T / 32)
        for (int i = tid & 31; i < w; i += 32)
          Uinv[i + (int64_t)(c0 + c) * ldu] = (i < c0 + 32) ? Xs[i + c * Wp] : T(0);
    }
  }
  CF_MARK(42);
}

template <typename T>
size_t cf_smem_bytes(int nb) {
  return (size_t)(3 * 32 * 32 * nb + 4 * 32 * TS + 64) * sizeof(T) + 16;
}

// One barrier slot per launch (arrival counter + breakdown flag), zeroed on
// the launch's stream; 4096 slots in rotation.
__device__ int g_cf_sync[4096 * 2];

int* next_sync_slot() {
  static std::atomic<unsigned> ticket{0};
  static int* base = nullptr;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!base) {
      void* p = nullptr;
      if (cudaGetSymbolAddress(&p, g_cf_sync) != cudaSuccess) return nullptr;
      base = static_cast<int*>(p);
    }
  }
  return base + 2 * (ticket.fetch_add(1) % 4096u);
}

template <typename T>
int coop_factor_t(cudaStream_t st, T* D, int64_t ld, int w, int mode, T* Linv, int64_t ldl,
                     T* Uinv, int64_t ldu, int* info_dev, int64_t col_base, T* sgn) {
  const int nb = (w + 31) / 32;
  const size_t smem = cf_smem_bytes<T>(nb);
  ABFT_TRY(ensure_smem_attr((const void*)coop_factor_kernel<T>, (int)smem));
  int* sync = next_sync_slot();
  if (!sync) {
    set_last_error("coop_factor: barrier slots unavailable");
    return -1;
  }
  CUDA_TRY(cudaMemsetAsync(sync, 0, 2 * sizeof(int), st));
  // cooperative launch: the nb CTAs are co-resident (anywhere on the chip --
  // no GPC co-location as a thread-block cluster would need, so it also runs
  // beside a persistent GEMM that leaves a few SMs free)
  void* args[] = {&D, &ld, &w, &mode, &Linv, &ldl, &Uinv, &ldu, &info_dev, &col_base, &sgn, &sync};
  count_launch();
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)coop_factor_kernel<T>, dim3(nb), dim3(CF_T),
                                       args, smem, st));
  return 0;
}

bool cluster_disabled() {
  static const int v = [] {
    const char* e = getenv("ABFT_NO_CLUSTER_FACTOR");  // A/B knob: 1 = one-CTA diag_factor
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return v == 1;
}

}  // namespace

int diag_factor_fast(cudaStream_t st, double* D, int64_t ld, int w, int mode, double* Linv,
                     int64_t ldl, double* Uinv, int64_t ldu, int* info_dev, int64_t col_base,
                     double* sgn) {
  if (w <= 0) return 0;
  // the multi-CTA kernel exchanges panels / inverse blocks through D, Linv, Uinv
  if (w > 32 * CF_MAXB || cluster_disabled() || !Linv || (mode != 1 && !Uinv))
    return diag_factor(st, D, ld, w, mode, Linv, ldl, Uinv, ldu, info_dev, col_base, sgn);
  return coop_factor_t(st, D, ld, w, mode, Linv, ldl, Uinv, ldu, info_dev, col_base, sgn);
}

int diag_factor_fast(cudaStream_t st, float* D, int64_t ld, int w, int mode, float* Linv,
                     int64_t ldl, float* Uinv, int64_t ldu, int* info_dev, int64_t col_base,
                     float* sgn) {
  if (w <= 0) return 0;
  if (w > 32 * CF_MAXB || cluster_disabled() || !Linv || (mode != 1 && !Uinv))
    return diag_factor(st, D, ld, w, mode, Linv, ldl, Uinv, ldu, info_dev, col_base, sgn);
  return coop_factor_t(st, D, ld, w, mode, Linv, ldl, Uinv, ldu, info_dev, col_base, sgn);
}

}  // namespace abft
