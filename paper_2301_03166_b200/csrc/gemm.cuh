#pragma once
#include "common.cuh"

namespace abft {

// Checksum outputs of the fused epilogue for an fb x fb block grid over D:
// col plain cp[cp_step*bi + col*cp_ld], col weighted cw[...], row plain
// rp[row + bj*rp_ld], block max bm[bi + bj*bm_ld] (all block-local indexing
// relative to D's origin). The GEMM's work unit is a 64-column strip of a
// block, so row sums and the block max are first written per strip into the
// scratch arrays rpp[row + (bj*fb/64 + s)*rpp_ld] and bmp[bi + (...)*bmp_ld]
// (M x nbc*fb/64 and nbr x nbc*fb/64) and combined in a fixed order.
struct FusedSums {
  double* cp = nullptr;
  int64_t cp_ld = 0, cp_step = 1;
  double* cw = nullptr;
  int64_t cw_ld = 0, cw_step = 1;
  double* rp = nullptr;
  int64_t rp_ld = 0;
  double* bm = nullptr;
  int64_t bm_ld = 0;
  double* rpp = nullptr;  // per-strip row sums (scratch)
  int64_t rpp_ld = 0;
  double* bmp = nullptr;  // per-strip max|x| (scratch)
  int64_t bmp_ld = 0;
};

struct GemmWorkspace {
  double* ptr = nullptr;
  int64_t elems = 0;
};

// D(MxN) = beta*C + alpha*op(A)*op(B), all column-major fp64 on the device.
// ta/tb: 'N' or 'T'. C may alias D (in-place update). splits <= 0 picks a
// split-K factor automatically (needs workspace, else falls back to 1).
int gemm(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, const double* C, int64_t ldc,
         double* D, int64_t ldd, GemmWorkspace* ws, int splits = 0);

int gemm_splits_for(int M, int N, int K, int num_sms);

// As gemm() (no split-K) but the epilogue also produces the per-block
// checksums of D on an fb x fb grid (fb = 128 or 256): the verify-side read
// of encode/verify_correct without a separate pass over D.
int gemm_fused_sums(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                    const double* C, int64_t ldc, double* D, int64_t ldd, int fb,
                    const FusedSums& sums, int max_ctas = 0);
bool gemm_can_fuse(int fb);
// split-K factor gemm() would use for this shape and workspace
int gemm_effective_splits(int M, int N, int K, const GemmWorkspace* ws, int splits = 0,
                          int max_ctas = 0);

// gemm() (split-K allowed) on at most max_ctas SMs per launch
int gemm_capped(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha,
                const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                const double* C, int64_t ldc, double* D, int64_t ldd, GemmWorkspace* ws,
                int max_ctas);

// gemm() without split-K on at most max_ctas SMs (leaves SMs for a concurrent
// side-stream kernel).
int gemm_reserved(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha,
                  const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                  const double* C, int64_t ldc, double* D, int64_t ldd, int max_ctas);

}  // namespace abft
