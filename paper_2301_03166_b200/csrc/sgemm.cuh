#pragma once
#include "gemm.cuh"

namespace abft {

// fp32 GEMM on tcgen05 (kind::tf32, 3xTF32 split for fp32 accuracy):
// D(MxN) = beta*C + alpha*op(A)*op(B), column-major, ta/tb 'N' or 'T'.
// `ws` holds the split K-major operand copies (sgemm_workspace_elems floats).
// `fs` (optional): fused per-block checksums of D on a 128 x 128 grid (the
// block size must be 128; sums in fp64, written directly -- no strip
// scratch is used).
// `splits` > 1: split-K -- one launch runs (tile, K-slice) units, each
// slice's MMA chain accumulating separately (this also bounds the chain
// depth of the tensor core's truncating fp32 accumulation), then a
// fixed-order reduction adds the partials (workspace grows by splits*M*N).
int64_t sgemm_workspace_elems(int M, int N, int K, int splits = 1);
int64_t sgemm_partial_elems(int M, int N, int splits);
int sgemm_tc(cudaStream_t st, char ta, char tb, int M, int N, int K, float alpha, const float* A,
             int64_t lda, const float* B, int64_t ldb, float beta, const float* C, int64_t ldc,
             float* D, int64_t ldd, float* ws, int64_t ws_elems, const FusedSums* fs = nullptr,
             int max_ctas = 0, int splits = 1);

// hi/lo split of an R x K operand into K-major rows (hi[r * ldo + k]);
// trans = 0: src (r, k) at r + k*lds, 1: at k + r*lds. Columns K..kpad-1 = 0.
int sgemm_split_operand(cudaStream_t st, const float* src, int64_t lds, int R, int K, int kpad,
                        int trans, float* hi, float* lo, int64_t ldo);

// the GEMM over operands already split (A'(m, k) = ah[m * lda_k + k] + al[..],
// B'(n, k) likewise = op(B)(k, n)); `part` holds the split-K partials.
int sgemm_tc_presplit(cudaStream_t st, int M, int N, int K, float alpha, const float* ah,
                      const float* al, int64_t lda_k, const float* bh, const float* bl, int64_t ldb_k,
                      float beta, const float* C, int64_t ldc, float* D, int64_t ldd, float* part,
                      int64_t part_elems, int max_ctas = 0, int splits = 1);

}  // namespace abft
