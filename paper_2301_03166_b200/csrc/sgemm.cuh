#pragma once
#include "gemm.cuh"

namespace abft {

// fp32 GEMM on tcgen05 (kind::tf32, 3xTF32 split for fp32 accuracy):
// D(MxN) = beta*C + alpha*op(A)*op(B), column-major, ta/tb 'N' or 'T'.
// `ws` holds the split K-major operand copies (sgemm_workspace_elems floats).
// `fs` (optional): fused per-block checksums of D on a 128 x 128 grid (the
// block size must be 128; sums in fp64, written directly -- no strip
// scratch is used).
int64_t sgemm_workspace_elems(int M, int N, int K);
int sgemm_tc(cudaStream_t st, char ta, char tb, int M, int N, int K, float alpha, const float* A,
             int64_t lda, const float* B, int64_t ldb, float beta, const float* C, int64_t ldc,
             float* D, int64_t ldd, float* ws, int64_t ws_elems, const FusedSums* fs = nullptr,
             int max_ctas = 0);

}  // namespace abft
