#pragma once
#include "common.cuh"

namespace abft {

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

}  // namespace abft
