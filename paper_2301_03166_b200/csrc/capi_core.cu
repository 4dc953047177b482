// Library-level C-ABI entry points (no context): version, errors, device-pointer GEMM.
#include "abft_b200.h"
#include "gemm.cuh"

using namespace abft;

extern "C" {

ABFT_API int abft_version(void) { return 100; }

ABFT_API const char* abft_last_error(void) { return last_error(); }

ABFT_API int abft_device_count(int* count) {
  CUDA_TRY(cudaGetDeviceCount(count));
  return 0;
}

ABFT_API int abft_dev_dgemm(void* stream, char transa, char transb, int64_t m, int64_t n,
                            int64_t k, double alpha, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double beta, const double* C,
                            int64_t ldc, double* D, int64_t ldd) {
  if (m < 0 || n < 0 || k < 0 || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) {
    set_last_error("abft_dev_dgemm: bad dimensions");
    return ABFT_E_INVALID;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // split-K workspace: sized for the request, freed after the call
  GemmWorkspace ws;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int splits = gemm_splits_for((int)m, (int)n, (int)k, sms);
  if (splits > 1) {
    ws.elems = m * n * splits;
    CUDA_TRY(cudaMallocAsync(&ws.ptr, ws.elems * sizeof(double), st));
  }
  int rc = gemm(st, transa, transb, (int)m, (int)n, (int)k, alpha, A, lda, B, ldb, beta, C, ldc, D,
                ldd, &ws, splits);
  if (ws.ptr) cudaFreeAsync(ws.ptr, st);
  return rc;
}

}  // extern "C"
