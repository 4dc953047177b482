// Library-level C-ABI entry points (no context): version, errors, device-pointer GEMM.
#include "abft_b200.h"
#include "abft_kernels.cuh"
#include "gemm.cuh"
#include "panel.cuh"
#include "sgemm.cuh"

using namespace abft;

namespace {
// Register-resident DMMA loop: 8 independent accumulators per warp.
__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
  double s = 0.0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5678) out[0] = s;
}
}  // namespace

extern "C" {

ABFT_API int abft_version(void) { return 100; }

ABFT_API long long abft_launch_count(void) { return launch_count(); }

ABFT_API int abft_noise_stats(int enable) {
  noise_stats_enable(enable != 0);
  return 0;
}

ABFT_API int abft_noise_read(double* out3, int reset) { return noise_stats_read(out3, reset != 0); }

ABFT_API const char* abft_last_error(void) { return last_error(); }

ABFT_API int abft_device_count(int* count) {
  CUDA_TRY(cudaGetDeviceCount(count));
  return 0;
}

ABFT_API int abft_probe_dmma_peak(int iters, double* tflops) {
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  CUDA_TRY(cudaMalloc(&out, sizeof(double)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int warps = 16, blocks = 2 * sms;
  count_launch();
  dmma_peak_kernel<<<blocks, warps * 32>>>(out, iters / 10 + 1);  // warm-up
  cudaEventRecord(e0);
  count_launch();
  dmma_peak_kernel<<<blocks, warps * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  CUDA_TRY(err);
  const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * warps;
  *tflops = flops / (ms * 1e-3) / 1e12;
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

// fp32 device-pointer GEMM on tcgen05 (3xTF32): D = beta*C + alpha*op(A)*op(B)
ABFT_API int abft_dev_sgemm_splitk(void* stream, char transa, char transb, int64_t m, int64_t n,
                                   int64_t k, float alpha, const float* A, int64_t lda,
                                   const float* B, int64_t ldb, float beta, const float* C,
                                   int64_t ldc, float* D, int64_t ldd, int splits) {
  if (m < 0 || n < 0 || k < 1 || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX || splits < 1) {
    set_last_error("abft_dev_sgemm: bad dimensions");
    return ABFT_E_INVALID;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t wse = sgemm_workspace_elems((int)m, (int)n, (int)k, splits);
  float* ws = nullptr;
  CUDA_TRY(cudaMallocAsync(&ws, wse * sizeof(float), st));
  int rc = sgemm_tc(st, transa, transb, (int)m, (int)n, (int)k, alpha, A, lda, B, ldb, beta, C, ldc,
                    D, ldd, ws, wse, nullptr, 0, splits);
  cudaFreeAsync(ws, st);
  return rc;
}

ABFT_API int abft_dev_sgemm(void* stream, char transa, char transb, int64_t m, int64_t n, int64_t k,
                            float alpha, const float* A, int64_t lda, const float* B, int64_t ldb,
                            float beta, const float* C, int64_t ldc, float* D, int64_t ldd) {
  return abft_dev_sgemm_splitk(stream, transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                               D, ldd, 1);
}

// Diagonal-block factorization on device pointers (the PD kernel of
// linalg.py:219-238; mode 2 = the sign-shifted LU of the QR reconstruction).
// variant 0: one-CTA diag_factor + tri_inverse; 1: the cluster kernel.
// info_dev: device int, 1 + column of the first breakdown (0 if none).
ABFT_API int abft_dev_diag_factor(void* stream, int variant, int mode, int64_t w, double* D,
                                  int64_t ld, double* Linv, int64_t ldl, double* Uinv,
                                  int64_t ldu, int* info_dev, double* sgn) {
  if (w < 1 || w > 256 || mode < 0 || mode > 2 || variant < 0 || variant > 1) {
    set_last_error("abft_dev_diag_factor: bad arguments");
    return ABFT_E_INVALID;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return variant ? diag_factor_fast(st, D, ld, (int)w, mode, Linv, ldl, Uinv, ldu, info_dev, 0, sgn)
                 : diag_factor(st, D, ld, (int)w, mode, Linv, ldl, Uinv, ldu, info_dev, 0, sgn);
}

ABFT_API int abft_dev_sdiag_factor(void* stream, int variant, int mode, int64_t w, float* D,
                                   int64_t ld, float* Linv, int64_t ldl, float* Uinv, int64_t ldu,
                                   int* info_dev, float* sgn) {
  if (w < 1 || w > 256 || mode < 0 || mode > 2 || variant < 0 || variant > 1) {
    set_last_error("abft_dev_sdiag_factor: bad arguments");
    return ABFT_E_INVALID;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return variant ? diag_factor_fast(st, D, ld, (int)w, mode, Linv, ldl, Uinv, ldu, info_dev, 0, sgn)
                 : diag_factor(st, D, ld, (int)w, mode, Linv, ldl, Uinv, ldu, info_dev, 0, sgn);
}

}  // extern "C"
