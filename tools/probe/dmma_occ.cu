// Can one warp per SMSP (4 warps/SM) saturate DMMA with a GEMM-like ILP pattern?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters) {
  double a[8], b[4], c[8][4][2];
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; i++) b[i] = 1.0 + i * 1e-3;
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) c[i][j][0] = c[i][j][1] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 4; j++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][j][0]), "+d"(c[i][j][1]) : "d"(a[i]), "d"(b[j]));
  }
  double s = 0; for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += c[i][j][0] + c[i][j][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 1; w <= 8; w *= 2) {
    for (int r = 0; r < 2; r++) {
      int it = 4000;
      cudaEventRecord(e0); k<<<148, 32 * w>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r) printf("warps/SM %d: %.2f TFLOP/s\n", w, 2.0 * 256 * 32 * it * 148.0 * w / ms / 1e9);
    }
  }
  return 0;
}
