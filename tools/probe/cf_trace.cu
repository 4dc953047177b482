// Phase timeline of the cluster diagonal-block factorization (globaltimer per
// CTA): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DCF_TRACE
//   -I paper_2301_03166_b200/csrc tools/probe/cf_trace.cu
//   paper_2301_03166_b200/csrc/{panel,gemm,abft_kernels}.cu -o tools/probe/cf_trace
#include "../../paper_2301_03166_b200/csrc/small_factor.cu"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int w = argc > 1 ? atoi(argv[1]) : 256, mode = argc > 2 ? atoi(argv[2]) : 0;
  std::vector<double> h(w * w);
  for (int i = 0; i < w; ++i)
    for (int j = 0; j < w; ++j) h[i + j * w] = (i == j ? w + 1.0 : 0.0) + 0.5 * ((i * 7 + j * 13) % 17) / 17.0;
  double *D, *L, *U, *S;
  int* info;
  cudaMalloc(&D, w * w * 8);
  cudaMalloc(&L, w * w * 8);
  cudaMalloc(&U, w * w * 8);
  cudaMalloc(&S, w * 8);
  cudaMalloc(&info, 4);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(D, h.data(), w * w * 8, cudaMemcpyHostToDevice);
    cudaMemset(info, 0, 4);
    abft::diag_factor_fast(0, D, w, w, mode, L, w, mode == 1 ? nullptr : U, w, info, 0, S);
    cudaDeviceSynchronize();
  }
  long long tr[8][64];
  cudaMemcpyFromSymbol(tr, abft::g_cf_trace, sizeof(tr));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  long long clk[4];
  cudaMemcpyFromSymbol(clk, abft::g_cf_clk, sizeof(clk));
  printf("diag block pivots 0-7/8-15/16-23/24-31 cycles: %lld %lld %lld %lld\n", clk[0], clk[1], clk[2], clk[3]);
  const int nb = (w + 31) / 32;
  long long t0 = tr[0][0];
  for (int r = 0; r < nb; ++r) {
    printf("CTA %d:", r);
    for (int s = 0; s < 64; ++s) {
      if ((s >= 4 * nb + 1 && s < 40) || tr[r][s] < t0 || tr[r][s] - t0 > 100000000) continue;
      printf(" %d:%.1f", s, (tr[r][s] - t0) * 1e-3);
    }
    printf("\n");
  }
  return 0;
}
