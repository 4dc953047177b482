// Probe: cost of cooperative_groups grid.sync() vs a sense-reversal global barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void cg_sync(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) { x = x * 1.0000001 + 1.0; g.sync(); }
  if (x == 0.5) out[0] = x;
}
__device__ unsigned int g_count = 0;
__device__ volatile unsigned int g_gen = 0;
__global__ void my_sync(int iters, double* out) {
  double x = threadIdx.x;
  unsigned int gen = 0;
  for (int i = 0; i < iters; ++i) {
    x = x * 1.0000001 + 1.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      gen = g_gen;
      __threadfence();
      unsigned int arrived = atomicAdd(&g_count, 1) + 1;
      if (arrived == gridDim.x) { g_count = 0; __threadfence(); g_gen = gen + 1; }
      else { while (g_gen == gen) { } }
      __threadfence();
    }
    __syncthreads();
  }
  if (x == 0.5) out[0] = x;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  for (int G : {32, 74, 148}) {
    for (int rep = 0; rep < 2; ++rep) {
      void* args[] = {&iters, &o};
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)cg_sync, dim3(G), dim3(256), args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)my_sync, dim3(G), dim3(256), args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms2; cudaEventElapsedTime(&ms2, e0, e1);
      if (rep) printf("G=%3d: cg grid.sync %.2f us/sync, custom barrier %.2f us/sync\n", G, ms * 1e3 / iters, ms2 * 1e3 / iters);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
