// Shared device/host helpers for the B200 ABFT factorization library.
//
// Everything here is sm_100a-specific: TMA (cp.async.bulk.tensor) + mbarrier
// pipelines and FP64 DMMA (mma.sync ... f64, lowered to DMMA.8x8x4). tcgen05
// has no f64 kind on sm_100a (ptxas rejects .kind::f64), so DMMA is the only
// FP64 tensor path on this part; see DESIGN.md §3.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#define ABFT_DEVINL __device__ __forceinline__

namespace abft {

// ---------------------------------------------------------------------------
// error plumbing (host)
// ---------------------------------------------------------------------------
void set_last_error(const char* fmt, ...);
const char* last_error();
// number of kernels this library has launched (bench.py's gpu_launches)
void count_launch();
long long launch_count();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
int ensure_smem_attr(const void* fn, int bytes);

#define CUDA_TRY(expr)                                                          \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::abft::set_last_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr,        \
                             cudaGetErrorString(_e));                           \
      return -1000 - (int)_e;                                                   \
    }                                                                           \
  } while (0)

#define ABFT_TRY(expr)              \
  do {                              \
    int _rc = (expr);               \
    if (_rc != 0) return _rc;       \
  } while (0)

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier + TMA
// ---------------------------------------------------------------------------
ABFT_DEVINL uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

ABFT_DEVINL void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

ABFT_DEVINL void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

ABFT_DEVINL void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

ABFT_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Consumer-side stage release for TMA pipelines fed by ld.shared readers.
ABFT_DEVINL void consumer_release(uint64_t* bar, int lane) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __threadfence_block();
  __syncwarp();
  if (lane == 0) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
  }
}

ABFT_DEVINL bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

ABFT_DEVINL void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

ABFT_DEVINL void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Bulk prefetch of a 2-D tensor box into L2 (no shared-memory destination).
ABFT_DEVINL void tma_prefetch_l2_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

ABFT_DEVINL void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).
// Fragment ownership (lane = 4*g + j): a = A[g][j], b = B[j][g],
// c0/c1 = C[g][2j], C[g][2j+1].
ABFT_DEVINL void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

ABFT_DEVINL double2 lds_f64x2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// Deterministic warp sum.
ABFT_DEVINL double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
ABFT_DEVINL double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------
// Host: tensor-map creation for a column-major fp64 (sub-)matrix.
// ---------------------------------------------------------------------------
// A matrix view: element (i, j) at ptr[i + j * ld]; rows x cols.
struct MatView {
  const double* ptr;
  int64_t ld;
  int64_t rows;
  int64_t cols;
};

// Build a 2-D TMA map whose inner dimension is the contiguous one. `box_inner`
// x `box_outer` elements per load. The base pointer is aligned down to 16
// bytes (TMA requirement); the returned `shift` (0 or 1 elements) must be added
// to the inner coordinate of every load.
int make_tma_map(CUtensorMap* map, const double* ptr, int64_t ld, int64_t inner, int64_t outer,
                 int box_inner, int box_outer, bool swizzle128, int* shift);

}  // namespace abft
