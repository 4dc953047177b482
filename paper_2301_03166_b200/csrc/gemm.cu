// FP64 GEMM for the trailing-matrix updates: D = beta*C + alpha*op(A)*op(B).
//
// B200 design (kernel K3):
//  * FP64 tensor cores through DMMA (mma.sync m8n8k4 f64); tcgen05 has no f64
//    kind on sm_100a, so this is the fastest FP64 datapath on the part
//    (measured 37.1 TFLOP/s issue peak, profiles/fp64_peak_r01.txt).
//  * Warp-specialised: one producer warp issues TMA (cp.async.bulk.tensor)
//    loads into a 6-stage mbarrier ring; 8 consumer warps run DMMA out of
//    shared memory with 64x32 register-blocked warp tiles (CTA tile 128x128).
//  * Shared-memory layouts are chosen per operand orientation so every
//    fragment read is a conflict-free ld.shared.v2.f64: m/n-contiguous tiles are
//    dense, k-contiguous tiles use the TMA 128-byte swizzle.
//  * Split-K (deterministic, ordered partial reduction) for the long-K /
//    few-tile shapes of left-looking Cholesky and the QR V^T C product.
// The reference computes these products with numpy/OpenBLAS dgemm:
//   LU   m[pe:n,pe:n] -= l21 @ u12           (pkg/src/slackwise/simulator.py:148)
//   Chol m[p:n,p:pe]  -= m[p:n,0:p] @ m[p:pe,0:p].T   (simulator.py:141)
//   QR   mid = t.T @ (v.T @ c); c -= v @ mid  (simulator.py:154-157)
#include "gemm.cuh"

#include <cstdarg>
#include <cstring>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <tuple>
#include <vector>

#include <cudaTypedefs.h>

namespace abft {

// ---------------------------------------------------------------------------
// error string (thread-local so concurrent contexts do not clobber each other)
// ---------------------------------------------------------------------------
static thread_local char g_last_error[1024] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_last_error; }

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }

// Function attributes belong to a device context: the dynamic shared-memory
// opt-in is applied once per (kernel, device, size), thread-safely.
int ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::vector<std::tuple<const void*, int, int>> done;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& t : done)
    if (std::get<0>(t) == fn && std::get<1>(t) == dev && std::get<2>(t) >= bytes) return 0;
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.emplace_back(fn, dev, bytes);
  return 0;
}

// ---------------------------------------------------------------------------
// TMA descriptor creation through the driver entry point (no -lcuda needed)
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tma_map(CUtensorMap* map, const double* ptr, int64_t ld, int64_t inner, int64_t outer,
                 int box_inner, int box_outer, bool swizzle128, int* shift) {
  auto fn = get_encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return -20;
  }
  if (ld % 2 != 0) {
    set_last_error("leading dimension %lld must be even for TMA", (long long)ld);
    return -21;
  }
  uintptr_t addr = reinterpret_cast<uintptr_t>(ptr);
  int sh = static_cast<int>((addr & 15u) / 8u);
  const void* base = reinterpret_cast<const void*>(addr - sh * 8);
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner + sh),
                        static_cast<cuuint64_t>(outer < 1 ? 1 : outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 8)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld ld=%lld box=%dx%d",
                   (int)r, (long long)inner, (long long)outer, (long long)ld, box_inner, box_outer);
    return -22;
  }
  *shift = sh;
  return 0;
}

// ---------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------
namespace {

// Persistent multi-warpgroup DMMA GEMM.
//   * grid = #SMs CTAs; each CTA walks work units (tiles, or whole b x b
//     checksum blocks in fused mode) u = blockIdx.x + i*gridDim.x.
//   * NWG consumer warpgroups own units i = w (mod NWG), each with its own
//     TMA ring fed by its own producer warp (the last warpgroup). Groups start
//     one main loop apart and then run free: while one group runs its
//     epilogue (C load, D store, checksum partials) the others keep the DMMA
//     pipe busy. One warp per SM sub-partition reaches only ~83% of the DMMA
//     issue rate with this instruction stream, so the trailing-update shapes
//     (K = b) use three groups (32x32 warp tiles); long-K products use two
//     (64x32 warp tiles, fewer shared-memory reads per DMMA).
constexpr int BN = 64, BK = 16;
constexpr int WG_THREADS = 128;
constexpr int MAXFB = 256;
// per-WG fused-checksum accumulators: col plain/weighted [2 wm halves][fb][2],
// row plain [2 wn halves][fb], warp max [4]
constexpr int SUM_DOUBLES = 2 * MAXFB * 2 + 2 * MAXFB + 4;

template <int NWG>
struct Cfg;
template <>
struct Cfg<2> {
  static constexpr int WTM = 64, BM = 128, STAGES = 4;
};
template <>
struct Cfg<3> {
  static constexpr int WTM = 32, BM = 64, STAGES = 3;
};
template <int NWG>
struct Geo {
  static constexpr int BM = Cfg<NWG>::BM, STAGES = Cfg<NWG>::STAGES, WTM = Cfg<NWG>::WTM;
  static constexpr int RP = WTM / 16;  // 16-row fragment groups per warp
  static constexpr int THREADS = (NWG + 1) * WG_THREADS;
  static constexpr int A_BYTES = BM * BK * 8;
  static constexpr int B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr int NBARS = NWG * 2 * STAGES + NWG;
  static constexpr int SMEM_BYTES = NWG * RING_BYTES + 1024 + NBARS * 8 + NWG * SUM_DOUBLES * 8;
  // registers: producer warpgroup drops to REG_P, consumers rise to REG_C
  static constexpr int REG_P = NWG == 2 ? 40 : 32;
  static constexpr int REG_C = NWG == 2 ? 232 : 160;
};

struct KParams {
  int M, N, K;
  int a_shift, b_shift;
  int k_per_split;
  int tiles_m, tiles_n, splits;
  const double* C;
  int64_t ldc;
  double* D;
  int64_t ldd;
  double alpha, beta;
  int vec;               // 1 if C/D allow 16-byte row-pair accesses
  int prefetch_c;        // 1: TMA-prefetch each C tile into L2 when its main loop starts
  int c_shift;
  // fused checksums: each warpgroup owns whole fb x fb blocks (fb = 128/256)
  int fuse, fb, ntm_b, ntn_b, nbr_b, nbc_b;
  int unit_group;        // block rows per unit group (fused mode rasterization)
  FusedSums sums;
  int partial;           // 1: write raw acc to D (= split workspace slice z)
  int64_t split_stride;  // elements between split slices in partial mode
};

// Shared-memory layouts (all TMA SWIZZLE_128B, 1024-byte aligned):
//  * m/n-contiguous tiles (A-N, B-T): 16-row boxes [chunk][k][16] -- element
//    (k, r) at chunk*2048 + k*128 + (((r%16)/2) ^ (k&7))*16 + (r&1)*8;
//  * k-contiguous tiles (A-T, B-N): [r][16 k] -- (k, r) at
//    r*128 + ((k/2) ^ (r&7))*16 + (k&1)*8.
// A ld.shared.v2.f64 issued by a warp is served in four 8-lane phases; the
// fragment -> row/column maps below make every phase touch 8 distinct 16-byte
// chunks (conflict-free), which needs the permutation pm() on k-contiguous
// tiles.
ABFT_DEVINL int pm(int g) { return (g >> 1) + 4 * (g & 1); }

// Row of accumulator fragment (rp, e) for lane group g inside the warp tile.
template <bool AT>
ABFT_DEVINL int row_of(int rp, int e, int g) {
  if (AT) return 16 * rp + 8 * e + pm(g);
  return 16 * rp + 2 * g + e;
}
// Column of accumulator fragment (cf, c8) inside the warp tile.
// B-N: wn + 8cf + pm(c8);  B-T: cf=(cp,f): wn + 16cp + 2c8 + f.
template <bool BT>
ABFT_DEVINL int col_of(int cf, int c8) {
  if (BT) return 16 * (cf >> 1) + 2 * c8 + (cf & 1);
  return 8 * cf + pm(c8);
}

// Work unit of a warpgroup: plain mode = one tile; fused mode = one
// fb x BN strip of a checksum block (ntm_b tiles stacked vertically): its
// column sums are complete, its row sums / max are per-strip partials.
// Strips (not whole blocks) keep the tail of each trailing update balanced.
ABFT_DEVINL int unit_tiles(const KParams& p) { return p.fuse ? p.ntm_b : 1; }
ABFT_DEVINL int total_units(const KParams& p) {
  return p.fuse ? p.nbr_b * p.tiles_n : p.tiles_m * p.tiles_n * p.splits;
}
// Fused-mode unit -> (block row, 64-column strip), grouped so the units in
// flight at any moment cover a compact patch of GROUP block rows: their A
// panels (GROUP x fb rows) and B strips stay L2-resident and are reused
// instead of re-read from DRAM (plain column-major order re-read the whole
// L21 panel per strip column: 1.7x the algorithmic DRAM traffic).
ABFT_DEVINL void unit_coords(const KParams& p, int unit, int* bi, int* tcol) {
  const int G = p.unit_group;
  const int per_group = G * p.tiles_n;
  const int g = unit / per_group, r = unit - g * per_group;
  const int rows_g = min(G, p.nbr_b - g * G);
  *bi = g * G + r % rows_g;
  *tcol = r / rows_g;
}
template <int BM>
ABFT_DEVINL void fused_tile(const KParams& p, int unit, int u, int* m0, int* n0, int* bi, int* bj,
                            int* tm, int* tn) {
  int tcol;
  unit_coords(p, unit, bi, &tcol);
  *bj = tcol / p.ntn_b;
  *tn = tcol % p.ntn_b;
  *tm = u;
  *m0 = *bi * p.fb + u * BM;
  *n0 = tcol * BN;
}
template <int BM>
ABFT_DEVINL void tile_coords(const KParams& p, int t, int* m0, int* n0, int* z) {
  const int tm = t % p.tiles_m;
  const int r = t / p.tiles_m;
  *m0 = tm * BM;
  *n0 = (r % p.tiles_n) * BN;
  *z = r / p.tiles_n;
}

template <bool AT, bool BT, int NWG>
__global__ void __launch_bounds__(Geo<NWG>::THREADS, 1)
    dgemm_tma_dmma(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapC, KParams p) {
  using G = Geo<NWG>;
  constexpr int BM = G::BM, STAGES = G::STAGES, RP = G::RP, WTM = G::WTM;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NWG * G::RING_BYTES);
  // bars[w*2*STAGES + s] = full, bars[w*2*STAGES + STAGES + s] = empty,
  // bars[NWG*2*STAGES + w] = start token of warpgroup w
  double* sums_base = reinterpret_cast<double*>(bars + G::NBARS);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int units = total_units(p);
  const int upt = unit_tiles(p);

  if (threadIdx.x == 0) {
    for (int w = 0; w < NWG; ++w) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&bars[w * 2 * STAGES + s], 1);
        mbar_init(&bars[w * 2 * STAGES + STAGES + s], 4);
      }
      mbar_init(&bars[NWG * 2 * STAGES + w], 4);
    }
    mbar_fence_init();
  }
  for (int i = threadIdx.x; i < NWG * SUM_DOUBLES; i += G::THREADS) sums_base[i] = 0.0;
  __syncthreads();

  if (warp >= 4 * NWG) {
    // ===== producers: warp 4*NWG + w feeds ring w =====
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(G::REG_P));
    const int w = warp - 4 * NWG;
    if (w < NWG && lane == 0) {
      tma_prefetch_desc(&mapA);
      tma_prefetch_desc(&mapB);
      uint64_t* full = bars + w * 2 * STAGES;
      uint64_t* empty = full + STAGES;
      uint8_t* ring = smem + w * G::RING_BYTES;
      uint32_t q = 0;
      for (int i = w;; i += NWG) {
        const int unit = blockIdx.x + i * gridDim.x;
        if (unit >= units) break;
        for (int u = 0; u < upt; ++u) {
          int m0, n0, z = 0;
          if (p.fuse) {
            int bi, bj, tm, tn;
            fused_tile<BM>(p, unit, u, &m0, &n0, &bi, &bj, &tm, &tn);
          } else {
            tile_coords<BM>(p, unit, &m0, &n0, &z);
          }
          if (m0 >= p.M || n0 >= p.N) continue;
          const int kbeg = z * p.k_per_split;
          const int kend = min(p.K, kbeg + p.k_per_split);
          const int nkt = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
          if (p.prefetch_c) tma_prefetch_l2_2d(&mapC, m0 + p.c_shift, n0);
          for (int kt = 0; kt < nkt; ++kt, ++q) {
            const int s = q % STAGES;
            if (q >= STAGES) mbar_wait(&empty[s], ((q / STAGES) - 1) & 1);
            uint8_t* sa = ring + s * G::STAGE_BYTES;
            uint8_t* sb = sa + G::A_BYTES;
            const int k0 = kbeg + kt * BK;
            mbar_arrive_expect_tx(&full[s], G::STAGE_BYTES);
            if (AT) {
              tma_load_2d(sa, &mapA, &full[s], k0 + p.a_shift, m0);
            } else {
#pragma unroll
              for (int mc = 0; mc < BM / 16; ++mc)
                tma_load_2d(sa + mc * 2048, &mapA, &full[s], m0 + 16 * mc + p.a_shift, k0);
            }
            if (BT) {
#pragma unroll
              for (int nc = 0; nc < BN / 16; ++nc)
                tma_load_2d(sb + nc * 2048, &mapB, &full[s], n0 + 16 * nc + p.b_shift, k0);
            } else {
              tma_load_2d(sb, &mapB, &full[s], k0 + p.b_shift, n0);
            }
          }
        }
      }
    }
    return;
  }

  // ===== consumers =====
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(G::REG_C));
  const int wg = warp >> 2;
  const int wi = warp & 3;
  const int g = lane >> 2, j = lane & 3;
  const int wm = (wi & 1) * WTM;
  const int wn = (wi >> 1) * 32;
  uint64_t* full = bars + wg * 2 * STAGES;
  uint64_t* empty = full + STAGES;
  uint64_t* tok = bars + NWG * 2 * STAGES;
  const uint32_t ring = smem_u32(smem + wg * G::RING_BYTES);
  // fused-checksum accumulators of this warpgroup
  double* colacc = sums_base + wg * SUM_DOUBLES;   // [2][MAXFB][2]
  double* rowacc = colacc + 2 * MAXFB * 2;         // [2][MAXFB]
  double* wmax = rowacc + 2 * MAXFB;               // [4]
  uint32_t q = 0;
  int jt = 0;  // tiles processed by this WG

  for (int i = wg;; i += NWG) {
    const int unit = blockIdx.x + i * gridDim.x;
    if (unit >= units) break;
    double mx = 0.0;
    int bi = 0, bj = 0;
    for (int u = 0; u < upt; ++u) {
      int m0, n0, z = 0, tm = 0, tn = 0;
      if (p.fuse)
        fused_tile<BM>(p, unit, u, &m0, &n0, &bi, &bj, &tm, &tn);
      else
        tile_coords<BM>(p, unit, &m0, &n0, &z);
      if (m0 >= p.M || n0 >= p.N) continue;
      const int kbeg = z * p.k_per_split;
      const int kend = min(p.K, kbeg + p.k_per_split);
      const int nkt = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

      double acc[2 * RP][4][2];
#pragma unroll
      for (int a = 0; a < 2 * RP; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

      // start offset: group w begins its first main loop when group w-1 has
      // finished its first one
      if (wg > 0 && jt == 0) mbar_wait(&tok[wg], 0);
      __syncwarp();

      int prev_s = -1;
      for (int kt = 0; kt < nkt; ++kt, ++q) {
        const int s = q % STAGES;
        mbar_wait(&full[s], (q / STAGES) & 1);
        __syncwarp();  // mma.sync.aligned needs the whole warp converged
        // Release the previous stage one step late: its shared-memory reads
        // fed DMMAs issued before this wait loop (a hard scheduling boundary),
        // so they have completed -- no fence needed on the steady path.
        if (prev_s >= 0 && lane == 0) mbar_arrive(&empty[prev_s]);
        const uint32_t sa = ring + s * G::STAGE_BYTES;
        const uint32_t sb = sa + G::A_BYTES;
#pragma unroll
        for (int ks = 0; ks < BK; ks += 8) {
          double b[4][2];
          if (!BT) {
            // [n][16 k]: n = wn + 8cf + pm(g), k = ks+2j (+ss in the pair)
#pragma unroll
            for (int cf = 0; cf < 4; ++cf) {
              const int n = wn + 8 * cf + pm(g);
              double2 v = lds_f64x2(sb + n * 128 + ((((ks >> 1) + j) ^ (n & 7)) << 4));
              b[cf][0] = v.x;
              b[cf][1] = v.y;
            }
          } else {
            // [n/16][k][16 n]: n = wn + 16cp + 2g (+f in the pair), k = ks+2j+ss
#pragma unroll
            for (int cp = 0; cp < 2; ++cp)
#pragma unroll
              for (int ss = 0; ss < 2; ++ss) {
                const int k = ks + 2 * j + ss;
                double2 v = lds_f64x2(sb + ((wn >> 4) + cp) * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
                b[2 * cp][ss] = v.x;
                b[2 * cp + 1][ss] = v.y;
              }
          }
          double a[RP][2][2];
#pragma unroll
          for (int rp = 0; rp < RP; ++rp) {
            if (!AT) {
              // [m/16][k][16 m]: m = wm + 16rp + 2g (+e in the pair), k = ks+2j+ss
#pragma unroll
              for (int ss = 0; ss < 2; ++ss) {
                const int k = ks + 2 * j + ss;
                double2 v = lds_f64x2(sa + ((wm >> 4) + rp) * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
                a[rp][ss][0] = v.x;
                a[rp][ss][1] = v.y;
              }
            } else {
              // [m][16 k]: m = wm + 16rp + 8e + pm(g)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int m = wm + 16 * rp + 8 * e + pm(g);
                double2 v = lds_f64x2(sa + m * 128 + ((((ks >> 1) + j) ^ (m & 7)) << 4));
                a[rp][0][e] = v.x;
                a[rp][1][e] = v.y;
              }
            }
          }
#pragma unroll
          for (int ss = 0; ss < 2; ++ss)
#pragma unroll
            for (int rp = 0; rp < RP; ++rp)
#pragma unroll
              for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int cf = 0; cf < 4; ++cf)
                  dmma_8x8x4(acc[2 * rp + e][cf][0], acc[2 * rp + e][cf][1], a[rp][ss][e], b[cf][ss]);
        }
        prev_s = s;
      }
      // last stage of the tile: fenced release (no later wait orders its reads)
      if (prev_s >= 0) consumer_release(&empty[prev_s], lane);
      if (wg + 1 < NWG && jt == 0 && lane == 0) mbar_arrive(&tok[wg + 1]);
      ++jt;

      // ===== epilogue =====
      // Pass 1 (per row-pair group, C loads batched): out = alpha*acc + beta*C,
      // computed in place in the accumulator registers and stored.
      double* D = p.partial ? p.D + (int64_t)z * p.split_stride : p.D;
      const bool use_c = !p.partial && p.beta != 0.0;
#pragma unroll
      for (int rp = 0; rp < RP; ++rp) {
        // rows of fragments (rp, 0) / (rp, 1): adjacent for A-N, 8 apart for A-T
        const int row0 = m0 + wm + row_of<AT>(rp, 0, g);
        const int row1 = m0 + wm + row_of<AT>(rp, 1, g);
        const bool rv0 = row0 < p.M, rv1 = row1 < p.M;
        const bool pairv = !AT && p.vec && rv1;  // 16-byte row-pair access
        double cv[4][2][2];
#pragma unroll
        for (int cf = 0; cf < 4; ++cf)
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) {
            cv[cf][tt][0] = cv[cf][tt][1] = 0.0;
            const int col = n0 + wn + col_of<BT>(cf, 2 * j + tt);
            if (!use_c || col >= p.N) continue;
            const double* c = p.C + (int64_t)col * p.ldc;
            if (pairv) {
              const double2 v = *reinterpret_cast<const double2*>(c + row0);
              cv[cf][tt][0] = v.x;
              cv[cf][tt][1] = v.y;
            } else {
              if (rv0) cv[cf][tt][0] = c[row0];
              if (rv1) cv[cf][tt][1] = c[row1];
            }
          }
#pragma unroll
        for (int cf = 0; cf < 4; ++cf)
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) {
            const int col = n0 + wn + col_of<BT>(cf, 2 * j + tt);
            const bool cvld = col < p.N;
            double o0 = acc[2 * rp][cf][tt], o1 = acc[2 * rp + 1][cf][tt];
            if (!p.partial) {
              o0 = fma(p.alpha, o0, p.beta * cv[cf][tt][0]);
              o1 = fma(p.alpha, o1, p.beta * cv[cf][tt][1]);
            }
            // rows/cols outside D contribute nothing to the checksums
            o0 = (rv0 && cvld) ? o0 : 0.0;
            o1 = (rv1 && cvld) ? o1 : 0.0;
            acc[2 * rp][cf][tt] = o0;
            acc[2 * rp + 1][cf][tt] = o1;
            if (!cvld) continue;
            double* d = D + (int64_t)col * p.ldd;
            if (pairv && !p.partial) {
              *reinterpret_cast<double2*>(d + row0) = make_double2(o0, o1);
            } else {
              if (rv0) d[row0] = o0;
              if (rv1) d[row1] = o1;
            }
          }
      }
      // Pass 2 (fused checksums) from the output registers. Lane sums are
      // combined with reduce-scatter butterflies (each exchange halves the
      // values still carried), so every lane ends up owning complete sums.
      if (p.fuse) {
        // row sums over this warp's 32 columns: 2*RP rows per lane group,
        // reduced over the 4 j-lanes
        double rv[2 * RP];
#pragma unroll
        for (int rp = 0; rp < RP; ++rp) {
          double rs0 = 0.0, rs1 = 0.0;
#pragma unroll
          for (int cf = 0; cf < 4; ++cf)
#pragma unroll
            for (int tt = 0; tt < 2; ++tt) {
              rs0 += acc[2 * rp][cf][tt];
              rs1 += acc[2 * rp + 1][cf][tt];
              mx = fmax(mx, fmax(fabs(acc[2 * rp][cf][tt]), fabs(acc[2 * rp + 1][cf][tt])));
            }
          rv[2 * rp] = rs0;
          rv[2 * rp + 1] = rs1;
        }
        {
          constexpr int NR = 2 * RP;  // 4 (three warpgroups) or 8 (two)
          const bool h1 = (j & 2) != 0, h0 = (j & 1) != 0;
#pragma unroll
          for (int i = 0; i < NR / 2; ++i) {
            const double snd = h1 ? rv[i] : rv[i + NR / 2];
            rv[i] = (h1 ? rv[i + NR / 2] : rv[i]) + __shfl_xor_sync(0xffffffffu, snd, 2);
          }
#pragma unroll
          for (int i = 0; i < NR / 4; ++i) {
            const double snd = h0 ? rv[i] : rv[i + NR / 4];
            rv[i] = (h0 ? rv[i + NR / 4] : rv[i]) + __shfl_xor_sync(0xffffffffu, snd, 1);
          }
#pragma unroll
          for (int i = 0; i < NR / 4; ++i) {
            const int q = (h1 ? NR / 2 : 0) + (h0 ? NR / 4 : 0) + i;  // rv index = 2*rp + e
            const int r = tm * BM + wm + row_of<AT>(q >> 1, q & 1, g);
            rowacc[(wn >> 5) * MAXFB + r] += rv[i];
          }
        }
        // column plain / index-weighted sums over this warp's WTM rows:
        // 16 values (cf, tt, plain|weighted) reduced over the 8 g-lanes
        const int wbase = tm * BM + wm;
        double v[16];
#pragma unroll
        for (int cf = 0; cf < 4; ++cf)
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) {
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int rp = 0; rp < RP; ++rp) {
              const double x0 = acc[2 * rp][cf][tt], x1 = acc[2 * rp + 1][cf][tt];
              const double w0 = (double)(wbase + row_of<AT>(rp, 0, g));
              const double w1 = (double)(wbase + row_of<AT>(rp, 1, g));
              a0 += x0 + x1;
              a1 += w0 * x0 + w1 * x1;
            }
            v[(cf * 2 + tt) * 2 + 0] = a0;
            v[(cf * 2 + tt) * 2 + 1] = a1;
          }
        const bool g2 = (g & 4) != 0, g1 = (g & 2) != 0, g0 = (g & 1) != 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double snd = g2 ? v[i] : v[i + 8];
          v[i] = (g2 ? v[i + 8] : v[i]) + __shfl_xor_sync(0xffffffffu, snd, 16);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double snd = g1 ? v[i] : v[i + 4];
          v[i] = (g1 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, snd, 8);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double snd = g0 ? v[i] : v[i + 2];
          v[i] = (g0 ? v[i + 2] : v[i]) + __shfl_xor_sync(0xffffffffu, snd, 4);
        }
        // this lane now owns (cf, tt) = (g >> 1, g & 1): plain v[0], weighted v[1]
        const int c = tn * BN + wn + col_of<BT>(g >> 1, 2 * j + (g & 1));
        colacc[((wi & 1) * MAXFB + c) * 2 + 0] += v[0];
        colacc[((wi & 1) * MAXFB + c) * 2 + 1] += v[1];
      }
    }
    if (p.fuse) {
      // strip finished: combine the halves in a fixed order and publish the
      // complete column sums and the strip's partial row sums / max
      int bi_u, tcol_u;
      unit_coords(p, unit, &bi_u, &tcol_u);
      const int tn = tcol_u % p.ntn_b;
      mx = warp_max(mx);
      if (lane == 0) wmax[wi] = mx;
      asm volatile("bar.sync %0, 128;\n" ::"r"(1 + wg) : "memory");
      const int tid = threadIdx.x & 127;
      const int rows_b = min(p.fb, p.M - bi * p.fb);
      const int c0s = tn * BN;
      const int cols_s = min(BN, p.N - (bj * p.fb + c0s));
      const FusedSums& fs = p.sums;
      for (int c = tid; c < cols_s; c += 128) {
        const int cc = c0s + c;
        const int64_t gc = (int64_t)bj * p.fb + cc;
        fs.cp[fs.cp_step * bi + gc * fs.cp_ld] = colacc[cc * 2 + 0] + colacc[(MAXFB + cc) * 2 + 0];
        fs.cw[fs.cw_step * bi + gc * fs.cw_ld] = colacc[cc * 2 + 1] + colacc[(MAXFB + cc) * 2 + 1];
      }
      const int64_t scol = (int64_t)bj * p.ntn_b + tn;
      for (int r = tid; r < rows_b; r += 128)
        fs.rpp[(int64_t)bi * p.fb + r + scol * fs.rpp_ld] = rowacc[r] + rowacc[MAXFB + r];
      if (tid == 0)
        fs.bmp[bi + scol * fs.bmp_ld] = fmax(fmax(wmax[0], wmax[1]), fmax(wmax[2], wmax[3]));
      asm volatile("bar.sync %0, 128;\n" ::"r"(1 + wg) : "memory");
      for (int t = tid; t < 4 * BN; t += 128) {
        const int half = t / (2 * BN), rem = t % (2 * BN);
        colacc[(half * MAXFB + c0s + (rem >> 1)) * 2 + (rem & 1)] = 0.0;
      }
      for (int t = tid; t < 2 * MAXFB; t += 128) rowacc[t] = 0.0;
      asm volatile("bar.sync %0, 128;\n" ::"r"(1 + wg) : "memory");
    }
  }
}

// Row sums and block max of the fused epilogue: fixed-order combination of
// the per-strip partials (rows x nbc and nbr x nbc outputs).
__global__ void fused_combine(int M, int N, int fb, int ntn, FusedSums s) {
  const int nbr = (M + fb - 1) / fb, nbc = (N + fb - 1) / fb;
  const int64_t nrow = (int64_t)M * nbc;
  const int64_t total = nrow + (int64_t)nbr * nbc;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < nrow) {
      const int r = static_cast<int>(idx % M);
      const int bj = static_cast<int>(idx / M);
      const int ns = (min(fb, N - bj * fb) + BN - 1) / BN;
      const double* src = s.rpp + r + (int64_t)bj * ntn * s.rpp_ld;
      double v = 0.0;
      for (int t = 0; t < ns; ++t) v += src[(int64_t)t * s.rpp_ld];
      s.rp[r + (int64_t)bj * s.rp_ld] = v;
    } else {
      const int64_t t2 = idx - nrow;
      const int bi = static_cast<int>(t2 % nbr);
      const int bj = static_cast<int>(t2 / nbr);
      const int ns = (min(fb, N - bj * fb) + BN - 1) / BN;
      double m = 0.0;
      for (int t = 0; t < ns; ++t) m = fmax(m, s.bmp[bi + ((int64_t)bj * ntn + t) * s.bmp_ld]);
      s.bm[bi + (int64_t)bj * s.bm_ld] = m;
    }
  }
}

// D = beta*C + alpha * sum_z W[z]   (ordered, deterministic)
__global__ void splitk_reduce(int M, int N, int splits, const double* __restrict__ W,
                              int64_t ldw, int64_t stride, const double* C, int64_t ldc, double* D,
                              int64_t ldd, double alpha, double beta) {
  const int64_t total = (int64_t)M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(idx % M);
    const int jcol = static_cast<int>(idx / M);
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += W[z * stride + i + jcol * ldw];
    const double c = beta != 0.0 ? C[i + (int64_t)jcol * ldc] : 0.0;
    D[i + (int64_t)jcol * ldd] = fma(alpha, s, beta * c);
  }
}

template <bool AT, bool BT, int NWG>
int launch_kernel(cudaStream_t st, const CUtensorMap& ma, const CUtensorMap& mb,
                  const CUtensorMap& mc, const KParams& kp, int max_ctas) {
  using G = Geo<NWG>;
  ABFT_TRY(ensure_smem_attr((const void*)dgemm_tma_dmma<AT, BT, NWG>, G::SMEM_BYTES));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = kp.fuse ? kp.nbr_b * kp.nbc_b : kp.tiles_m * kp.tiles_n * kp.splits;
  const int cap = (max_ctas > 0 && max_ctas < sms) ? max_ctas : sms;
  const int grid = total < cap ? total : cap;
  count_launch();
  dgemm_tma_dmma<AT, BT, NWG><<<grid, G::THREADS, G::SMEM_BYTES, st>>>(ma, mb, mc, kp);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int NWG>
int launch_any(cudaStream_t st, bool AT, bool BT, const CUtensorMap& ma, const CUtensorMap& mb,
               const CUtensorMap& mc, const KParams& kp, int max_ctas) {
  if (AT && BT) return launch_kernel<true, true, NWG>(st, ma, mb, mc, kp, max_ctas);
  if (AT) return launch_kernel<true, false, NWG>(st, ma, mb, mc, kp, max_ctas);
  if (BT) return launch_kernel<false, true, NWG>(st, ma, mb, mc, kp, max_ctas);
  return launch_kernel<false, false, NWG>(st, ma, mb, mc, kp, max_ctas);
}

}  // namespace

// Split-K factor from a wave model of the persistent kernel: units are
// handed out round-robin, so a launch takes ceil(units / SMs) unit-times;
// a unit costs (K-slice + fixed prologue/epilogue) DMMA steps on a
// BM x 64 tile, and every extra slice adds a partial write + read-back.
// Short-K products (the rank-b trailing updates) never split.
int gemm_splits_for(int M, int N, int K, int num_sms) {
  if (K <= 4 * BK * 8) return 1;
  const int maxs = std::min(32, K / (8 * BK));  // keep >= 128 of K per split
  const double step_s = 2.0 * 64 / 0.25e12;  // seconds per k per tile row (64-wide tile, one SM)
  int best = 1;
  double best_t = 0.0;
  for (int s = 1; s <= std::max(1, maxs); ++s) {
    const int kps = ((K + s - 1) / s + BK - 1) / BK * BK;
    const int se = (K + kps - 1) / kps;
    if (se != s) continue;
    const int bm = kps <= 1024 ? 64 : 128;
    const int64_t units = (int64_t)((M + bm - 1) / bm) * ((N + BN - 1) / BN) * se;
    const int64_t waves = (units + num_sms - 1) / num_sms;
    double t = (double)waves * (kps + 256) * bm * step_s;
    if (se > 1) t += (double)se * M * N * 16.0 / 6.0e12 + 5e-6;
    if (s == 1 || t < 0.98 * best_t) {
      best = s;
      best_t = t;
    }
  }
  return best;
}

// The split-K factor gemm() uses for this shape (requested `splits` <= 0:
// the wave model; then capped by the workspace), so a product computed in
// column windows can reproduce the full product's K partition bit for bit.
int gemm_effective_splits(int M, int N, int K, const GemmWorkspace* ws, int splits, int max_ctas) {
  if (splits <= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // a capped launch (look-ahead side streams) deals its units over fewer CTAs
    if (max_ctas > 0 && max_ctas < sms) sms = max_ctas;
    splits = gemm_splits_for(M, N, K, sms);
  }
  int kps = ((K + splits - 1) / splits + BK - 1) / BK * BK;
  splits = (K + kps - 1) / kps;
  const int64_t slice = (int64_t)M * N;
  if (splits > 1 && (!ws || ws->ptr == nullptr || ws->elems < slice * splits)) {
    const int64_t cap = (ws && ws->ptr) ? ws->elems / slice : 0;
    if (cap >= 2) {
      splits = static_cast<int>(cap < splits ? cap : splits);
      kps = ((K + splits - 1) / splits + BK - 1) / BK * BK;
      splits = (K + kps - 1) / kps;
    } else {
      splits = 1;
    }
  }
  return splits;
}

static int gemm_impl(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha,
                     const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                     const double* C, int64_t ldc, double* D, int64_t ldd, GemmWorkspace* ws,
                     int splits, const FusedSums* fs, int fb, int max_ctas) {
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0) {
    // D = beta*C (alpha*0)
    if (beta == 0.0 && C == D) return 0;
    count_launch();
    splitk_reduce<<<256, 256, 0, st>>>(M, N, 0, nullptr, 1, 0, C, ldc, D, ldd, alpha, beta);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  const bool AT = (ta == 'T' || ta == 't');
  const bool BT = (tb == 'T' || tb == 't');
  if (fs) splits = 1;
  splits = gemm_effective_splits(M, N, K, ws, splits, max_ctas);
  const int kps = splits > 1 ? ((K + splits - 1) / splits + BK - 1) / BK * BK : K;
  const int64_t ldw = M;
  const int64_t slice = ldw * N;

  // three warpgroups (64x64 tiles) for short-K products such as the rank-b
  // trailing updates, two (128x64 tiles) for long K
  static const int nwg_env = [] {
    const char* e = getenv("ABFT_GEMM_NWG");  // A/B knob: force 2 or 3 consumer warpgroups
    const int v = e ? atoi(e) : 0;
    return (v == 2 || v == 3) ? v : 0;
  }();
  const int nwg = nwg_env ? nwg_env : ((kps <= 1024) ? 3 : 2);
  const int BM = nwg == 3 ? Cfg<3>::BM : Cfg<2>::BM;
  CUtensorMap ma, mb;
  int sha = 0, shb = 0;
  if (AT)
    ABFT_TRY(make_tma_map(&ma, A, lda, K, M, BK, BM, true, &sha));
  else
    ABFT_TRY(make_tma_map(&ma, A, lda, M, K, 16, BK, true, &sha));
  if (BT)
    ABFT_TRY(make_tma_map(&mb, B, ldb, N, K, 16, BK, true, &shb));
  else
    ABFT_TRY(make_tma_map(&mb, B, ldb, K, N, BK, BN, true, &shb));

  KParams kp;
  kp.M = M;
  kp.N = N;
  kp.K = K;
  kp.a_shift = sha;
  kp.b_shift = shb;
  kp.k_per_split = kps;
  kp.alpha = alpha;
  kp.beta = beta;
  kp.tiles_m = (M + BM - 1) / BM;
  kp.tiles_n = (N + BN - 1) / BN;
  kp.splits = splits;
  kp.fuse = 0;
  kp.fb = 0;
  kp.ntm_b = kp.ntn_b = kp.nbr_b = kp.nbc_b = 0;
  if (fs) {
    kp.fuse = 1;
    kp.fb = fb;
    kp.ntm_b = fb / BM;
    kp.ntn_b = fb / BN;
    kp.nbr_b = (M + fb - 1) / fb;
    kp.nbc_b = (N + fb - 1) / fb;
    kp.sums = *fs;
    static int ug = [] {
      const char* e = getenv("ABFT_UNIT_GROUP");
      const int v = e ? atoi(e) : 0;
      return v > 0 ? v : 16;  // ABFT_UNIT_GROUP=100000 restores plain column-major strips
    }();
    kp.unit_group = ug;
  }
  if (splits > 1) {
    kp.C = nullptr;
    kp.ldc = 0;
    kp.D = ws->ptr;
    kp.ldd = ldw;
    kp.partial = 1;
    kp.split_stride = slice;
    kp.vec = 0;
  } else {
    kp.C = C;
    kp.ldc = ldc;
    kp.D = D;
    kp.ldd = ldd;
    kp.partial = 0;
    kp.split_stride = 0;
    const bool cv = (beta == 0.0) || ((reinterpret_cast<uintptr_t>(C) & 15) == 0 && ldc % 2 == 0);
    const bool dv = (reinterpret_cast<uintptr_t>(D) & 15) == 0 && ldd % 2 == 0;
    kp.vec = (cv && dv) ? 1 : 0;
  }
  CUtensorMap mc;
  memset(&mc, 0, sizeof(mc));
  kp.prefetch_c = 0;
  kp.c_shift = 0;
  if (!kp.partial && beta != 0.0 && (ldc % 2) == 0) {
    int shc = 0;
    if (make_tma_map(&mc, C, ldc, M, N, BM, BN, false, &shc) == 0) {
      kp.prefetch_c = 1;
      kp.c_shift = shc;
    }
  }
  int rc = nwg == 3 ? launch_any<3>(st, AT, BT, ma, mb, mc, kp, max_ctas)
                    : launch_any<2>(st, AT, BT, ma, mb, mc, kp, max_ctas);
  if (rc) return rc;
  if (fs) {
    const int64_t work = (int64_t)M * kp.nbc_b + (int64_t)kp.nbr_b * kp.nbc_b;
    int blocks = static_cast<int>((work + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    count_launch();
    fused_combine<<<blocks, 256, 0, st>>>(M, N, fb, kp.ntn_b, *fs);
    CUDA_TRY(cudaGetLastError());
  }
  if (splits > 1) {
    int blocks = static_cast<int>(((int64_t)M * N + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    count_launch();
    splitk_reduce<<<blocks, 256, 0, st>>>(M, N, splits, ws->ptr, ldw, slice, C, ldc, D, ldd, alpha,
                                          beta);
    CUDA_TRY(cudaGetLastError());
  }
  return 0;
}

int gemm(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, const double* C, int64_t ldc,
         double* D, int64_t ldd, GemmWorkspace* ws, int splits) {
  return gemm_impl(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, D, ldd, ws, splits,
                   nullptr, 0, 0);
}

bool gemm_can_fuse(int fb) { return fb == 128 || fb == 256; }

int gemm_capped(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha,
                const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                const double* C, int64_t ldc, double* D, int64_t ldd, GemmWorkspace* ws,
                int max_ctas) {
  return gemm_impl(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, D, ldd, ws, 0,
                   nullptr, 0, max_ctas);
}

int gemm_reserved(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha,
                  const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                  const double* C, int64_t ldc, double* D, int64_t ldd, int max_ctas) {
  return gemm_impl(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, D, ldd, nullptr, 1,
                   nullptr, 0, max_ctas);
}

int gemm_fused_sums(cudaStream_t st, char ta, char tb, int M, int N, int K, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                    const double* C, int64_t ldc, double* D, int64_t ldd, int fb,
                    const FusedSums& sums, int max_ctas) {
  if (!gemm_can_fuse(fb)) {
    set_last_error("fused checksums need b = 128 or 256 (got %d)", fb);
    return -1;
  }
  if (K <= 0) {
    set_last_error("fused checksums need K > 0");
    return -1;
  }
  if (!sums.rpp || !sums.bmp) {
    set_last_error("fused checksums need the per-strip scratch arrays");
    return -1;
  }
  return gemm_impl(st, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, D, ldd, nullptr, 1,
                   &sums, fb, max_ctas);
}

}  // namespace abft
