// FP32 GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32) for the
// s* factorizations: D = beta*C + alpha*op(A)*op(B), column-major fp32.
//
// FP32 accuracy from TF32 tensor cores (3xTF32): each operand is split once
// into hi = rna_tf32(x) and lo = x - hi, and every k-step issues
//   acc += A_lo B_hi + A_hi B_lo + A_hi B_hi
// (the lo*lo term is below fp32 resolution). The split kernel also writes
// both operands K-major, so the MMA always reads the canonical K-major
// 128-byte-swizzled shared-memory layout TMA produces.
//
// Kernel structure (persistent, one CTA per SM, 320 threads):
//   warp 0      TMA producer: 4 boxes (A_hi, A_lo, B_hi, B_lo) per 32-wide
//               k-block into a 3-stage mbarrier ring (64 KB per stage)
//   warp 1      allocates 256 TMEM columns; one lane issues tcgen05.mma
//               (M=128, N=128, K=8) into a double-buffered TMEM accumulator
//               and commits stages / finished tiles to mbarriers
//   warps 2..9  epilogue, two warps per TMEM lane quarter (each owns half
//               the tile's columns): tcgen05.ld 32x32b.x32 (one row per thread),
//               D = beta*C + alpha*acc with warp-coalesced column accesses,
//               and (fused mode, checksum block = tile = 128 x 128) the
//               block's column plain / index-weighted sums, row sums and
//               max|x| accumulated in fp64 -- the verify-side checksums of
//               abft.py:118-135 without another pass over D.
// The TMEM double buffer lets the epilogue of tile i overlap the MMAs of
// tile i+1.
#include "sgemm.cuh"

#include <cstdlib>
#include <cstring>
#include <mutex>

#include <cudaTypedefs.h>

namespace abft {

namespace {

constexpr int TBM = 128, TBN = 128, TBK = 32;  // TBK fp32 = one 128-byte swizzle row
constexpr int TSTAGES = 3;
constexpr int T_A_BYTES = TBM * TBK * 4;
constexpr int T_B_BYTES = TBN * TBK * 4;
constexpr int T_STAGE_BYTES = 2 * T_A_BYTES + 2 * T_B_BYTES;  // 64 KB
constexpr int T_THREADS = 384;  // producer, MMA issuer, 8 epilogue warps, 2 converter warps
constexpr int T_TMEM_COLS = 256;  // two 128-column fp32 accumulators
constexpr int T_TP = 17;          // padded 32 x 16 transpose tile
// smem: ring | barriers (2*ST + 4) | tmem slot | per-warp transpose tiles |
//        per-warp column partials (double) | warp max
constexpr int T_BAR_OFF = TSTAGES * T_STAGE_BYTES;
constexpr int T_TR_OFF = T_BAR_OFF + 256;
constexpr int T_TR_BYTES = 8 * 32 * T_TP * 4;
constexpr int T_COL_OFF = T_TR_OFF + T_TR_BYTES;
// per-tile cross-warp partials, double-buffered by tile parity so one
// named barrier per tile suffices: column sums [4 quarters][TBN][2] fp32,
// row sums [2 halves][TBM] fp32, warp maxima [8] fp32
constexpr int T_PART_FLOATS = 4 * TBN * 2 + 2 * TBM + 8;
constexpr int T_COL_BYTES = 2 * T_PART_FLOATS * 4;
constexpr int T_SMEM = T_COL_OFF + T_COL_BYTES + 1024;

struct SParams {
  int M, N, K;
  int tiles_m, tiles_n, nkb;
  const float* C;
  int64_t ldc;
  float* D;
  int64_t ldd;
  float alpha, beta;
  int fuse;
  int prefetch_c;  // 1: TMA-prefetch each tile's C box into L2 ahead of its epilogue
  // split-K: unit u = (tile u % tiles, split u / tiles) runs k-blocks
  // [split * kbs, min(nkb, (split + 1) * kbs)) and writes alpha * acc to
  // D + split * dstride (a partial; beta = 0, no fused sums)
  int splits, kbs;
  int64_t dstride;
  // raw operands: TMA brings the unsplit fp32 box into the hi slot and the
  // converter warps form hi = rna_tf32(x) / lo = x - hi in shared memory
  // (elementwise, so the 128-byte swizzle is preserved) -- no split pass
  int raw_a, raw_b;
  FusedSums sums;
};

// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05 / UMMA):
// start address >> 4, LBO 16 B (unused for swizzled K-major), SBO 1024 B
// (8 rows x 128 B), descriptor version 1, layout type 2 = SWIZZLE_128B.
ABFT_DEVINL uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(16u >> 4) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor: kind::tf32, fp32 accumulate, both K-major,
// M = 128, N = 128.
constexpr uint32_t IDESC = (1u << 4)            // c_format F32
                           | (2u << 7)          // a_format TF32
                           | (2u << 10)         // b_format TF32
                           | ((uint32_t)(TBN >> 3) << 17)
                           | ((uint32_t)(TBM >> 4) << 24);

ABFT_DEVINL void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(IDESC), "r"(accum));
}

ABFT_DEVINL void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

ABFT_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
ABFT_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

ABFT_DEVINL void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(T_THREADS, 1)
    sgemm_tc05_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                      const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl,
                      const __grid_constant__ CUtensorMap mC, SParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + T_BAR_OFF);
  uint64_t* empty = full + TSTAGES;
  uint64_t* tfull = empty + TSTAGES;   // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint64_t* conv = tempty + 2;         // [TSTAGES] raw operands converted
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv + TSTAGES);
  float* trs = reinterpret_cast<float*>(smem + T_TR_OFF);
  float* parts = reinterpret_cast<float*>(smem + T_COL_OFF);   // [2 parities][T_PART_FLOATS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = p.tiles_m * p.tiles_n;
  const int units = tiles * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 2);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(T_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      tma_prefetch_desc(&mAh);
      tma_prefetch_desc(&mAl);
      tma_prefetch_desc(&mBh);
      tma_prefetch_desc(&mBl);
      uint32_t q = 0;
      for (int t = blockIdx.x; t < units; t += gridDim.x) {
        const int tt = t % tiles, sp = t / tiles;
        const int tm = tt % p.tiles_m, tn = tt / p.tiles_m;
        const int kb0 = sp * p.kbs, kb1 = min(p.nkb, kb0 + p.kbs);
        // the epilogue of this tile reads C long after its operands stream in:
        // pull the C box into L2 now so those loads do not pay DRAM latency
        if (p.prefetch_c) tma_prefetch_l2_2d(&mC, tm * TBM, tn * TBN);
        for (int kb = kb0; kb < kb1; ++kb, ++q) {
          const int s = q % TSTAGES;
          if (q >= TSTAGES) mbar_wait(&empty[s], ((q / TSTAGES) - 1) & 1);
          uint8_t* st = smem + s * T_STAGE_BYTES;
          mbar_arrive_expect_tx(&full[s], T_STAGE_BYTES - (p.raw_a ? T_A_BYTES : 0) -
                                              (p.raw_b ? T_B_BYTES : 0));
          tma_load_2d(st, &mAh, &full[s], kb * TBK, tm * TBM);
          if (!p.raw_a) tma_load_2d(st + T_A_BYTES, &mAl, &full[s], kb * TBK, tm * TBM);
          tma_load_2d(st + 2 * T_A_BYTES, &mBh, &full[s], kb * TBK, tn * TBN);
          if (!p.raw_b) tma_load_2d(st + 2 * T_A_BYTES + T_B_BYTES, &mBl, &full[s], kb * TBK, tn * TBN);
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    uint32_t q = 0;
    int it = 0;
    for (int t = blockIdx.x; t < units; t += gridDim.x, ++it) {
      const int acc = it & 1, use = it >> 1;
      const int kb0 = (t / tiles) * p.kbs, kb1 = min(p.nkb, kb0 + p.kbs);
      if (use >= 1) mbar_wait(&tempty[acc], (use - 1) & 1);
      tc_fence_after();
      const uint32_t dt = tmem_base + (uint32_t)(acc * TBN);
      for (int kb = kb0; kb < kb1; ++kb, ++q) {
        const int s = q % TSTAGES;
        mbar_wait((p.raw_a | p.raw_b) ? &conv[s] : &full[s], (q / TSTAGES) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t st = smem_u32(smem + s * T_STAGE_BYTES);
#pragma unroll
          for (int ks = 0; ks < TBK / 8; ++ks) {
            const uint32_t off = ks * 32;  // 8 tf32 = 32 bytes along K
            const uint64_t ah = sdesc(st + off), al = sdesc(st + T_A_BYTES + off);
            const uint64_t bh = sdesc(st + 2 * T_A_BYTES + off);
            const uint64_t bl = sdesc(st + 2 * T_A_BYTES + T_B_BYTES + off);
            mma_tf32(dt, al, bh, (kb > kb0 || ks) ? 1u : 0u);
            mma_tf32(dt, ah, bl, 1u);
            mma_tf32(dt, ah, bh, 1u);
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp >= 10) {
    // ===== converters (warps 10, 11): raw fp32 -> hi (in place) + lo =====
    if (p.raw_a | p.raw_b) {
      const int ct = threadIdx.x - 320;  // 0..63
      uint32_t q = 0;
      for (int t = blockIdx.x; t < units; t += gridDim.x) {
        const int kb0 = (t / tiles) * p.kbs, kb1 = min(p.nkb, kb0 + p.kbs);
        for (int kb = kb0; kb < kb1; ++kb, ++q) {
          const int s = q % TSTAGES;
          mbar_wait(&full[s], (q / TSTAGES) & 1);
          uint8_t* st = smem + s * T_STAGE_BYTES;
#pragma unroll
          for (int op = 0; op < 2; ++op) {
            if (op == 0 ? !p.raw_a : !p.raw_b) continue;
            float4* hi = reinterpret_cast<float4*>(st + (op == 0 ? 0 : 2 * T_A_BYTES));
            float4* lo = reinterpret_cast<float4*>(st + (op == 0 ? T_A_BYTES : 2 * T_A_BYTES + T_B_BYTES));
#pragma unroll 4
            for (int j = ct; j < T_A_BYTES / 16; j += 64) {
              float4 x = hi[j], h, l;
              uint32_t u;
              asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.x));
              h.x = __uint_as_float(u);
              asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.y));
              h.y = __uint_as_float(u);
              asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.z));
              h.z = __uint_as_float(u);
              asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x.w));
              h.w = __uint_as_float(u);
              l.x = x.x - h.x;
              l.y = x.y - h.y;
              l.z = x.z - h.z;
              l.w = x.w - h.w;
              hi[j] = h;
              lo[j] = l;
            }
          }
          // generic-proxy stores -> visible to the tensor core's async proxy
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&conv[s]))
                         : "memory");
        }
      }
    }
  } else {
    // ===== epilogue (warps 2..9): two warps per TMEM lane quarter, each
    // owning half of the tile's columns =====
    const int quarter = warp & 3;               // TMEM lane quarter of this warp
    const int half = (warp - 2) >> 2;           // column half of the tile
    const int row_t = quarter * 32 + lane;      // row within the tile
    float* tr = trs + (warp - 2) * 32 * T_TP;   // this warp's 32 x 17 transpose tile
    const int etid = threadIdx.x - 64;          // 0..255
    // kernel parameters hoisted into registers once
    const float* Cg = p.C;  // may alias D (in-place update): every element is read before it is written
    const int64_t ldc = p.ldc, ldd = p.ldd;
    const float alpha = p.alpha, beta = p.beta;
    const int M = p.M, N = p.N;
    const bool use_c = beta != 0.0f, fuse = p.fuse != 0;
    constexpr int HN = TBN / 2;  // columns per warp
    float cv[HN];
    auto load_c = [&](int tu, float* dst) {
      const int tt = tu % tiles;
      const int tm2 = tt % p.tiles_m, tn2 = tt / p.tiles_m;
      const int m2 = tm2 * TBM + row_t;
      const int cb2 = tn2 * TBN + half * HN;
      const bool int2 = (tm2 + 1) * TBM <= M && tn2 * TBN + TBN <= N;
      const float* crow = Cg + m2 + (int64_t)cb2 * ldc;
      if (use_c && int2) {
#pragma unroll
        for (int j = 0; j < HN; ++j) dst[j] = __ldg(crow + (int64_t)j * ldc);
      } else {
#pragma unroll
        for (int j = 0; j < HN; ++j)
          dst[j] = (use_c && m2 < M && cb2 + j < N) ? __ldg(crow + (int64_t)j * ldc) : 0.0f;
      }
    };
    int it = 0;
    for (int t = blockIdx.x; t < units; t += gridDim.x, ++it) {
      const int acc = it & 1, use = it >> 1;
      const int tt = t % tiles;
      const int tm = tt % p.tiles_m, tn = tt / p.tiles_m;

      const int m = tm * TBM + row_t;
      const bool rv = m < M;
      const int c_base = tn * TBN + half * HN;
      // interior tiles take an unpredicated path (no per-element bounds)
      const bool interior = (tm + 1) * TBM <= M && tn * TBN + TBN <= N;
      // the thread's C row segment (64 values, L2-resident thanks to the
      // producer's prefetch): loaded at the end of the previous tile's
      // epilogue (software pipelining across tiles), or here for the first
      if (it == 0) load_c(t, cv);
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      // in-tile sums in fp32 (<= 128 terms: error <= ~128 eps32 max|x|, 50x
      // below tau32), converted to fp64 once per published checksum
      float rsum = 0.0f, mx = 0.0f;
      float* drow = p.D + (p.dstride ? (int64_t)(t / tiles) * p.dstride : 0) + m + (int64_t)c_base * ldd;
#pragma unroll
      for (int cc = 0; cc < HN / 32; ++cc) {
        float v[32];
        tmem_ld32(tmem_base + (uint32_t)(acc * TBN + half * HN + cc * 32) +
                      ((uint32_t)(quarter * 32) << 16),
                  v);
        if (interior) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = fmaf(beta, cv[cc * 32 + j], alpha * v[j]);
            drow[(int64_t)(cc * 32 + j) * ldd] = v[j];
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const bool ok = rv && c_base + cc * 32 + j < N;
            const float o = fmaf(beta, cv[cc * 32 + j], alpha * v[j]);
            if (ok) drow[(int64_t)(cc * 32 + j) * ldd] = o;
            v[j] = ok ? o : 0.0f;
          }
        }
        if (fuse) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            rsum += v[j];
            mx = fmaxf(mx, fabsf(v[j]));
          }
          // column sums over this warp's 32 rows, 16 columns per transpose
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
            for (int j = 0; j < 16; ++j) tr[lane * T_TP + j] = v[hh * 16 + j];
            __syncwarp();
            {
              // all 32 lanes: lane l < 16 forms column l's plain sum, lane
              // l + 16 its index-weighted sum (one FADD / FFMA per element)
              const int cl = lane & 15;
              const bool wtd = lane >= 16;
              float a = 0.0f;
#pragma unroll 8
              for (int r = 0; r < 32; ++r) {
                const float x = tr[r * T_TP + cl];
                a = fmaf(wtd ? (float)(quarter * 32 + r) : 1.0f, x, a);
              }
              const int col = half * HN + cc * 32 + hh * 16 + cl;
              float* cq = parts + acc * T_PART_FLOATS + quarter * TBN * 2;
              cq[col * 2 + (wtd ? 1 : 0)] = a;
            }
            __syncwarp();
          }
        }
      }
      // accumulator drained: hand TMEM back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      // next tile's C loads go out now; their latency hides behind the
      // cross-warp combine below and the next accumulator wait
      if (t + (int)gridDim.x < units) load_c(t + gridDim.x, cv);
      if (fuse) {
        const FusedSums& fs = p.sums;
        float* pp = parts + acc * T_PART_FLOATS;
        float* rowp = pp + 4 * TBN * 2;
        float* wmx = rowp + 2 * TBM;
        rowp[half * TBM + row_t] = rsum;
        mx = warp_max(mx);
        if (lane == 0) wmx[warp - 2] = mx;
        // one barrier per tile: the partials are double-buffered by parity,
        // and the barrier of tile i+1 orders this combine before tile i+2
        // overwrites the buffer
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        if (etid < TBN) {
          const int gc = tn * TBN + etid;
          if (gc < N) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              s0 += (double)pp[(qq * TBN + etid) * 2 + 0];
              s1 += (double)pp[(qq * TBN + etid) * 2 + 1];
            }
            fs.cp[fs.cp_step * tm + (int64_t)gc * fs.cp_ld] = s0;
            fs.cw[fs.cw_step * tm + (int64_t)gc * fs.cw_ld] = s1;
          }
          // row etid of the tile: the two column halves in a fixed order
          const int mr = tm * TBM + etid;
          if (mr < M)
            fs.rp[mr + (int64_t)tn * fs.rp_ld] = (double)rowp[etid] + (double)rowp[TBM + etid];
        }
        if (etid == 0) {
          float bmx = 0.0f;
          for (int w8 = 0; w8 < 8; ++w8) bmx = fmaxf(bmx, wmx[w8]);
          fs.bm[tm + (int64_t)tn * fs.bm_ld] = (double)bmx;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                 "n"(T_TMEM_COLS)
                 : "memory");
  }
}

// hi = rna_tf32(x), lo = x - hi, written K-major: out[r * ldo + k].
// trans = 0: src is (R x K) column-major (element (r, k) at r + k * lds),
//            transposed through a 32 x 33 shared tile;
// trans = 1: src already holds (r, k) at k + r * lds (a plain copy).
// Columns K..kpad-1 are written as zeros.
__global__ void tf32_split_kernel(const float* __restrict__ src, int64_t lds, int R, int K, int kpad,
                                  int trans, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t ldo) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  if (!trans) {
    for (int i = ty; i < 32; i += 8) {
      const int r = r0 + tx, k = k0 + i;
      tile[i][tx] = (r < R && k < K) ? src[r + (int64_t)k * lds] : 0.0f;
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
      const int r = r0 + i, k = k0 + tx;
      if (r < R && k < kpad) {
        const float x = (k < K) ? tile[tx][i] : 0.0f;
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(x));
        const float hf = __uint_as_float(h);
        hi[(int64_t)r * ldo + k] = hf;
        lo[(int64_t)r * ldo + k] = x - hf;
      }
    }
  } else {
    for (int i = ty; i < 32; i += 8) {
      const int r = r0 + i, k = k0 + tx;
      if (r < R && k < kpad) {
        const float x = (k < K) ? src[k + (int64_t)r * lds] : 0.0f;
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(x));
        const float hf = __uint_as_float(h);
        hi[(int64_t)r * ldo + k] = hf;
        lo[(int64_t)r * ldo + k] = x - hf;
      }
    }
  }
}

// split-K reduction: D = beta*C + sum_s P_s (fixed order, column-major M x N,
// partials at ldp = M). C may alias D.
__global__ void splitk_reduce_f32(int M, int N, int S, const float* __restrict__ P, int64_t pstride,
                                  float beta, const float* C, int64_t ldc, float* D, int64_t ldd) {
  const int64_t total = (int64_t)M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / M, i = e - j * M;
    float acc = 0.0f;
    for (int s2 = 0; s2 < S; ++s2) acc += __ldg(P + s2 * pstride + e);
    if (beta != 0.0f) acc = fmaf(beta, C[i + j * ldc], acc);
    D[i + j * ldd] = acc;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 2-D map over a K-major fp32 array (rows x ldk, K contiguous), box 32 x 128, 128B swizzle.
int kmajor_map(CUtensorMap* map, const float* base, int64_t rows, int64_t K, int64_t ldk) {
  auto fn = encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return -20;
  }
  // K extent = the operand's own K (columns past it are zero-filled by TMA)
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)(rows < 1 ? 1 : rows)};
  cuuint64_t strides[1] = {(cuuint64_t)(ldk * 4)};
  cuuint32_t box[2] = {TBK, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled(fp32) failed (%d): rows=%lld ldk=%lld", (int)r,
                   (long long)rows, (long long)ldk);
    return -22;
  }
  return 0;
}

}  // namespace

int64_t sgemm_workspace_elems(int M, int N, int K, int splits) {
  const int64_t ldk = (K + 3) / 4 * 4;
  return 2 * ((int64_t)M + N) * ldk + 64 + sgemm_partial_elems(M, N, splits);
}

int64_t sgemm_partial_elems(int M, int N, int splits) {
  return splits > 1 ? (int64_t)splits * M * N + 64 : 0;
}

int sgemm_split_operand(cudaStream_t st, const float* src, int64_t lds, int R, int K, int kpad,
                        int trans, float* hi, float* lo, int64_t ldo) {
  if (R <= 0 || K <= 0) return 0;
  if (kpad < K) kpad = K;
  dim3 g((unsigned)((kpad + 31) / 32), (unsigned)((R + 31) / 32));
  count_launch();
  tf32_split_kernel<<<g, 256, 0, st>>>(src, lds, R, K, kpad, trans, hi, lo, ldo);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

namespace {

float* align256(float* q) {
  return reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(q) + 255) & ~uintptr_t(255));
}

// the tcgen05 launch over K-major split operands (A' row m = row m of op(A),
// B' row n = column n of op(B), both ld elements apart, K contiguous)
int launch_tc(cudaStream_t st, int M, int N, int K, float alpha, const float* ah, const float* al,
              int64_t lda_k, const float* bh, const float* bl, int64_t ldb_k, float beta, const float* C,
              int64_t ldc, float* D, int64_t ldd, float* part, int64_t part_elems, const FusedSums* fs,
              int max_ctas, int splits, int raw_a = 0, int raw_b = 0) {
  CUtensorMap mah, mal, mbh, mbl;
  ABFT_TRY(kmajor_map(&mah, ah, M, K, lda_k));
  ABFT_TRY(kmajor_map(&mal, al, M, K, lda_k));
  ABFT_TRY(kmajor_map(&mbh, bh, N, K, ldb_k));
  ABFT_TRY(kmajor_map(&mbl, bl, N, K, ldb_k));
  SParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.tiles_m = (M + TBM - 1) / TBM;
  p.tiles_n = (N + TBN - 1) / TBN;
  p.nkb = (K + TBK - 1) / TBK;
  if (splits > p.nkb) splits = p.nkb;
  if (splits < 1) splits = 1;
  p.kbs = (p.nkb + splits - 1) / splits;
  splits = (p.nkb + p.kbs - 1) / p.kbs;  // no empty splits
  p.splits = splits;
  p.raw_a = raw_a;
  p.raw_b = raw_b;
  p.alpha = alpha;
  p.fuse = 0;
  p.prefetch_c = 0;
  CUtensorMap mc;
  memset(&mc, 0, sizeof(mc));
  float* pbase = nullptr;
  if (splits > 1) {
    if (fs) {
      set_last_error("sgemm_tc: fused sums need splits == 1");
      return -1;
    }
    pbase = align256(part);
    if (!part || pbase + (int64_t)splits * M * N > part + part_elems) {
      set_last_error("sgemm_tc: split-K partial workspace too small");
      return -1;
    }
    p.C = nullptr;
    p.ldc = M;
    p.D = pbase;
    p.ldd = M;
    p.beta = 0.0f;
    p.dstride = (int64_t)M * N;
  } else {
    p.C = C;
    p.ldc = ldc;
    p.D = D;
    p.ldd = ldd;
    p.beta = (C == nullptr) ? 0.0f : beta;
    p.dstride = 0;
    p.fuse = fs ? 1 : 0;
    if (fs) p.sums = *fs;
    // only worth a descriptor when CTAs run several tiles (the prefetch for
    // tile i+1 overlaps tile i); tiny launches stay host-cheap
    if (p.beta != 0.0f && (reinterpret_cast<uintptr_t>(C) & 15) == 0 && (ldc % 4) == 0 &&
        (int64_t)p.tiles_m * p.tiles_n > 148) {
      auto fn = encode_fn();
      cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)N};
      cuuint64_t strides[1] = {(cuuint64_t)(ldc * 4)};
      cuuint32_t box[2] = {TBM, TBN};
      cuuint32_t estr[2] = {1, 1};
      if (fn && fn(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(C), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        p.prefetch_c = 1;
    }
  }
  ABFT_TRY(ensure_smem_attr((const void*)sgemm_tc05_kernel, T_SMEM));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (max_ctas > 0 && max_ctas < sms) sms = max_ctas;
  const int units = p.tiles_m * p.tiles_n * splits;
  const int grid = units < sms ? units : sms;
  count_launch();
  sgemm_tc05_kernel<<<grid, T_THREADS, T_SMEM, st>>>(mah, mal, mbh, mbl, mc, p);
  CUDA_TRY(cudaGetLastError());
  if (splits > 1) {
    const int64_t total = (int64_t)M * N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4 * (int64_t)sms);
    count_launch();
    splitk_reduce_f32<<<blocks, 256, 0, st>>>(M, N, splits, pbase, (int64_t)M * N,
                                              C ? beta : 0.0f, C, ldc, D, ldd);
    CUDA_TRY(cudaGetLastError());
  }
  return 0;
}

}  // namespace

int sgemm_tc(cudaStream_t st, char ta, char tb, int M, int N, int K, float alpha, const float* A,
             int64_t lda, const float* B, int64_t ldb, float beta, const float* C, int64_t ldc,
             float* D, int64_t ldd, float* ws, int64_t ws_elems, const FusedSums* fs, int max_ctas,
             int splits) {
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0) {
    set_last_error("sgemm_tc needs K > 0");
    return -1;
  }
  const int64_t ldk = (K + 3) / 4 * 4;
  if (!ws || ws_elems < sgemm_workspace_elems(M, N, K, splits)) {
    set_last_error("sgemm_tc workspace too small");
    return -1;
  }
  // K-major sources ('T' A, 'N' B) go to the kernel raw (split in shared
  // memory) when TMA can address them directly
  static const bool raw_ok = [] {
    const char* e = getenv("ABFT_SGEMM_RAW");
    return !(e && e[0] == '0');
  }();
  auto tma_ok = [](const float* q, int64_t ld) {
    return (reinterpret_cast<uintptr_t>(q) & 15) == 0 && (ld % 4) == 0;
  };
  // 256-byte aligned operand copies inside the workspace
  float* ah = align256(ws);
  float* al = align256(ah + (int64_t)M * ldk);
  float* bh = align256(al + (int64_t)M * ldk);
  float* bl = align256(bh + (int64_t)N * ldk);
  float* part = bl + (int64_t)N * ldk;
  if (part > ws + ws_elems) {
    set_last_error("sgemm_tc workspace too small (alignment)");
    return -1;
  }
  // A: op(A) is M x K. 'N': (m, k) at m + k*lda -> transpose; 'T': (m, k) at k + m*lda -> copy.
  const bool AT = (ta == 'T' || ta == 't');
  const bool BT = (tb == 'T' || tb == 't');
  // the converter re-splits an operand box for every tile that reads it:
  // worth it only while the operand is read by at most two tile rows /
  // columns (else the one-time split pass is cheaper)
  const int tiles_m = (M + TBM - 1) / TBM, tiles_n = (N + TBN - 1) / TBN;
  const bool raw_a = raw_ok && AT && tiles_n <= 2 && tma_ok(A, lda);
  const bool raw_b = raw_ok && !BT && tiles_m <= 2 && tma_ok(B, ldb);
  if (!raw_a) ABFT_TRY(sgemm_split_operand(st, A, lda, M, K, (int)ldk, AT ? 1 : 0, ah, al, ldk));
  // op(B) is K x N; B' row n = column n of op(B): 'N': (k, n) at k + n*ldb -> copy;
  // 'T': (k, n) at n + k*ldb -> transpose.
  if (!raw_b) ABFT_TRY(sgemm_split_operand(st, B, ldb, N, K, (int)ldk, BT ? 0 : 1, bh, bl, ldk));
  return launch_tc(st, M, N, K, alpha, raw_a ? A : ah, raw_a ? A : al, raw_a ? lda : ldk,
                   raw_b ? B : bh, raw_b ? B : bl, raw_b ? ldb : ldk, beta, C, ldc, D, ldd, part,
                   ws + ws_elems - part, fs, max_ctas, splits, raw_a, raw_b);
}

int sgemm_tc_presplit(cudaStream_t st, int M, int N, int K, float alpha, const float* ah,
                      const float* al, int64_t lda_k, const float* bh, const float* bl, int64_t ldb_k,
                      float beta, const float* C, int64_t ldc, float* D, int64_t ldd, float* part,
                      int64_t part_elems, int max_ctas, int splits) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  if ((lda_k % 4) || (ldb_k % 4) || (reinterpret_cast<uintptr_t>(ah) & 15) ||
      (reinterpret_cast<uintptr_t>(al) & 15) || (reinterpret_cast<uintptr_t>(bh) & 15) ||
      (reinterpret_cast<uintptr_t>(bl) & 15)) {
    set_last_error("sgemm_tc_presplit: operands must be 16-byte aligned with ld % 4 == 0");
    return -1;
  }
  return launch_tc(st, M, N, K, alpha, ah, al, lda_k, bh, bl, ldb_k, beta, C, ldc, D, ldd, part,
                   part_elems, nullptr, max_ctas, splits);
}

}  // namespace abft
