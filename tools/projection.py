"""Per-iteration critical-path projection of the block-cyclic ABFT
factorizations on G B200s. Not a measurement: a model whose
constants come from the 1-GPU measurements in profiles/ (stated below), so the
G = 1 column can be checked against the measured bench lines.

  python tools/projection.py [--n 32768] [--b 256] [--bw 400] [--diag-us 470]

Per iteration k (p = k b, m = n - p rows, owner o = k mod G):
  LU  (cross-rank look-ahead, csrc/dist.cu update_lu_lookahead):
      T_k = max(U_k, C_{k+1})   U_k = trailing update of one rank's columns
      C_{k+1} = column-block update + diagonal factor + L21 GEMM + broadcast
  QR  (cross-rank look-ahead): U_k = V^T C, T^T W, C -= V mid on the rank's
      columns; C_{k+1} = column update + tensor-core panel + broadcast (V, T)
  Cholesky left-looking (today's dist path, no look-ahead):
      T_k = partial panel GEMM (K = p / G) + sum-reduce + owner encode/verify
            + diagonal factor + L21 GEMM
  Cholesky right-looking + look-ahead (the design of DESIGN.md §7):
      T_k = max(U_k, C_{k+1}), U_k = lower-triangular rank-b update of the
      rank's columns, C_{k+1} = its block column update + verify + diag + PU +
      broadcast
GEMM time: persistent wave model of the DMMA kernel (64 x 64 tiles, one unit
per SM per wave) at the measured per-SM rate of the fused trailing update
(30.0 TFLOP/s over 148 SMs, profiles/bench_lu32k_r02.json); the diagonal
factorization at its measured one-CTA latency (~470 us, tools/prof/diag_probe.py);
collectives alpha + bytes / bw (alpha = 20 us, bw = NCCL broadcast / reduce
bus bandwidth over NVLink 5, 400 GB/s assumed -- below the 900 GB/s link rate).
"""
from __future__ import annotations

import argparse
import math

PEAK = 37.06e12          # measured DMMA issue peak per GPU (abft_probe_dmma_peak)
SMS = 148
RATE_SM = 30.0e12 / SMS  # measured fused trailing-update rate per SM


def gemm_t(m, n, k, sms=SMS, tile=64):
    if m <= 0 or n <= 0 or k <= 0:
        return 0.0
    units = math.ceil(m / tile) * math.ceil(n / tile)
    waves = math.ceil(units / sms)
    return waves * (2.0 * tile * tile * k) / RATE_SM + 5e-6


def coll_t(nbytes, bw, G, alpha=20e-6):
    return alpha + nbytes / bw if G > 1 else 0.0


def local_cols(n, b, g, G, k0):
    """columns of rank g among global blocks > k0"""
    nb = -(-n // b)
    return sum(min(b, n - j * b) for j in range(k0 + 1, nb) if j % G == g)


def project(kind, n, b, G, bw, diag_s, qr_panel_s_per_row):
    nb = -(-n // b)
    total = 0.0
    for k in range(nb):
        p, pe = k * b, min(k * b + b, n)
        m = n - p
        if kind == "lu":
            cols = max(local_cols(n, b, g, G, k) for g in range(G))
            U = gemm_t(n - pe, cols, b)
            chain = (gemm_t(n - pe, b, b) + diag_s + gemm_t(n - pe - b, b, b) +
                     coll_t(8 * (n - pe) * b, bw, G)) if k + 1 < nb else 0.0
            total += max(U, chain)
        elif kind == "qr":
            cols = max(local_cols(n, b, g, G, k) for g in range(G))
            U = gemm_t(b, cols, m) + gemm_t(m, cols, b)  # V^T C (split-K-less model) + C -= V mid
            panel = qr_panel_s_per_row * (m - b) + 3 * diag_s
            chain = (gemm_t(m, b, b) + panel + coll_t(8 * (m * b + b * b), bw, G)) if k + 1 < nb else 0.0
            total += max(U, chain)
        elif kind == "chol_left":
            Kp = math.ceil(p / G)
            part = gemm_t(m, b, Kp)
            red = coll_t(8 * m * (b + 1), bw, G)
            owner = diag_s + gemm_t(m - b, b, b) + 2 * (8 * m * b) / 6.5e12
            total += part + red + owner
        elif kind == "chol_right":
            # lower-triangular update: rank's columns j > k, rows >= j b
            # one launch over the rank's column blocks j > k with the tiles
            # above each block's diagonal skipped (rows >= j b only)
            worst = 0.0
            for g in range(G):
                units = sum(math.ceil((n - j * b) / 64) * math.ceil(min(b, n - j * b) / 64)
                            for j in range(k + 1, nb) if j % G == g)
                worst = max(worst, math.ceil(units / SMS) * 2.0 * 64 * 64 * b / RATE_SM)
            chain = (gemm_t(m - b, b, b) + diag_s + gemm_t(m - 2 * b, b, b) +
                     coll_t(8 * (m - b) * b, bw, G)) if k + 1 < nb else 0.0
            total += max(worst, chain)
    flops = {"lu": 2 * n ** 3 / 3, "qr": 4 * n ** 3 / 3,
             "chol_left": n ** 3 / 3, "chol_right": n ** 3 / 3}[kind]
    return flops / total / 1e12, flops / total / (G * PEAK)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--bw", type=float, default=400.0, help="collective bus bandwidth, GB/s")
    ap.add_argument("--diag-us", type=float, default=470.0)
    ap.add_argument("--qr-panel-us-per-krow", type=float, default=18.0,
                    help="tensor-core panel time per 1000 rows (measured ~0.6 ms at 32768)")
    a = ap.parse_args()
    print(f"# N={a.n} b={a.b} collective bw {a.bw} GB/s, diagonal factor {a.diag_us} us")
    print(f"{'kind':12s} " + " ".join(f"G={G:<2d} TF/s (frac)" for G in (1, 2, 4, 8)))
    for kind in ("lu", "qr", "chol_left", "chol_right"):
        row = []
        for G in (1, 2, 4, 8):
            tf, fr = project(kind, a.n, a.b, G, a.bw * 1e9, a.diag_us * 1e-6,
                             a.qr_panel_us_per_krow * 1e-9)
            row.append(f"{tf:7.1f} ({fr:4.2f})  ")
        print(f"{kind:12s} " + " ".join(row))


if __name__ == "__main__":
    main()
