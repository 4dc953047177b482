#!/bin/bash
# ncu --set full with source-level sampling of one fused LU trailing-update GEMM
# (N=32768, an early iteration) and one plain (scheme none) launch.
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:dgemm_tma_dmma -s 40 -c 1 -o gpurun_out/prof_gemmsrc_full_$TAG \
  python bench.py --profile-only > gpurun_out/prof_gemmsrc_full_$TAG.log 2>&1; echo "gemm fused rc=$?"
timeout 1200 $NCU -k regex:dgemm_tma_dmma -s 40 -c 1 -o gpurun_out/prof_gemmsrc_none_$TAG \
  python bench.py --profile-only --scheme none > gpurun_out/prof_gemmsrc_none_$TAG.log 2>&1; echo "gemm none rc=$?"
