#!/bin/bash
# ncu --set full with source-level sampling of the first LU N=32768 trailing
# update (dgemm launch #3 of iteration 0: L21, U12, next block column, then the
# fused rest), FULL (fused checksum epilogue) and scheme none (plain).
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:dgemm_tma_dmma -s 3 -c 1 -o gpurun_out/prof_gemmsrc_full_$TAG \
  python bench.py --profile-only > gpurun_out/prof_gemmsrc_full_$TAG.log 2>&1; echo "gemm fused rc=$?"
timeout 900 $NCU -k regex:dgemm_tma_dmma -s 3 -c 1 -o gpurun_out/prof_gemmsrc_none_$TAG \
  python bench.py --profile-only --scheme none > gpurun_out/prof_gemmsrc_none_$TAG.log 2>&1; echo "gemm none rc=$?"
