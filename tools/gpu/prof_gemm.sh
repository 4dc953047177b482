#!/bin/bash
# ncu --set full of the first LU N=32768 iterations' DMMA GEMM launches (the
# trailing update is the longest one), fused (FULL) and plain (scheme none)
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:dgemm_tma_dmma -c 10 -o gpurun_out/prof_gemm_full_$TAG \
  python bench.py --profile-only > gpurun_out/prof_gemm_full_$TAG.log 2>&1; echo "gemm fused rc=$?"
timeout 1200 $NCU -k regex:dgemm_tma_dmma -c 10 -o gpurun_out/prof_gemm_none_$TAG \
  python bench.py --profile-only --scheme none > gpurun_out/prof_gemm_none_$TAG.log 2>&1; echo "gemm none rc=$?"
