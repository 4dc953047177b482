#!/bin/bash
# LU fused GEMM source-level ncu + fp32 launch lists (sgetrf / spotrf, FULL and none)
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:dgemm_tma_dmma -s 40 -c 1 -o gpurun_out/prof_gemmsrc_full_$TAG \
  python bench.py --profile-only > gpurun_out/prof_gemmsrc_full_$TAG.log 2>&1; echo "gemm fused rc=$?"
for s in full none; do
  for k in lu cholesky; do
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
      --log-file gpurun_out/launches_s${k}_${s}_$TAG.csv python bench.py --precision f32 --kind $k --n 16384 --b 128 --scheme $s --profile-only > gpurun_out/launches_s${k}_${s}_$TAG.log 2>&1; echo "launches s$k $s rc=$?"
  done
done
