#!/bin/bash
# Cholesky PD on the cluster kernel vs the one-CTA kernel (dpotrf N=32768, spotrf N=16384) + tests
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_factorizations.py tests/test_gpu_fused.py tests/test_gpu_single.py -m gpu -x -q -k "cholesky or chol or c1 or run_protected or criterion" > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"
for cl in 1 0; do
  ABFT_CHOL_CLUSTER=$cl timeout 900 python bench.py --kind cholesky --no-cpu --no-e2e --steps 3 > gpurun_out/bench_chol_cl${cl}_$TAG.json 2> gpurun_out/bench_chol_cl${cl}_$TAG.err; echo "chol cl=$cl rc=$?"
  ABFT_CHOL_CLUSTER=$cl timeout 900 python bench.py --kind cholesky --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_schol_cl${cl}_$TAG.json 2> gpurun_out/bench_schol_cl${cl}_$TAG.err; echo "schol cl=$cl rc=$?"
done
