#!/bin/bash
# Round-2 late checkpoint: GPU tests, smoke, every bench line (no ncu).
set -u
TAG=${1:-r02g}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/tests_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/bench_lu_$TAG.json 2> gpurun_out/bench_lu_$TAG.err; echo "bench lu rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "bench ref rc=$?"
for k in cholesky qr; do
  timeout 1200 python bench.py --kind $k --no-cpu > gpurun_out/bench_${k}_$TAG.json 2> gpurun_out/bench_${k}_$TAG.err; echo "bench $k rc=$?"
done
for k in lu cholesky qr; do
  timeout 900 python bench.py --kind $k --precision f32 --n 16384 --b 128 --no-cpu > gpurun_out/bench_s${k}_$TAG.json 2> gpurun_out/bench_s${k}_$TAG.err; echo "bench s$k rc=$?"
done
