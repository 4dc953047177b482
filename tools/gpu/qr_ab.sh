#!/bin/bash
# QR panel: GPU tests, then dgeqrf / sgeqrf benches with the tensor-core panel
# (default) and the cooperative per-column panel (ABFT_QR_PANEL=coop).
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_$TAG.json 2> gpurun_out/bench_qr_$TAG.err; echo "qr rc=$?"
timeout 900 python bench.py --kind qr --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_sqr_$TAG.json 2> gpurun_out/bench_sqr_$TAG.err; echo "sqr rc=$?"
ABFT_QR_PANEL=coop timeout 900 python bench.py --kind qr --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_sqr_coop_$TAG.json 2> gpurun_out/bench_sqr_coop_$TAG.err; echo "sqr coop rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_qr_$TAG.csv python bench.py --kind qr --profile-only > gpurun_out/launches_qr_$TAG.log 2>&1; echo "launches rc=$?"
