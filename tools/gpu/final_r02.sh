#!/bin/bash
# Round-2 checkpoint: GPU tests, smoke, every bench line, launch lists, ncu of
# the small-factor kernel and the QR panel's tall GEMM.
set -u
TAG=${1:-r02z}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/bench_lu_$TAG.json 2> gpurun_out/bench_lu_$TAG.err; echo "bench lu rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "bench ref rc=$?"
for k in cholesky qr; do
  timeout 1200 python bench.py --kind $k --no-cpu > gpurun_out/bench_${k}_$TAG.json 2> gpurun_out/bench_${k}_$TAG.err; echo "bench $k rc=$?"
done
for k in lu cholesky qr; do
  timeout 900 python bench.py --kind $k --precision f32 --n 16384 --b 128 --no-cpu > gpurun_out/bench_s${k}_$TAG.json 2> gpurun_out/bench_s${k}_$TAG.err; echo "bench s$k rc=$?"
done
for k in lu qr; do
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches_${k}_$TAG.csv python bench.py --kind $k --profile-only > gpurun_out/launches_${k}_$TAG.log 2>&1; echo "launches $k rc=$?"
done
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:coop_factor -c 3 -o gpurun_out/prof_cf_$TAG python bench.py --kind qr --profile-only > gpurun_out/prof_cf_$TAG.log 2>&1; echo "ncu cf rc=$?"
for k in lu cholesky qr; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches_s${k}_$TAG.csv python bench.py --kind $k --precision f32 --n 16384 --b 128 --profile-only > gpurun_out/launches_s${k}_$TAG.log 2>&1; echo "launches s$k rc=$?"
done
