#!/bin/bash
# One GPU session: tests, bench, launch list, ncu --set full of the top kernel.
# usage: tools/gpu/round.sh [tag] [what...]   what in {tests,bench,launches,full}
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-tests bench launches full}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for w in $WHAT; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?" ;;
    smoke) timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" ;;
    benchall) for k in cholesky qr; do timeout 1200 python bench.py --kind $k --no-cpu --no-e2e > gpurun_out/bench_${k}_$TAG.json 2> gpurun_out/bench_${k}_$TAG.err; echo "bench $k rc=$?"; done ;;
    launches) timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
        --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?" ;;
    full) timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_dmma -s 40 -c 2 \
        -o gpurun_out/prof_gemm_$TAG python bench.py --profile-only > gpurun_out/prof_gemm_$TAG.log 2>&1; echo "full rc=$?" ;;
  esac
done
