#!/bin/bash
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "diag_factor" > gpurun_out/tests_sf_$TAG.log 2>&1; echo "sf tests rc=$?"
for v in 0 1; do for m in 0 1 2; do python tools/prof/diag_probe.py $v $m 256 20; done; done > gpurun_out/diag_probe_$TAG.txt 2>&1
for v in 0 1; do python tools/prof/diag_probe.py $v 1 128 20; done >> gpurun_out/diag_probe_$TAG.txt 2>&1
ABFT_QR_LA_SMS=16 timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_cf_$TAG.json 2> gpurun_out/bench_qr_cf_$TAG.err; echo "qr cf rc=$?"
ABFT_QR_LA_SMS=0 timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_cf0_$TAG.json 2> gpurun_out/bench_qr_cf0_$TAG.err; echo "qr cf la0 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:coop_factor -c 1 -o gpurun_out/prof_cf_$TAG python tools/prof/diag_probe.py 1 0 256 1 > gpurun_out/prof_cf_$TAG.log 2>&1; echo "ncu rc=$?"
