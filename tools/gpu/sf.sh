#!/bin/bash
# cluster diagonal-block factorization: kernel tests, QR tests, dgeqrf / sgeqrf benches + launch list
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "diag_factor" > gpurun_out/tests_sf_$TAG.log 2>&1; echo "sf tests rc=$?"
timeout 900 python -m pytest tests/test_gpu_factorizations.py tests/test_gpu_fused.py tests/test_gpu_single.py -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"
for s in 16 8; do
  ABFT_QR_LA_SMS=$s timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_la${s}_$TAG.json 2> gpurun_out/bench_qr_la${s}_$TAG.err; echo "qr la=$s rc=$?"
done
ABFT_QR_LA_SMS=0 timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_la0_$TAG.json 2> gpurun_out/bench_qr_la0_$TAG.err; echo "qr la=0 rc=$?"
timeout 900 python bench.py --kind qr --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_sqr_$TAG.json 2> gpurun_out/bench_sqr_$TAG.err; echo "sqr rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches_qr_$TAG.csv python bench.py --kind qr --profile-only > gpurun_out/launches_qr_$TAG.log 2>&1; echo "launches rc=$?"
