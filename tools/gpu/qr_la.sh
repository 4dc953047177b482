#!/bin/bash
# QR look-ahead: QR/fused GPU tests, then dgeqrf N=32768 at several side-stream SM counts.
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_factorizations.py tests/test_gpu_fused.py -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"
for s in 16 8 24 0; do
  ABFT_QR_LA_SMS=$s timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_la${s}_$TAG.json 2> gpurun_out/bench_qr_la${s}_$TAG.err; echo "qr la=$s rc=$?"
done
