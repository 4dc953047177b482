set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "diag_factor" > gpurun_out/tests_sf.log 2>&1; echo "sf tests rc=$?"
for v in 0 1; do for m in 0 1 2; do python tools/prof/diag_probe.py $v $m 256 20; done; done > gpurun_out/diag_probe.txt 2>&1
for v in 0 1; do python tools/prof/diag_probe.py $v 1 128 20; done >> gpurun_out/diag_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_factorizations.py tests/test_gpu_fused.py tests/test_gpu_single.py tests/test_distributed.py -m gpu -x -q > gpurun_out/tests_q.log 2>&1; echo "tests rc=$?"
ABFT_QR_LA_SMS=16 timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_coop16.json 2>&1; echo "qr16 rc=$?"
ABFT_QR_LA_SMS=12 timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_coop12.json 2>&1; echo "qr12 rc=$?"
timeout 900 python bench.py --kind qr --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_sqr_coop.json 2>&1; echo "sqr rc=$?"
timeout 900 python bench.py --kind cholesky --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_schol_coop.json 2>&1; echo "schol rc=$?"
ABFT_CHOL_CLUSTER=1 timeout 900 python bench.py --kind cholesky --no-cpu --no-e2e --steps 2 > gpurun_out/bench_chol_coop.json 2>&1; echo "chol rc=$?"
