set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_factorizations.py -m gpu -x -q > gpurun_out/tests_adapt.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --kind qr --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/bench_qr_adapt.json 2>&1; echo "qr rc=$?"
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench_lu_adapt.json 2>&1; echo "lu rc=$?"
ABFT_LU_COOP=0 timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench_lu_nocoop.json 2>&1; echo "lu0 rc=$?"
