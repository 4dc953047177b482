set -u
mkdir -p gpurun_out
for v in 1 0; do
  ABFT_LU_COOP=$v timeout 900 python bench.py --kind lu --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_slu_coop$v.json 2>&1; echo "slu $v rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_single.py -m gpu -x -q > gpurun_out/tests_single.log 2>&1; echo "tests rc=$?"
