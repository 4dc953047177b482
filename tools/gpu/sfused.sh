set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_single.py tests/test_gpu_sgemm.py -m gpu -x -q > gpurun_out/tests_sfused.log 2>&1; echo "tests rc=$?"
for k in lu qr cholesky; do
timeout 900 python bench.py --kind $k --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_s${k}_fused.json 2>&1; echo "s$k rc=$?"
done
