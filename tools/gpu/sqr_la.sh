set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_single.py tests/test_governor.py -m gpu -x -q > gpurun_out/tests_sqr.log 2>&1; echo "tests rc=$?"
for s in 16 24 0; do
ABFT_QR_LA_SMS=$s timeout 900 python bench.py --kind qr --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_sqr_la$s.json 2>&1; echo "sqr $s rc=$?"
done
timeout 900 python bench.py --kind cholesky --no-cpu --no-e2e --steps 2 > gpurun_out/bench_chol_tmu.json 2>&1; echo "chol rc=$?"
