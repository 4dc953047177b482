set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_single.py tests/test_gpu_fused.py -q -x -k "streamed" 2>&1 | tail -3
timeout 900 python bench.py --kind cholesky --precision f32 --n 16384 --b 128 --no-cpu --no-overhead --steps 3 > gpurun_out/bench_schol_si.json 2>gpurun_out/bench_schol_si.err; echo "schol rc=$?"
