set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1

timeout 1200 python bench.py --kind cholesky --no-cpu --no-overhead --steps 3 > gpurun_out/bench_chol_si.json 2>gpurun_out/bench_chol_si.err; echo "chol rc=$?"
