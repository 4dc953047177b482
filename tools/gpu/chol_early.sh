set -u
mkdir -p gpurun_out
for e in 0 64 80 96; do
  ABFT_CHOL_EARLY=$e timeout 600 python bench.py --kind cholesky --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --no-overhead --steps 3 > gpurun_out/bench_sce_$e.json 2>&1; echo "early $e rc=$?"
done

