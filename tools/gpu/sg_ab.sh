set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "single or sgemm or s_ or f32 or fp32" 2>&1 | tail -3
for k in lu qr cholesky; do
  timeout 600 python bench.py --kind $k --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_s${k}_sg.json 2>&1; echo "s$k rc=$?"
done
