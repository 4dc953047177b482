set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for k in cholesky lu qr; do
  timeout 600 python bench.py --kind $k --precision f32 --n 16384 --b 128 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_s${k}_bs.json 2>&1; echo "s$k rc=$?"
done
timeout 900 python bench.py --kind lu --no-cpu --no-e2e --no-overhead --steps 3 > gpurun_out/bench_lu_bs.json 2>&1; echo "lu rc=$?"
