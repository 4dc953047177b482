set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for l in 400 800 1200 1600; do
ABFT_QR_LA_LAT_US=$l timeout 900 python bench.py --kind qr --no-cpu --no-e2e --no-overhead --steps 3 --warmup 1 > gpurun_out/bench_qr_lat$l.json 2>&1; echo "lat $l rc=$?"
done
