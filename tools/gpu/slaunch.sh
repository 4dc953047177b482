set -u
TAG=${1:-r02s}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in lu cholesky qr; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches_s${k}_$TAG.csv python bench.py --kind $k --precision f32 --n 16384 --b 128 --profile-only > gpurun_out/launches_s${k}_$TAG.log 2>&1; echo "launches s$k rc=$?"
done
