set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:blocksum --launch-skip 21 -c 2 -o gpurun_out/bs_schol python bench.py --kind cholesky --precision f32 --n 16384 --b 128 --profile-only > gpurun_out/bs_prof.log 2>&1; echo rc=$?
