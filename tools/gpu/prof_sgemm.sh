set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:sgemm_tc05 -s 3 -c 1 -o gpurun_out/prof_sgemm_full python bench.py --precision f32 --kind lu --n 16384 --b 128 --profile-only > gpurun_out/prof_sgemm_full.log 2>&1; echo "full rc=$?"
timeout 900 $NCU -k regex:sgemm_tc05 -s 3 -c 1 -o gpurun_out/prof_sgemm_none python bench.py --precision f32 --kind lu --n 16384 --b 128 --scheme none --profile-only > gpurun_out/prof_sgemm_none.log 2>&1; echo "none rc=$?"
