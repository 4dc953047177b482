#!/bin/bash
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for v in 0 1; do for m in 0 1; do python tools/prof/diag_probe.py $v $m 256 20; done; done > gpurun_out/diag_probe_$TAG.txt 2>&1
python tools/prof/diag_probe.py 1 1 128 20 >> gpurun_out/diag_probe_$TAG.txt 2>&1
python tools/prof/diag_probe.py 0 1 128 20 >> gpurun_out/diag_probe_$TAG.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:coop_factor -c 1 -o gpurun_out/prof_cf_$TAG python tools/prof/diag_probe.py 1 0 256 1 > gpurun_out/prof_cf_$TAG.log 2>&1; echo "ncu rc=$?"
