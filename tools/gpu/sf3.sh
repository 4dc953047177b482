set -u
./tools/probe/cf_trace 256 0 > gpurun_out/cf_trace.txt 2>&1
./tools/probe/cf_trace 256 1 >> gpurun_out/cf_trace.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "diag_factor" > gpurun_out/tests_sf.log 2>&1; echo "sf tests rc=$?"
for v in 0 1; do for m in 0 1 2; do python tools/prof/diag_probe.py $v $m 256 20; done; done > gpurun_out/diag_probe.txt 2>&1
for v in 0 1; do python tools/prof/diag_probe.py $v 1 128 20; done >> gpurun_out/diag_probe.txt 2>&1
