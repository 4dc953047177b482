#!/bin/bash
mkdir -p gpurun_out
for nb in "1024 256" "4096 256" "4096 128"; do
  set -- $nb
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    tools/debug/dist_lu_debug.py $1 $2 > gpurun_out/dbg_$1_$2.log 2>&1; echo "dbg $1 $2 rc=$?"; grep -E "ok|FAIL" gpurun_out/dbg_$1_$2.log
done
timeout 600 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/dist_tests.log 2>&1; echo "dist tests rc=$?"; tail -15 gpurun_out/dist_tests.log
