#!/bin/bash
# 2 ranks sharing one GPU over gloo: exercises bench.py's N>1 path end to end.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/dist_tests.log 2>&1; echo "dist tests rc=$?"
for k in lu qr cholesky; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --dist-backend gloo --kind $k --order 4096 --steps 2 --warmup 1 --no-cpu \
    > gpurun_out/dist_bench_$k.json 2> gpurun_out/dist_bench_$k.err; echo "dist bench $k rc=$?"
done
