#!/bin/bash
# A/B of two builds on the same box: default library vs build_ab/libabft_old.so
for i in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export ABFT_LIB=$PWD/build_ab/libabft_old.so; else unset ABFT_LIB; fi
    timeout 600 python bench.py --no-cpu --no-e2e --no-overhead > gpurun_out/ab_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],3), round(d['profile_ms']['tmu_gemm'],1))"
  done
done
