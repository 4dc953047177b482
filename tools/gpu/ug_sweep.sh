#!/bin/bash
mkdir -p gpurun_out
for g in 0 16 32 64 128; do
  ABFT_UNIT_GROUP=$g timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/ug_$g.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ug_$g.json').read().strip().splitlines()[-1]); print('group $g', round(d['value'],3), round(d['abft_overhead_pct'],2), round(d['profile_ms']['tmu_gemm'],1))"
done
