#!/bin/bash
# A/B of library builds on the L2-resident workloads (C3, P100 bench lines; under gpurun), alternating twice.
# Usage: bash scripts/ab_small.sh name1 name2 ...   (scratch_libs/libkr_<name>.so)
for rep in 1 2; do
  for lib in "$@"; do
    cp scratch_libs/libkr_$lib.so paper_1804_01583_b200/libkrylov_reach.so
    for cfg in C3 P100; do
      timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abs_$lib.log 2>&1
      python -c "
import json; d=json.loads([l for l in open('gpurun_out/abs_$lib.log') if l.startswith('{')][-1])
print('$lib $cfg:', round(d['value'],1), 'steps/s', round(d['ms_per_step'],4), 'ms per run; step', round(d['fused_step']['ms_mean']*1000,2), 'us')"
    done
  done
done
