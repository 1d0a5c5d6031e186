#!/bin/bash
# A/B of library builds (scratch_libs/libkr_<name>.so copied over the in-tree library in the box's copy of the
# repo): per-step times of C5 and C4 (scripts/step_profile.py) and the dense C5D bench line, alternating twice.
# Usage (under gpurun): bash scripts/ab_libs.sh name1 name2 ...

for rep in 1 2; do
  for lib in "$@"; do
    cp scratch_libs/libkr_$lib.so paper_1804_01583_b200/libkrylov_reach.so
    for cfg in C5 C4; do echo "$lib $cfg: $(python scripts/step_profile.py $cfg | cut -d: -f2)"; done
    timeout 300 python bench.py --config C5D --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abl_$lib.log 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/abl_$lib.log') if l.startswith('{')][-1])
print('$lib C5D:', round(d['value'],1), 'steps/s step', round(d['fused_step']['ms_mean'],4), 'frac', round(d['roofline']['frac'],4), d['clocks'])"
  done
done
