#!/bin/bash
# A/B of runtime switches on one library build (under gpurun): per-step times of C5 and C4 (scripts/step_profile.py)
# and the dense C5D bench line, alternating twice. Usage: bash scripts/ab_env.sh "label:VAR=1 VAR2=x" "base:" ...
for rep in 1 2; do
  for spec in "$@"; do
    lab=${spec%%:*}; envs=${spec#*:}
    for cfg in C5 C4; do echo "$lab $cfg: $(env $envs python scripts/step_profile.py $cfg | cut -d: -f2)"; done
    env $envs timeout 300 python bench.py --config C5D --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abe_$lab.log 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/abe_$lab.log') if l.startswith('{')][-1])
print('$lab C5D:', round(d['value'],1), 'steps/s step', round(d['fused_step']['ms_mean'],4), 'frac', round(d['roofline']['frac'],4), d['clocks'])"
  done
done
