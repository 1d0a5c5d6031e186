#!/bin/bash
# A/B of the fused step kernel versions (KR_STEP_V=1: v1, 4 y-strided cells per thread; default v2: 2 x 2 cells):
# C5 + its dense companion C5D and C4, alternating, same box. Usage (under gpurun): bash scripts/ab_step.sh tag
tag=${1:-x}
for rep in 1 2; do
  for v in 2 1; do
    for cfg in C5 C4; do
      KR_STEP_V=$v timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${tag}_v${v}_${cfg}_$rep.log 2>&1
      python - "$v" "$cfg" "gpurun_out/ab_${tag}_v${v}_${cfg}_$rep.log" <<'PY'
import json, sys
v, cfg, f = sys.argv[1:4]
try:
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
except Exception as e:
    print(f"v{v} {cfg} FAILED {e}"); sys.exit()
fs = d["fused_step"]
out = f"v{v} {cfg}: {d['value']:.1f} steps/s step {fs['ms_mean']:.4f} ms frac {d['roofline']['frac']:.4f} sm {d['clocks']['sm_mhz']} {d['clocks']['reasons']}"
if "dense" in d:
    dd = d["dense"]
    out += f" | dense {dd['value']:.1f} steps/s step {dd['fused_step']['ms_mean']:.4f} ms frac {dd['roofline']['frac']:.4f} sm {dd['clocks']['sm_mhz']} {dd['clocks']['reasons']}"
print(out)
PY
    done
  done
done
