#!/bin/bash
# A/B of the multi-CTA slab reduction (KR_RED_CTAS=1 = the former one-CTA reduce) + the GPU suite.
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_red.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_red.log
for rep in 1 2; do
for g in 1 default; do
  if [ $g = default ]; then unset KR_RED_CTAS; else export KR_RED_CTAS=$g; fi
  for c in C5 C4 C3; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"red=$g $c\", round(d[\"value\"],2), round(d[\"ms_per_step\"],3), round(d[\"iter_ms_mean\"],3))"; done
done
done
