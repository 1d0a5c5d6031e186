#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_next1.py -q --timeout 600 -p no:cacheprovider > gpurun_out/next1_f.log 2>&1; echo rc=$?; tail -2 gpurun_out/next1_f.log
for kd in 1536 0 3000; do
  KR_KDOUBLE=$kd timeout 600 python scripts/adaptive_timing.py 30 100 200 400 > gpurun_out/adapt_kd$kd.log 2>&1; echo kd=$kd rc=$?
  cat gpurun_out/adapt_kd$kd.log | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['m'], d['k'], d['checkpoints'], round(d['iter_ms'],1), round(d['large_ms'],1), d['center_max'])"
done
