#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -1
for lib in new old; do
  if [ $lib = old ]; then export KR_LIB_PATH=scratch_libs/libkr_old.so; else unset KR_LIB_PATH; fi
  for c in C5 C3 P100; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$lib $c\", round(d[\"value\"],2), round(d[\"ms_per_step\"],3))"; done
done
