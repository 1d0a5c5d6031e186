#!/bin/bash
# A/B (diagnostics): committed library (scratch_libs/libkr_old.so) vs working tree, sparse C5 + dense start
for r in 1 2; do
  python scripts/vslab_timing.py 1000 1 | sed 's/^/new /'
  KR_LIB_PATH=scratch_libs/libkr_old.so python scripts/vslab_timing.py 1000 1 | sed 's/^/old /'
  python scripts/kernel_probe2.py 1000 40 | sed 's/^/new /'
  KR_LIB_PATH=scratch_libs/libkr_old.so python scripts/kernel_probe2.py 1000 40 | sed 's/^/old /'
done
