#!/bin/bash
# A/B: the committed library vs a previous build (scratch_libs/libkr_old.so), alternating, C5 recipe
for r in 1 2; do
  python scripts/vslab_timing.py 1000 1 | sed 's/^/new /'
  KR_LIB_PATH=scratch_libs/libkr_old.so python scripts/vslab_timing.py 1000 1 | sed 's/^/old /'
done
