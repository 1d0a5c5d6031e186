#!/bin/bash
# A/B of the in-tree library against scratch_libs/libkr_old.so: per-step device times (C5, C4), alternating.
for rep in 1 2; do
for lib in new old; do
  if [ $lib = old ]; then export KR_LIB_PATH=scratch_libs/libkr_old.so; else unset KR_LIB_PATH; fi
  for c in ${CONFIGS:-C5 C4}; do
    python scripts/step_times.py $c 3 2>&1 | python -c "
import sys
L=sys.stdin.read().splitlines(); it=L[0].split()[-1]; v=[float(x) for x in L[1].split(':')[1].split()]
mid=v[2:-1]; print('$lib $c iter', it, 'step1 %.3f step2 %.3f mean3..k-1 %.4f' % (v[0], v[1], sum(mid)/len(mid)))"
  done
done
done
