#!/bin/bash
# A/B of library builds (LIBS) on the virtual-slab C5 recipe (the z-slab code path of the multi-GPU run).
for rep in 1 2; do
for lib in ${LIBS:-cur}; do
  export KR_LIB_PATH=scratch_libs/libkr_$lib.so
  echo -n "$lib "; python scripts/vslab_timing.py 1000 ${SLABS:-2 8} 2>&1 | tr '\n' ' '; echo
done
done
