#!/bin/bash
# ncu full captures of a late (dense-data) fused step launch, Dirichlet and general-BC variants, m=400.
for kind in dir bc; do
  timeout 300 python scripts/dense_probe.py $kind 400 1200 > gpurun_out/dense_$kind.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lz_step_kernel -s 1100 -c 1 \
     -o gpurun_out/prof_dense_$kind python scripts/dense_probe.py $kind 400 1200 > gpurun_out/ncu_dense_$kind.log 2>&1
  echo $kind=$?
done
KR_MAX_EV=8000 KR_STEP_TRACE=gpurun_out/p1000b_steps.txt timeout 900 python scripts/adaptive_timing.py 1000 > gpurun_out/p1000b.log 2>&1; echo p1000=$?
cat gpurun_out/dense_*.log gpurun_out/p1000b.log
