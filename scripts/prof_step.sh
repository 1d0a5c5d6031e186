#!/bin/bash
# ncu --set full of one step-kernel launch (launch 20 of the run) for the given config;
# the summary (scripts/ncu_summary.py) is written on the box, the report kept only with KEEP=1 (gpurun_out <= 64 MiB).
# Usage (under gpurun): bash scripts/prof_step.sh tag cfg
tag=$1; cfg=$2
D="python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense"
$D > gpurun_out/plain_${tag}.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:lz_step_kernel -s 20 -c 1 -o gpurun_out/prof_${tag} $D > gpurun_out/ncu_${tag}.log 2>&1; echo ncu_$tag=$?
python scripts/ncu_summary.py gpurun_out/prof_${tag}.ncu-rep > gpurun_out/ncu_${tag}_summary.txt 2>&1
[ "$KEEP" = "1" ] || rm -f gpurun_out/prof_${tag}.ncu-rep
