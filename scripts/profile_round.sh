#!/bin/bash
# Round profiling bundle (one GPU, under gpurun): bench line, reference arm, ncu launch list (C5),
# DRAM traffic of the C5 step kernel, and a full ncu capture of the step kernel on C4.
tag=${1:-r01}
B="python bench.py --steps 5 --warmup 3"
timeout 900 $B > gpurun_out/bench_$tag.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo ref=$?
L="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$L > gpurun_out/plain_l_$tag.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_$tag.csv $L > gpurun_out/ncu_launch_$tag.log 2>&1; echo launches=$?
$L > gpurun_out/plain_t_$tag.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:lz_step_kernel -s 10 -c 2 --csv --log-file gpurun_out/traffic_c5_$tag.csv $L > gpurun_out/ncu_traffic_$tag.log 2>&1; echo traffic=$?
C4="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$C4 > gpurun_out/plain_c4_$tag.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:lz_step_kernel -s 12 -c 1 -o gpurun_out/prof_c4_$tag $C4 > gpurun_out/ncu_full_$tag.log 2>&1; echo full=$?
