#!/bin/bash
# Bench lines for every config, the reference arm, the C5 launch list, the C5 step-kernel DRAM traffic and a
# full ncu capture of the step kernel on C4. Usage (under gpurun): bash scripts/refresh_profiles.sh <tag>
tag=${1:-x}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5_$tag.log 2>&1; echo c5=$?
for c in C3 C4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${c,,}_$tag.log 2>&1; echo $c=$?; done
for c in P100 C2 C2T; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${c,,}_$tag.log 2>&1; echo $c=$?; done
timeout 900 python bench.py --config H100 --steps 3 --warmup 3 > gpurun_out/bench_h100_$tag.log 2>&1; echo h100=$?
timeout 1200 python bench.py --config P1000 --steps 1 --warmup 3 --no-e2e > gpurun_out/bench_p1000_$tag.log 2>&1; echo p1000=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo ref=$?
L="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$L > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_$tag.csv $L > /dev/null 2>&1; echo launches=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:lz_step_kernel -s 10 -c 2 --csv --log-file gpurun_out/traffic_c5_$tag.csv $L > /dev/null 2>&1; echo traffic=$?
C4="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lz_step_kernel -s 12 -c 1 -o gpurun_out/prof_c4_$tag $C4 > /dev/null 2>&1; echo full=$?
