#!/bin/bash
# Bench lines for profiles/: headline C5 (with the oracle baseline) and the NEXT workloads.
tag=${1:-final}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5_$tag.log 2>&1; echo c5=$?
timeout 600 python bench.py --config P100 --steps 5 --warmup 3 > gpurun_out/bench_p100_$tag.log 2>&1; echo p100=$?
timeout 900 python bench.py --config H100 --steps 3 --warmup 3 > gpurun_out/bench_h100_$tag.log 2>&1; echo h100=$?
timeout 600 python bench.py --config C2T --steps 5 --warmup 3 > gpurun_out/bench_c2t_$tag.log 2>&1; echo c2t=$?
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 > gpurun_out/bench_c2_$tag.log 2>&1; echo c2=$?
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$tag.log 2>&1; echo c3=$?
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_$tag.log 2>&1; echo c4=$?
timeout 1200 python bench.py --config P1000 --steps 1 --warmup 3 --no-e2e > gpurun_out/bench_p1000_$tag.log 2>&1; echo p1000=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo ref=$?
L="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$L > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_$tag.csv $L > /dev/null 2>&1; echo launches=$?
