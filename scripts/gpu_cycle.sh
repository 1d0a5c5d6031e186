#!/bin/bash
# One GPU round trip: parity tests, bench (C5), and an ncu capture of the step kernel on C4.
# Usage (under gpurun): bash scripts/gpu_cycle.sh [tag]
tag=${1:-x}
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$tag.log 2>&1; echo bench=$?
CMD2="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD2 > gpurun_out/plain_c4_$tag.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:lz_step_kernel -s 12 -c 1 -o gpurun_out/prof_c4_$tag $CMD2 > gpurun_out/ncu_full_$tag.log 2>&1; echo ncu=$?
