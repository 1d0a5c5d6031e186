#!/bin/bash
# NEXT-1 bench lines (the paper's heat model, adaptive k) + the default C5 line + GPU tests.
[ -n "$2" ] || timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu_$1.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_$1.log
[ -n "$2" ] || timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5_$1.log 2>&1; echo c5=$?
timeout 600 python bench.py --config P100 --steps 5 --warmup 3 > gpurun_out/bench_p100_$1.log 2>&1; echo p100=$?
timeout 900 python bench.py --config P1000 --steps 1 --warmup 3 --no-e2e > gpurun_out/bench_p1000_$1.log 2>&1; echo p1000=$?
