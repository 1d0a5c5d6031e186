#!/bin/bash
timeout 600 python scripts/kernel_probe.py 400 1000; timeout 600 python scripts/kernel_probe.py 1000 700
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next1.py tests/test_gpu_next2.py -q --timeout 600 -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --config C2T --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2t_o.log 2>&1; echo c2t=$?
timeout 600 python bench.py --config P100 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p100_o.log 2>&1; echo p100=$?
for c in c2t p100; do tail -1 gpurun_out/bench_${c}_o.log | cut -c1-600; done
