#!/bin/bash
# Bench lines for profiles/ (under gpurun): the headline C5 (with the dense companion, e2e and the full-size oracle
# baseline), the other workloads as context lines, the reference arm on a short run.
tag=${1:-r02}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c2.log 2>&1; echo c2=$?
timeout 600 python bench.py --config C2T --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c2t.log 2>&1; echo c2t=$?
timeout 600 python bench.py --config P100 --steps 5 --warmup 3 > gpurun_out/${tag}_bench_p100.log 2>&1; echo p100=$?
timeout 900 python bench.py --config H100 --steps 3 --warmup 3 > gpurun_out/${tag}_bench_h100.log 2>&1; echo h100=$?
timeout 1200 python bench.py --config P1000 --steps 1 --warmup 3 --no-e2e > gpurun_out/${tag}_bench_p1000.log 2>&1; echo p1000=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_reference.log 2>&1; echo ref=$?
for f in gpurun_out/${tag}_bench_*.log; do grep '^{' $f | tail -1 > ${f%.log}.jsonl; done
