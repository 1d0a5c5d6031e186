#!/bin/bash
# Round-2 GPU cycle: GPU tests, headline bench (C5 + dense companion C5D), ncu full capture of the step kernel
# on dense data (C5D) and the launch list of one C5 step. Usage (under gpurun): bash scripts/cycle_r2.sh tag [notest]
tag=${1:-x}
if [ "$2" != "notest" ]; then
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -x > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_$tag.log
fi
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5_$tag.log 2>&1; echo bench=$?
D="python bench.py --config C5D --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$D > gpurun_out/plain_c5d_$tag.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:lz_step_kernel -s 20 -c 1 -o gpurun_out/prof_c5d_$tag $D > gpurun_out/ncu_full_$tag.log 2>&1; echo ncu=$?
L="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_$tag.csv $L > /dev/null 2>&1; echo launches=$?
