#!/bin/bash
# Round-2 profiles (under gpurun): headline bench line, ncu launch list of one C5 bench step, ncu --set full
# summaries of the step kernel on C5 and C5D, the 10^9 paper-model adaptive run traced per step with clocks.
tag=${1:-r02}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c5.log 2>&1; echo bench=$?
L="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_c5.csv $L > /dev/null 2>&1; echo launches=$?
python scripts/launch_summary.py gpurun_out/${tag}_launches_c5.csv > gpurun_out/${tag}_launches_c5_summary.txt
bash scripts/prof_step.sh ${tag}_c5 C5
bash scripts/prof_step.sh ${tag}_c5d C5D
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/${tag}_p1000_smi.csv &
SMI=$!
KR_MAX_EV=8000 KR_STEP_TRACE=gpurun_out/${tag}_p1000_steps.txt timeout 900 python scripts/adaptive_timing.py 1000 > gpurun_out/${tag}_p1000.log 2>&1; echo p1000=$?
kill $SMI
python scripts/trace_summary.py gpurun_out/${tag}_p1000_steps.txt 1000000000 > gpurun_out/${tag}_p1000_trace_summary.txt
cat gpurun_out/${tag}_p1000.log gpurun_out/${tag}_p1000_trace_summary.txt
