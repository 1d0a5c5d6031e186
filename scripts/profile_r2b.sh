#!/bin/bash
# Round-2 (second session) profiles under gpurun: every bench line (final_bench.sh), the ncu launch list of one
# P100 adaptive run, ncu --set full summaries of the device eigen-solve (tridc_kernel, P100 at k = 544) and of the
# persistent multi-step Lanczos kernel (P100, fixed k = 64), and the 10^9 paper-model adaptive run traced per step.
tag=${1:-r02b}
bash scripts/final_bench.sh $tag
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_p100.csv \
    python scripts/tridc_timing.py child adaptive 100 0 > /dev/null 2>&1; echo launches=$?
python scripts/launch_summary.py gpurun_out/${tag}_launches_p100.csv > gpurun_out/${tag}_launches_p100_summary.txt
for K in tridc:544 multistep:64; do
  name=${K%%:*}; k=${K##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${name} -s 1 -c 1 -o gpurun_out/prof_${tag}_${name} \
      python scripts/tridc_timing.py child fixed 100 $k > /dev/null 2>&1; echo ncu_$name=$?
  python scripts/ncu_summary.py gpurun_out/prof_${tag}_${name}.ncu-rep > gpurun_out/${tag}_ncu_full_${name}.txt 2>&1
  python scripts/ncu_lines.py gpurun_out/prof_${tag}_${name}.ncu-rep 30 >> gpurun_out/${tag}_ncu_full_${name}.txt 2>&1
  rm -f gpurun_out/prof_${tag}_${name}.ncu-rep
done
KR_TRIDC_PROF=1 timeout 120 python scripts/tridc_timing.py child fixed 100 544 > gpurun_out/${tag}_tridc_phases.txt 2>&1
KR_LARGE_PROF=1 timeout 120 python scripts/tridc_timing.py child adaptive 100 0 > gpurun_out/${tag}_p100_evals.txt 2>&1
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/${tag}_p1000_smi.csv &
SMI=$!
KR_MAX_EV=8000 KR_STEP_TRACE=gpurun_out/${tag}_p1000_steps.txt timeout 900 python scripts/adaptive_timing.py 1000 > gpurun_out/${tag}_p1000.log 2>&1; echo p1000=$?
kill $SMI
python scripts/trace_summary.py gpurun_out/${tag}_p1000_steps.txt 1000000000 > gpurun_out/${tag}_p1000_trace_summary.txt
rm -f gpurun_out/${tag}_p1000_steps.txt
