#!/bin/bash
# Per-step trace of the paper's 10^9-state adaptive run (diagnostics): step-kernel ms and step-to-step ms
# for all steps, with nvidia-smi clocks / power sampled alongside.
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/p1000_smi.csv &
SMI=$!
KR_MAX_EV=8000 KR_STEP_TRACE=gpurun_out/p1000_steps.txt timeout 900 python scripts/adaptive_timing.py 1000 > gpurun_out/p1000_t.log 2>&1
echo rc=$?
kill $SMI
cat gpurun_out/p1000_t.log
