KR_STEP_V=2 timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py tests/test_gpu_next2.py tests/test_gpu_next4.py -m gpu -q --timeout 900 -p no:cacheprovider -k "dirs_heat or config2 or config1 or oscillator or edge or transpose or heater or next4 or dense_rand" > gpurun_out/pytest_spmm.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_spmm.log
for e in "" "KR_SPMM_PER_DIR=1"; do env $e timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2_$e.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/c2_$e.log') if l.startswith('{')][-1]); print('C2 $e', round(d['value']), 'steps/s', round(d['ms_per_step'],3), 'ms', d['roofline']['frac'])"; done
L="python bench.py --config P100 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
KR_STEP_V=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_p100.csv $L > /dev/null 2>&1; echo ncu=$?
python scripts/launch_summary.py gpurun_out/launches_p100.csv > gpurun_out/launches_p100_summary.txt; head -20 gpurun_out/launches_p100_summary.txt
L2="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $L2 > /dev/null 2>&1; echo ncu2=$?
python scripts/launch_summary.py gpurun_out/launches_c2.csv > gpurun_out/launches_c2_summary.txt; head -12 gpurun_out/launches_c2_summary.txt
