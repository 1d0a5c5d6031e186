#!/bin/bash
for kd in 3000 6000; do KR_KDOUBLE=$kd timeout 600 python scripts/adaptive_timing.py 1000 > gpurun_out/p1000_kd$kd.log 2>&1; echo kd=$kd; cat gpurun_out/p1000_kd$kd.log; done
python scripts/profile_next.py gemm > gpurun_out/pn_gemm2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"gemm_band_kernel" -s 26 -c 1 -o gpurun_out/prof_gemm2 python scripts/profile_next.py gemm > gpurun_out/ncu_gemm2.log 2>&1; echo ncu=$?
