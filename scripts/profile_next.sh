#!/bin/bash
python scripts/profile_next.py cgs > gpurun_out/pn_cgs.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:"cgs_(dots|update)_kernel" -s 1000 -c 2 -o gpurun_out/prof_cgs python scripts/profile_next.py cgs > gpurun_out/ncu_cgs.log 2>&1; echo cgs=$?
python scripts/profile_next.py gemm > gpurun_out/pn_gemm.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:"gemm_band_kernel|large_chain" -s 26 -c 2 -o gpurun_out/prof_gemm python scripts/profile_next.py gemm > gpurun_out/ncu_gemm.log 2>&1; echo gemm=$?
python scripts/profile_next.py lp > gpurun_out/pn_lp.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:"lp_step_kernel" -c 1 -o gpurun_out/prof_lp python scripts/profile_next.py lp > gpurun_out/ncu_lp.log 2>&1; echo lp=$?
cat gpurun_out/pn_*.log
