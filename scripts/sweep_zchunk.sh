#!/bin/bash
# z-chunk sweep of the fused step kernel (KR_ZCHUNK; default: the wave-efficiency model in kr_api.cu):
# per-step times of C5 (step 1 = compact u_1, no HBM reads) and C4. Usage (under gpurun): bash scripts/sweep_zchunk.sh
for zc in default 24 36 48 60 72 96 125; do
  e=""; [ "$zc" != default ] && e="KR_ZCHUNK=$zc"
  for cfg in C5 C4; do
    echo "zc=$zc $cfg: $(env $e python scripts/step_profile.py $cfg | cut -d: -f2)"
  done
done
