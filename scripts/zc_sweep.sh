#!/bin/bash
# z-chunk sweep of the C5 / C4 step kernel (under gpurun). Usage: bash scripts/zc_sweep.sh "40 59 80" [cfgs]
for zc in $1; do for cfg in ${2:-C5}; do echo "zc=$zc $cfg: $(KR_ZCHUNK=$zc python scripts/step_profile.py $cfg | cut -d: -f2)"; done; done
