#!/bin/bash
# Tile / z-chunk sweep of the fused step on C5 (and C4). Prints config and fused-step GB/s.
for cfg in C5 C4; do
for tile in 64x16 64x8 32x8; do
  for zc in auto; do
    if [ "$zc" = auto ]; then unset KR_ZCHUNK; else export KR_ZCHUNK=$zc; fi
    r=$(KR_TILE=$tile timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
    echo "$cfg tile=$tile zc=$zc $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), "steps/s", round(d["fused_step"]["gbs"],1), "GB/s", round(d["fused_step"]["pct_of_peak"],1), "%")' 2>/dev/null || echo "$r" | tail -2)"
  done
done
done
