#!/bin/bash
# Tile A/B (diagnostics): parity with the 64x32 / 512-thread tile, then C5 + dense-start timings per tile.
KR_TILE=64x32 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "stencil or virtual or config3 or config4 or config5 or determin" --timeout 600 -p no:cacheprovider 2>&1 | tail -1
KR_TILE=64x32 timeout 600 python -m pytest tests/test_gpu_next1.py -q -k "boundaries or adaptive_paper" --timeout 600 -p no:cacheprovider 2>&1 | tail -1
for t in 64x16 64x32 64x16 64x32; do
  echo "tile $t"; KR_TILE=$t python scripts/vslab_timing.py 1000 1; KR_TILE=$t python scripts/kernel_probe2.py 1000 40 2>&1 | grep -v "^$"
done
