for W in 296 0; do
  D="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense"
  KR_WIN=$W timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:lz_step_kernel -s 20 -c 3 $D 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/win=$W /"
done
