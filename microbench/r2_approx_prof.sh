#!/bin/bash
# vdKS / rdKS at C5: live per-call time and warm-cache per-kernel durations (ncu --cache-control none)
mkdir -p gpurun_out
TAG=${1:-ap}
timeout 300 python microbench/approx_c5.py 20 > gpurun_out/${TAG}_time.txt 2>&1
for m in vdks rdks; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv \
  --log-file gpurun_out/${TAG}_${m}_warm.csv python microbench/approx_c5.py 2 $m > /dev/null 2>&1
done
cat gpurun_out/${TAG}_time.txt
