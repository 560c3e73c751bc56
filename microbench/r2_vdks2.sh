#!/bin/bash
# vdKS slab path: parity tests, live C5 time, warm per-kernel durations
mkdir -p gpurun_out
TAG=${1:-vd}
timeout 600 python -m pytest tests/test_approx_gpu.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python microbench/approx_c5.py 20 vdks > gpurun_out/${TAG}_time.txt 2>&1

timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv \
  --log-file gpurun_out/${TAG}_vdks_warm.csv python microbench/approx_c5.py 2 vdks > /dev/null 2>&1
tail -3 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_time.txt
