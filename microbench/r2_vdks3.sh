#!/bin/bash
# vdKS hash-aggregated histogram A/B (DDKS_VDKS_NOHASH = the per-point RED kernel)
mkdir -p gpurun_out
TAG=${1:-vh}
timeout 600 python -m pytest tests/test_approx_gpu.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python microbench/approx_c5.py 20 vdks > gpurun_out/${TAG}_time.txt 2>&1
DDKS_VDKS_NOHASH=1 timeout 300 python microbench/approx_c5.py 20 vdks >> gpurun_out/${TAG}_time.txt 2>&1
timeout 300 python microbench/approx_c5.py 20 vdks >> gpurun_out/${TAG}_time.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv \
  --log-file gpurun_out/${TAG}_vdks_warm.csv python microbench/approx_c5.py 2 vdks > /dev/null 2>&1
tail -2 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_time.txt
