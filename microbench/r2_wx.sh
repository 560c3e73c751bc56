#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_r2_paths_gpu.py -m gpu -x -q -k "mid_n" > gpurun_out/r2wx_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2wx_pytest.log
tail -3 gpurun_out/r2wx_pytest.log
if grep -q "rc=0" gpurun_out/r2wx_pytest.log; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2wx_pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2wx_pytest_all.log
  tail -2 gpurun_out/r2wx_pytest_all.log
  python microbench/quick_time.py C2 10 2>&1
  DDKS_NO_WX=1 python microbench/quick_time.py C2 10 2>&1 | head -1
  python microbench/kd_threshold.py 3,4 10000,20000,30000 2>&1
fi
