#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2c5b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c5b_pytest.log
tail -2 gpurun_out/r2c5b_pytest.log
python microbench/kd_time.py C5 2 auto 4,6,7,7 4,8,8,8 4,6,8,8 4,8,10,10 2>&1
python microbench/kd_threshold.py 5 15000,30000,60000 2>&1
python microbench/kd_time.py C5 1 auto 2>&1 | tail -1
