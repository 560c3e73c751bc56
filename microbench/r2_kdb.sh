#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2kdb_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2kdb_pytest.log
tail -3 gpurun_out/r2kdb_pytest.log
python microbench/quick_time.py C3 10 2>&1
python microbench/kd_time.py C3 5 auto 1 2 2>&1
python microbench/kd_threshold.py 5,6,8 20000,30000,40000,60000 2>&1
