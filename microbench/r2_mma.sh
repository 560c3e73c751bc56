#!/bin/bash
TAG=${1:-r2m}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_r2_paths_gpu.py -m gpu -x -q -k "tensor_core" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -30 gpurun_out/${TAG}_pytest.log
if grep -q "rc=0" gpurun_out/${TAG}_pytest.log; then
  timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_all.log
  tail -3 gpurun_out/${TAG}_pytest_all.log
  timeout 300 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_C4.json 2> gpurun_out/${TAG}_bench_C4.err
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:k_perm_mma --log-file gpurun_out/${TAG}_mma_ncu.csv python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
fi
