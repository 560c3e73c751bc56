#!/bin/bash
TAG=${1:-r2c4}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "perm or c4" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_C4.json 2> gpurun_out/${TAG}_bench_C4.err
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active --clock-control none --csv -k regex:k_perm_count --log-file gpurun_out/${TAG}_perm_ncu.csv python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
