#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_approx_gpu.py -m gpu -x -q > gpurun_out/r2vd_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2vd_pytest.log
tail -2 gpurun_out/r2vd_pytest.log
python bench.py --workload C5 --method vdks --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('vdks C5 ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))"
DDKS_VDKS_THREAD=1 python bench.py --workload C5 --method vdks --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('vdks (thread per voxel) C5 ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))"
ncu --metrics gpu__time_duration.sum --csv python bench.py --workload C5 --method vdks --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "k_vox|k_prefix|k_minmax" | awk -F'","' '{print $5, $NF}' | tail -8
