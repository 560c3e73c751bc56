#!/bin/bash
TAG=${1:-r2c5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "kd or x0 or fuzz or c5 or r2_paths or shard" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --workload C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_C5.json 2> gpurun_out/${TAG}_bench_C5.err
tail -2 gpurun_out/${TAG}_pytest.log
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench_C5.json').read().strip().splitlines()[-1]); r=d['roofline']; print('C5', d['ms_per_step'], r['frac'], r.get('executed_frac'), r.get('executed',{}).get('compares_per_pair'), d['result'])"
