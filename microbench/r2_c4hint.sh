#!/bin/bash
mkdir -p gpurun_out
for H in 1000000 0; do
  DDKS_NVCC_EXTRA="-DDDKS_MBAR_HINT_NS=$H" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1
  echo "== hint $H"
  for i in 1 2; do python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('C4 ms/step', round(d['ms_per_step'],4), 'kern/launch', round(r['kernel_ms_per_launch'],4))"; done
done
