#!/bin/bash
mkdir -p gpurun_out
for V in "" "-DDDKS_S5R=2 -DDDKS_S5T=512" "-DDDKS_S5R=2 -DDDKS_S5T=768" "-DDDKS_S5R=4 -DDDKS_S5T=256"; do
  DDKS_NVCC_EXTRA="$V" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1 || { echo "build failed [$V]"; continue; }
  echo "== variant [$V]"
  python bench.py --workload C5 --method significance --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('significance C5 ms/step', round(d['ms_per_step'],2), 'count ms', round(d['roofline']['kernel_ms_per_launch'],2))"
done
