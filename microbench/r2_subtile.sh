#!/bin/bash
mkdir -p gpurun_out
for V in "-DDDKS_KD_SUBTILE=1" "-DDDKS_KD_SUBTILE=0"; do
  DDKS_NVCC_EXTRA="$V" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1
  echo "== variant [$V]"
  python microbench/kd_time.py C5 2 auto 2>&1 | tail -1
  python microbench/quick_time.py C3 10 2>&1 | head -1
  python microbench/kd_threshold.py 3,6 20000,40000 2>&1
done
DDKS_NVCC_EXTRA="-DDDKS_KD_SUBTILE=1" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "kd or x0 or fuzz or c5 or shard or significance" 2>&1 | tail -2
