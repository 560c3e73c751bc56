#!/bin/bash
# mbarrier suspend-time hint A/B: C5 (kd count), C3 / C2 (position-ordered counts)
mkdir -p gpurun_out
for H in 0 20000 1000000; do
  DDKS_NVCC_EXTRA="-DDDKS_MBAR_HINT_NS=$H" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1
  echo "== hint $H"
  python microbench/kd_time.py C5 2 auto 2>&1 | tail -1
  python microbench/quick_time.py C3 5 2>&1 | head -1
  python microbench/quick_time.py C2 10 2>&1 | head -1
done
