#!/bin/bash
# C5 kd count: loop-variant code size A/B (instruction-fetch stalls): unroll of the variants with undecided kd dims,
# and how many undecided dims get their own variant at K = 4
mkdir -p gpurun_out
for V in "" "-DDDKS_UNROLL_PARTIAL=4" "-DDDKS_UNROLL_PARTIAL=2" "-DDDKS_KD_OPEN4=3" "-DDDKS_KD_OPEN4=2" "-DDDKS_UNROLL_PARTIAL=4 -DDDKS_KD_OPEN4=3"; do
  DDKS_NVCC_EXTRA="$V" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1
  echo "== variant [$V]"
  python microbench/kd_time.py C5 2 auto 2>&1 | tail -1
done
