#!/bin/bash
# k_perm_count d=4 CTA-size sweep (C4b); each build variant compiled here on the box
mkdir -p gpurun_out
for T in 64 128 256; do
  DDKS_NVCC_EXTRA="-DDDKS_P4T=$T" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_perm_count --log-file gpurun_out/r2p_T$T.csv python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "T=$T $(grep k_perm_count gpurun_out/r2p_T$T.csv | awk -F'","' '{print $15}' | tr -d '"' | tr '\n' ' ')"
done
