#!/bin/bash
# C5 kd count geometry A/B under the one-dim path: R origins per thread x T threads (same 3072 origins / CTA), tiles
mkdir -p gpurun_out
for V in "-DDDKS_C5R=4 -DDDKS_C5T=512 -DDDKS_C5TILE=256 -DDDKS_C5S=3" "-DDDKS_C5R=4 -DDDKS_C5T=256 -DDDKS_C5TILE=256 -DDDKS_C5S=3" "-DDDKS_C5R=4 -DDDKS_C5T=384 -DDDKS_C5TILE=256 -DDDKS_C5S=3" "-DDDKS_C5R=6 -DDDKS_C5T=384 -DDDKS_C5TILE=256 -DDDKS_C5S=3" "-DDDKS_C5R=8 -DDDKS_C5T=256 -DDDKS_C5TILE=256 -DDDKS_C5S=3" "-DDDKS_C5R=4 -DDDKS_C5T=512 -DDDKS_C5TILE=256 -DDDKS_C5S=4"; do
  DDKS_NVCC_EXTRA="$V" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1 || { echo "build failed [$V]"; continue; }
  echo "== variant [$V]"
  python microbench/kd_time.py C5 2 auto 2>&1 | tail -1
done
