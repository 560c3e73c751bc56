#!/bin/bash
# ncu --set full of the vdKS slab-path kernels (C5, k = 16), exported to raw CSV
mkdir -p gpurun_out
TAG=${1:-vf}
O=gpurun_out
for kn in k_vox_ids k_vox_scatter k_vox_slab k_vox_orthants k_vox_outer; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -c 1 -o $O/${TAG}_$kn python microbench/approx_c5.py 1 vdks > /dev/null 2>&1
  ncu -i $O/${TAG}_$kn.ncu-rep --page raw --csv > $O/${TAG}_${kn}_raw.csv 2>/dev/null
  ncu -i $O/${TAG}_$kn.ncu-rep --page source --csv 2>/dev/null | gzip > $O/${TAG}_${kn}_source.csv.gz
  rm -f $O/${TAG}_$kn.ncu-rep
done
ls -la $O | grep $TAG
