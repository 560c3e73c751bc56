#!/bin/bash
# ncu --set full of vdKS/rdKS minmax and the voxel histogram (C5)
mkdir -p gpurun_out
TAG=${1:-vg}
O=gpurun_out
timeout 300 python microbench/approx_c5.py 20 > $O/${TAG}_time.txt 2>&1
for kn in k_minmax_vec k_vox_hist_vec k_vox_prefix_slab; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kn -c 1 -o $O/${TAG}_$kn python microbench/approx_c5.py 1 vdks > /dev/null 2>&1
  ncu -i $O/${TAG}_$kn.ncu-rep --page raw --csv > $O/${TAG}_${kn}_raw.csv 2>/dev/null
  ncu -i $O/${TAG}_$kn.ncu-rep --page source --csv 2>/dev/null | gzip > $O/${TAG}_${kn}_source.csv.gz
  rm -f $O/${TAG}_$kn.ncu-rep
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv \
  --log-file $O/${TAG}_vdks_warm.csv python microbench/approx_c5.py 2 vdks > /dev/null 2>&1
cat $O/${TAG}_time.txt
