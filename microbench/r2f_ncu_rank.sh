#!/bin/bash
# ncu --set full capture of the rank-lane count on one config (default C2): raw page -> gpurun_out/<tag>_full_rank_<cfg>_raw.csv
CFG=${1:-C2}; TAG=${2:-r2f}; O=gpurun_out; mkdir -p $O
timeout 300 python microbench/rank_one.py $CFG > $O/${TAG}_rank_one_$CFG.txt 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count_rank -s 1 -c 1 -o $O/${TAG}_full_rank_$CFG \
   python microbench/rank_one.py $CFG > /dev/null 2>&1
ncu -i $O/${TAG}_full_rank_$CFG.ncu-rep --page raw --csv > $O/${TAG}_full_rank_${CFG}_raw.csv 2>/dev/null
ncu -i $O/${TAG}_full_rank_$CFG.ncu-rep --page source --csv > $O/${TAG}_full_rank_${CFG}_source.csv 2>/dev/null
rm -f $O/${TAG}_full_rank_$CFG.ncu-rep
python profiles/ncu_summary.py $O/${TAG}_full_rank_${CFG}_raw.csv
