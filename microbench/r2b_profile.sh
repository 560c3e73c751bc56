#!/bin/bash
# Round-2 (second session) evidence pass: full GPU tests, smoke, bench lines (every config / method), ncu launch lists, ncu --set full
# captures of the dominant kernels, and the per-opcode instruction counts that check the in-kernel executed-compare
# counter. Usage: bash microbench/r2b_profile.sh TAG
TAG=${1:-r2b}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > $O/${TAG}_bench_default.json 2> $O/${TAG}_bench_default.err
for w in C1 C2 C3 C4; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 >> $O/${TAG}_bench_configs.jsonl 2>> $O/${TAG}_bench_configs.err
done
timeout 600 python bench.py --workload C3 --method significance --steps 10 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
timeout 600 python bench.py --workload C5 --method significance --steps 3 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
timeout 600 python bench.py --workload C5 --method vdks --steps 20 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
timeout 600 python bench.py --workload C5 --method rdks --steps 20 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
# launch lists (cold-cache, serialised; the kernel SHARE of the step is what must agree)
for w in C1 C2 C3 C4 C5; do
  st=2; [ $w = C5 ] && st=1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_$w.csv \
     python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
# full-set captures of the dominant kernels (subsets where the full launch is too long to replay); each report is
# exported to its raw-page CSV (+ a gzipped source page) and deleted: gpurun brings back at most 64 MiB
cap() {  # cap NAME KERNEL_REGEX CMD...
  local name=$1 kre=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -o $O/${TAG}_full_$name "$@" > /dev/null 2>&1
  if [ -f $O/${TAG}_full_$name.ncu-rep ]; then
    ncu -i $O/${TAG}_full_$name.ncu-rep --page raw --csv > $O/${TAG}_full_${name}_raw.csv 2>/dev/null
    ncu -i $O/${TAG}_full_$name.ncu-rep --page source --csv 2>/dev/null | gzip > $O/${TAG}_full_${name}_source.csv.gz
    rm -f $O/${TAG}_full_$name.ncu-rep
  fi
}
cap c5kd k_count python profiles/profile_run.py C5kd 200000
cap c3 k_count python profiles/profile_run.py C3
cap c2 k_count python profiles/profile_run.py C2
cap c4 k_count python profiles/profile_run.py C4
cap c4perm k_perm python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e
cap vdkshist k_vox_hist_vec python microbench/approx_c5.py 1 vdks
cap rdkskeys k_rd_keys_pt python microbench/approx_c5.py 1 rdks
cap rdkscompact k_rdb_compact python microbench/approx_c5.py 1 rdks
cap c4sorted k_pack_sorted python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e
cap vdksslab k_vox_prefix_slab python microbench/approx_c5.py 1 vdks
# DRAM traffic of the full-size C5 count launch and per-opcode counts for the executed-compare check
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum --clock-control none -k regex:k_count -s 3 -c 1 --csv --log-file $O/${TAG}_traffic_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for w in C2 C3 C4; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_count -c 1 --csv --log-file $O/${TAG}_traffic_$w.csv python profiles/profile_run.py $w > /dev/null 2>&1
done
timeout 900 ncu --metrics sass__inst_executed_per_opcode --print-metric-instances values --clock-control none -k regex:k_count -c 1 --csv --log-file $O/${TAG}_opcodes_c5kd.csv python profiles/profile_run.py C5kd 200000 > $O/${TAG}_opcodes_c5kd.log 2>&1
timeout 900 ncu --metrics sass__inst_executed_per_opcode --print-metric-instances values --clock-control none -k regex:k_count -c 1 --csv --log-file $O/${TAG}_opcodes_c3.csv python profiles/profile_run.py C3 > $O/${TAG}_opcodes_c3.log 2>&1
for m in vdks rdks; do
  timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
    --log-file $O/${TAG}_${m}_warm.csv python microbench/approx_c5.py 2 $m > /dev/null 2>&1
done
timeout 300 python microbench/graph_ab.py 30 > $O/${TAG}_graph_ab.txt 2>&1
timeout 300 python microbench/c4_parts.py > $O/${TAG}_c4_parts.txt 2>&1
./microbench/red_global > $O/${TAG}_red_global.txt 2>&1
du -sh $O; tail -2 $O/${TAG}_pytest_gpu.log; tail -1 $O/${TAG}_smoke.log
