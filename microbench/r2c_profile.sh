#!/bin/bash
# Round-2 second session, refresh after the fused mid-N kd ordering, the rdKS compaction geometry and the chunked H2D
# of host-input batches: GPU tests, bench lines of the changed configs / methods, launch lists, ncu captures.
TAG=${1:-r2c}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
for w in C1 C2 C3 C4; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 >> $O/${TAG}_bench_configs.jsonl 2>> $O/${TAG}_bench_configs.err
done
timeout 600 python bench.py --workload C3 --method significance --steps 10 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
timeout 600 python bench.py --workload C5 --method vdks --steps 20 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
timeout 600 python bench.py --workload C5 --method rdks --steps 20 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
for w in C3 C4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_$w.csv \
     python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_rdks.csv \
   python bench.py --workload C5 --method rdks --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cap() {  # cap NAME KERNEL_REGEX CMD...
  local name=$1 kre=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -o $O/${TAG}_full_$name "$@" > /dev/null 2>&1
  if [ -f $O/${TAG}_full_$name.ncu-rep ]; then
    ncu -i $O/${TAG}_full_$name.ncu-rep --page raw --csv > $O/${TAG}_full_${name}_raw.csv 2>/dev/null
    rm -f $O/${TAG}_full_$name.ncu-rep
  fi
}
cap kdbfused k_kdb_fused python profiles/profile_run.py C3
cap rdkscompact k_rdb_compact python microbench/approx_c5.py 1 rdks
timeout 300 python microbench/graph_ab.py 30 > $O/${TAG}_graph_ab.txt 2>&1
timeout 300 python microbench/c4_parts.py > $O/${TAG}_c4_parts.txt 2>&1
du -sh $O; tail -2 $O/${TAG}_pytest_gpu.log; tail -1 $O/${TAG}_smoke.log
