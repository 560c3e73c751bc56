#!/bin/bash
# Final refresh (round 2, second session): the cluster mid-N ordering and the rdKS bucket count -- GPU tests, smoke,
# bench lines of C1-C4 / significance C3 / vdKS / rdKS, launch lists of C3 and rdKS, ncu capture of k_kdb_cluster.
TAG=${1:-r2d}
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
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_C3.csv \
   python bench.py --workload C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_rdks.csv \
   python bench.py --workload C5 --method rdks --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kdb_cluster -c 1 -o $O/${TAG}_full_kdbcluster \
   python profiles/profile_run.py C3 > /dev/null 2>&1
ncu -i $O/${TAG}_full_kdbcluster.ncu-rep --page raw --csv > $O/${TAG}_full_kdbcluster_raw.csv 2>/dev/null; rm -f $O/${TAG}_full_kdbcluster.ncu-rep
timeout 300 python microbench/graph_ab.py 30 > $O/${TAG}_graph_ab.txt 2>&1
du -sh $O; tail -2 $O/${TAG}_pytest_gpu.log; tail -1 $O/${TAG}_smoke.log
