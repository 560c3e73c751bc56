#!/bin/bash
# Evidence pass on the code with the rank-lane count (round 2, last session): GPU tests, smoke, the default bench line
# (C5), C1-C4, significance C3 / vdKS / rdKS, launch lists of the default bench command and of C3, graph A/B.
TAG=${1:-r2f}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench_c5_default.json 2> $O/${TAG}_bench_c5_default.err
for w in C1 C2 C3 C4; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 >> $O/${TAG}_bench_configs.jsonl 2>> $O/${TAG}_bench_configs.err
done
timeout 600 python bench.py --workload C3 --method significance --steps 10 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
timeout 600 python bench.py --workload C5 --method vdks --steps 20 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
timeout 600 python bench.py --workload C5 --method rdks --steps 20 --warmup 3 >> $O/${TAG}_bench_methods.jsonl 2>> $O/${TAG}_bench_methods.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches_C5.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_C3.csv \
   python bench.py --workload C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 python microbench/graph_ab.py 30 > $O/${TAG}_graph_ab.txt 2>&1
du -sh $O; tail -2 $O/${TAG}_pytest_gpu.log; tail -2 $O/${TAG}_smoke.log; cat $O/${TAG}_bench_c5_default.json | head -c 600
bash microbench/r2f_ncu_rank.sh C3 $TAG > $O/${TAG}_ncu_full_rank_c3.json 2>/dev/null
bash microbench/r2f_ncu_rank.sh C2 $TAG > $O/${TAG}_ncu_full_rank_c2.json 2>/dev/null
rm -f $O/${TAG}_full_rank_*_source.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_C2.csv \
   python bench.py --workload C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
