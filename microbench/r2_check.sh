#!/bin/bash
# round-2 check: GPU tests, smoke, short bench lines for every config (device + e2e), launch list for C1/C2/C3
mkdir -p gpurun_out
TAG=${1:-r2}
nproc > gpurun_out/${TAG}_nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
for w in C1 C2 C3 C4; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
done
timeout 600 python bench.py --workload C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_C5.json 2> gpurun_out/${TAG}_bench_C5.err
for w in C1 C2 C3; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_$w.csv \
     python microbench/quick_time.py $w 3 > /dev/null 2>&1
done
tail -3 gpurun_out/${TAG}_pytest_gpu.log
