#!/bin/bash
TAG=${1:-r2s}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
for w in C1 C2; do timeout 300 python microbench/host_overhead.py $w >> gpurun_out/${TAG}_host.log 2>&1; done
timeout 300 python microbench/graph_time.py C1 C2 >> gpurun_out/${TAG}_host.log 2>&1
for w in C1 C2 C3; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err
done
tail -2 gpurun_out/${TAG}_pytest_gpu.log; cat gpurun_out/${TAG}_host.log
