#!/bin/bash
# profiling-probe overhead: old (per-warp tail atomics) vs new (one per CTA, clock probe sampled) library
mkdir -p gpurun_out
cp paper_2106_13706_b200/libddks.so /tmp/new.so
timeout 300 python microbench/prof_overhead.py C1 C2 C3 C4 > gpurun_out/profov_new.txt 2>&1
cp tmp_old/libddks.so paper_2106_13706_b200/libddks.so
timeout 300 python microbench/prof_overhead.py C1 C2 C3 C4 > gpurun_out/profov_old.txt 2>&1
cp /tmp/new.so paper_2106_13706_b200/libddks.so
timeout 300 python microbench/prof_overhead.py C1 C2 C3 C4 >> gpurun_out/profov_new.txt 2>&1
for w in C1 C2 C3; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/profov_bench_$w.json 2>/dev/null
done
cat gpurun_out/profov_*.txt
