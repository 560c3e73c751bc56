#!/bin/bash
# round-2 baseline: step breakdown of C1/C2/C3 (launch lists), ncu per-opcode availability on the C2 count kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for w in C1 C2 C3; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_$w.json 2> gpurun_out/r2b_bench_$w.err
done
for w in C1 C2 C3; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_$w.csv \
     python microbench/quick_time.py $w 3 > gpurun_out/r2b_ncu_$w.log 2>&1
done
timeout 300 ncu --metrics sass__inst_executed_per_opcode,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,smsp__sass_inst_executed_op_shared_atom.sum --clock-control none -k regex:k_count -c 1 --csv --log-file gpurun_out/r2b_opcode_c2.csv python profiles/profile_run.py C2 > gpurun_out/r2b_opc.log 2>&1
ls -la gpurun_out | tail -20
