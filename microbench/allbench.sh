set -x
mkdir -p gpurun_out
out=gpurun_out/r1_bench_methods_v8.jsonl
: > $out
for w in C1 C2 C3 C4; do python bench.py --workload $w --steps 20 --warmup 5 --cpu-seconds 10 2>>gpurun_out/allbench.err | tail -1 >> $out; done
python bench.py --workload C5 --steps 3 --warmup 3 --cpu-seconds 15 2>>gpurun_out/allbench.err | tail -1 >> $out
python bench.py --method significance --workload C3 --steps 10 --warmup 3 --cpu-seconds 10 2>>gpurun_out/allbench.err | tail -1 >> $out
python bench.py --method significance --workload C5 --steps 3 --warmup 3 --cpu-seconds 10 2>>gpurun_out/allbench.err | tail -1 >> $out
python bench.py --method vdks --workload C5 --steps 20 --warmup 5 --cpu-seconds 10 2>>gpurun_out/allbench.err | tail -1 >> $out
python bench.py --method rdks --workload C5 --steps 20 --warmup 5 --cpu-seconds 10 2>>gpurun_out/allbench.err | tail -1 >> $out
python bench.py --impl reference --steps 2 --warmup 3 2>>gpurun_out/allbench.err | tail -1 >> $out
for m in vdks rdks; do ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_${m}_v8.csv python bench.py --method $m --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; done
wc -l $out
