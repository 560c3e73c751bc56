# perm_mma stage variants: parity (tensor-core null tests) and C4 null timing per variant
cp paper_2106_13706_b200/libddks.so /tmp/o.so
for v in s3 s2; do
  cp variants/pm_$v.so paper_2106_13706_b200/libddks.so; echo "== $v"
  timeout 300 python -m pytest tests/test_r2_paths_gpu.py -x -q -k "tensor_core or groups" 2>&1 | tail -1
  timeout 120 python microbench/c4_parts.py 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_perm_mma -c 2 --csv python microbench/quick_time.py C4 1 2>&1 | grep k_perm_mma | awk -F'","' '{print $(NF-2), $NF}'
done
cp /tmp/o.so paper_2106_13706_b200/libddks.so
