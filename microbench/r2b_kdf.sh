# fused mid-N kd ordering (k_kdb_fused): parity of the kd tests, then C2 / C3 call and count times per variant
cp paper_2106_13706_b200/libddks.so /tmp/o.so
for v in base r4t128; do
  cp variants/kdf_$v.so paper_2106_13706_b200/libddks.so; echo "== $v"
  [ $v = base ] && timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_kd_scale_gpu.py tests/test_fuzz_gpu.py tests/test_kd_order_free_gpu.py tests/test_graph_gpu.py tests/test_significance_gpu.py -x -q 2>&1 | tail -2
  timeout 200 python microbench/kd_time.py C2 20 auto 1 2 2>&1 | grep -v Warn
  timeout 200 python microbench/kd_time.py C3 20 auto 1 2 2>&1 | grep -v Warn
  timeout 200 python microbench/quick_time.py C2 20 2>&1 | head -1
  timeout 200 python microbench/quick_time.py C3 20 2>&1 | head -1
done
cp /tmp/o.so paper_2106_13706_b200/libddks.so
