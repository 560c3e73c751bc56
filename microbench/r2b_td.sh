# two-dim register path A/B: parity of the kd / warp-x0 / fuzz tests and C5 / C3 timing per variant
cp paper_2106_13706_b200/libddks.so /tmp/o.so
for v in on off; do
  cp variants/td_$v.so paper_2106_13706_b200/libddks.so; echo "== $v"
  timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_kd_scale_gpu.py tests/test_fuzz_gpu.py tests/test_kd_order_free_gpu.py -x -q 2>&1 | tail -1
  timeout 200 python microbench/quick_time.py C5 4 2>&1 | head -1
  timeout 100 python microbench/kd_time.py 5:200000 5 auto 2>&1 | tail -1
done
cp /tmp/o.so paper_2106_13706_b200/libddks.so
