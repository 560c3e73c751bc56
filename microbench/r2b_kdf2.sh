# fused mid-N kd ordering, second version: parity of the kd tests, C2 / C3 call + count times, ncu kernel list of C3
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_kd_scale_gpu.py tests/test_fuzz_gpu.py tests/test_kd_order_free_gpu.py tests/test_graph_gpu.py tests/test_significance_gpu.py -x -q 2>&1 | tail -2
timeout 200 python microbench/kd_time.py C3 20 auto 1 2 3 2>&1 | grep -v Warn
timeout 200 python microbench/kd_time.py C2 20 auto 1 2 2>&1 | grep -v Warn
timeout 200 python microbench/kd_time.py 5:20000 20 auto 2>&1 | grep -v Warn
bash microbench/r2b_ncu_c3.sh
