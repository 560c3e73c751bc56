# cluster mid-N kd ordering (k_kdb_cluster): parity of the kd tests (cluster path and the fused fallback forced by
# DDKS_KD_FUSED), then C3 / C2-size / d=5 call + count times and the ncu launch list of C3
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_kd_scale_gpu.py tests/test_fuzz_gpu.py tests/test_kd_order_free_gpu.py tests/test_graph_gpu.py tests/test_significance_gpu.py -x -q 2>&1 | tail -2
DDKS_KD_FUSED=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_kd_order_free_gpu.py -x -q -k "kd or x0 or order" 2>&1 | tail -1
timeout 200 python microbench/kd_time.py C3 20 auto 2 3 2>&1 | grep -v Warn
DDKS_KD_FUSED=1 timeout 200 python microbench/kd_time.py C3 20 2 2>&1 | grep -v Warn
timeout 200 python microbench/kd_time.py C2 20 auto 2 2>&1 | grep -v Warn
timeout 200 python microbench/kd_time.py 5:20000 20 auto 2>&1 | grep -v Warn
bash microbench/r2b_ncu_c3.sh
python microbench/graph_ab.py 20 2>&1 | grep C3
