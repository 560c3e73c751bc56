# rdKS bucket count sweep (about N / DIV buckets per corner): parity of the rdKS tests and C5 / C2 call times
cp paper_2106_13706_b200/libddks.so /tmp/o.so
for v in d4 d8 d16 d32; do
  cp variants/rbk_$v.so paper_2106_13706_b200/libddks.so; echo "== $v"
  timeout 300 python -m pytest tests/test_approx_gpu.py -x -q -k rdks 2>&1 | tail -1
  timeout 120 python microbench/approx_c5.py 30 rdks 2>&1 | tail -1
done
cp /tmp/o.so paper_2106_13706_b200/libddks.so
