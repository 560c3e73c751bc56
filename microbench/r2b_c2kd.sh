cp paper_2106_13706_b200/libddks.so /tmp/orig.so
for v in base r8t128t256 r4t128t256 r4t256t256; do
  cp variants/c2_$v.so paper_2106_13706_b200/libddks.so
  echo "== $v"
  timeout 100 python microbench/kd_time.py C2 20 auto 1 2 3 2,4 2,8 3,3,3 4,8 2>&1 | grep -v Warn
done
cp /tmp/orig.so paper_2106_13706_b200/libddks.so
