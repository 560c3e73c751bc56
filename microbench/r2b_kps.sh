cp paper_2106_13706_b200/libddks.so /tmp/o.so
for v in t64 t128 t256; do cp variants/kps_$v.so paper_2106_13706_b200/libddks.so; echo "== $v"; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pack_sorted -c 3 --csv python microbench/quick_time.py C4 2 2>&1 | grep k_pack_sorted | awk -F'","' '{print $NF}'; done
cp /tmp/o.so paper_2106_13706_b200/libddks.so
