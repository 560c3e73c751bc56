#!/bin/bash
# A/B of prebuilt library variants (variants/<prefix>_*.so) under microbench/kd_time.py (call and count time per kd
# setting). usage: microbench/so_kd_ab.sh <prefix> <config> <reps> <setting>...
prefix=$1; cfg=$2; reps=$3; shift 3
cp paper_2106_13706_b200/libddks.so /tmp/libddks.orig.so
for so in variants/${prefix}_*.so; do
  cp "$so" paper_2106_13706_b200/libddks.so
  echo "== $(basename $so)"
  timeout 200 python microbench/kd_time.py $cfg $reps "$@" 2>&1 | grep -v Warn
done
cp /tmp/libddks.orig.so paper_2106_13706_b200/libddks.so
