#!/bin/bash
# A/B of prebuilt library variants (variants/<prefix>_*.so, built here with DDKS_NVCC_EXTRA): each is copied over
# paper_2106_13706_b200/libddks.so and timed with microbench/quick_time.py on the given config.
# usage: microbench/so_ab.sh <prefix> <config> [reps]
prefix=$1; cfg=$2; reps=${3:-20}
cp paper_2106_13706_b200/libddks.so /tmp/libddks.orig.so
for so in variants/${prefix}_*.so; do
  cp "$so" paper_2106_13706_b200/libddks.so
  echo "== $(basename $so)"
  timeout 120 python microbench/quick_time.py $cfg $reps 2>&1 | tail -2
done
cp /tmp/libddks.orig.so paper_2106_13706_b200/libddks.so
