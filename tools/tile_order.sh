#!/usr/bin/env bash
# Kernel 3 time and DRAM bytes per launch for each SHPLB_TILE_ORDER mode (dev tool, GPU box).
for m in 0 1 2; do
  SHPLB_TILE_ORDER=$m python tools/tune_fa.py paper_2603_10353_b200/lib/libshplb.so | sed "s/^/order=$m /" | cut -c1-200
  SHPLB_TILE_ORDER=$m TUNE_STEPS=1 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:fa_sparse -s 3 -c 1 python tools/tune_fa.py paper_2603_10353_b200/lib/libshplb.so 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | sed "s/^/order=$m /"
done
