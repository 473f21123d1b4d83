#!/bin/bash
# Per-launch time + DRAM bytes of the dominant kernels of one bench step, captured WITHOUT
# ncu's cache flush between kernels (--cache-control none: L2 state carries over from the
# previous kernel as in the real run) and without clock control.  Output: CSV launch lists in
# $OUT (default gpurun_out/ncu).  Usage: tools/ncu_traffic.sh <config> [extra bench args]
set -e
cfg=$1; shift
OUT=${OUT:-gpurun_out/ncu}
mkdir -p $OUT
case $cfg in
  cfg4) K='regex:k_sel|k_itemsets|k_pmt' ;;
  *) K='regex:k_hist|k_radix|k_spill|k_bitmap_query|k_bitmap_mobius|k_score|k_family' ;;
esac
ncu --cache-control none --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k "$K" --log-file $OUT/${cfg}_launches.csv python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline "$@" \
    > $OUT/${cfg}_bench_under_ncu.log 2>&1
