#!/bin/bash
mkdir -p gpurun_out/s17; O=gpurun_out/s17
ncu -i /tmp/s16_selg.ncu-rep --page source --csv --print-source cuda > $O/source_cuda.csv 2> $O/source_cuda.err || true
ls -la /tmp/*.ncu-rep > $O/ls.txt 2>&1
if [ ! -s $O/source_cuda.csv ]; then
  B="--steps 1 --warmup 3 --no-cpu-baseline"
  ncu -f --set full --import-source on --clock-control none -k regex:k_sel_gram -c 1 -o /tmp/s17_selg python bench.py --config cfg4 $B > $O/ncu_f.log 2>&1
  ncu -i /tmp/s17_selg.ncu-rep --page source --csv --print-source cuda > $O/source_cuda.csv 2> $O/source_cuda.err
fi
