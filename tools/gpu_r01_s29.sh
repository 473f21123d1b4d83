#!/bin/bash
mkdir -p gpurun_out/s29; O=gpurun_out/s29
for u in 8 16 48 128; do
  for dbg in 0 7; do
  CS_SEL_UNITS=$u CS_SEL_DEBUG=$dbg python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_u${u}_dbg$dbg.json 2> $O/err_u${u}_dbg$dbg.err
  done
done
