#!/bin/bash
mkdir -p gpurun_out/s28; O=gpurun_out/s28
for dbg in 0 1 2 3 4 7; do
  for dm in 1; do
  CS_SEL_DEBUG=$dbg python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_dbg$dbg.json 2> $O/bench_dbg$dbg.err
  done
done
