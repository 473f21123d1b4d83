#!/bin/bash
mkdir -p gpurun_out/s19; O=gpurun_out/s19
CS_TRACE=1 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
CS_TRACE=1 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
