#!/bin/bash
# round 2 session 7: more side streams (build with 7), narrow segment size
O=gpurun_out/s7d; mkdir -p $O
export CS_LIB_PATH=$PWD/tools/libcountgpu_s8.so
python tools/cfg5_classes.py 2000 CFG5_BENCH_OUTPUTS=1,CS_STREAMS=4 CFG5_BENCH_OUTPUTS=1,CS_STREAMS=6 CFG5_BENCH_OUTPUTS=1,CS_STREAMS=8 CFG5_BENCH_OUTPUTS=1,CS_STREAMS=4,CS_NARROW_SEG_ROWS=8388608 CFG5_BENCH_OUTPUTS=1,CS_STREAMS=4,CS_NARROW_SEG_ROWS=33554432 > $O/classes.txt 2>&1; cat $O/classes.txt
for st in 4 6 8; do CS_STREAMS=$st python bench.py --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2 streams $st', d['ms_per_step'], d['e2e']['ms_per_step'])"; done
