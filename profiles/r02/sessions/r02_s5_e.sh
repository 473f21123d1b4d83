#!/bin/bash
# round 2 session 5: growth-2 chunk default (3 runs each), 512-thread CTAs on cfg2 / cfg3 / cfg1
O=gpurun_out/s5e; mkdir -p $O
one() {  # config label env...
  c=$1; l=$2; shift; shift
  env "$@" python bench.py --config $c --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c $l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
for i in 1 2 3; do
one cfg2 new_default X=1
one cfg2 old_g4_min2000 CS_QB_GROWTH=4 CS_QB_MIN_CHUNK=2000
done
for i in 1 2; do
one cfg3 new_default X=1
one cfg3 old_g4_min2000 CS_QB_GROWTH=4 CS_QB_MIN_CHUNK=2000
done
one cfg2 t512 CS_LIB_PATH=$PWD/tools/libcountgpu_t512.so
one cfg3 t512 CS_LIB_PATH=$PWD/tools/libcountgpu_t512.so
one cfg1 t512 CS_LIB_PATH=$PWD/tools/libcountgpu_t512.so
one cfg1 t1024 X=1
CS_TRACE=1 python bench.py --no-cpu-baseline --no-dropin --steps 2 --warmup 1 2>&1 | grep -E "plan_build: (setup|upload)|cs_query_batch" | tail -12 > $O/trace_cfg2.txt; cat $O/trace_cfg2.txt
