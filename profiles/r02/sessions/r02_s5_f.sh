#!/bin/bash
# round 2 session 5: row segmentation of cfg2 / cfg3 for L2 locality
O=gpurun_out/s5f; mkdir -p $O
one() {  # config label env...
  c=$1; l=$2; shift; shift
  env "$@" python bench.py --config $c --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c $l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
one cfg2 seg4M X=1
one cfg2 seg512K CS_SEG_MAX_ROWS=524288
one cfg2 seg256K CS_SEG_MAX_ROWS=262144
one cfg2 seg128K CS_SEG_MAX_ROWS=131072
one cfg2 seg512K_noorder CS_SEG_MAX_ROWS=524288 CS_SEG_ORDER=0
one cfg3 seg4M X=1
one cfg3 seg512K CS_SEG_MAX_ROWS=524288
