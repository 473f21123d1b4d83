#!/bin/bash
# round 2 session 6: right shifts on the FMA pipe (IMAD.HI) in the K1 inner loops
O=gpurun_out/s6b; mkdir -p $O
one() {  # config label env...
  c=$1; l=$2; shift; shift
  env "$@" python bench.py --config $c --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c $l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
for c in cfg2 cfg3 cfg1; do
one $c base X=1
one $c fma CS_LIB_PATH=$PWD/tools/libcountgpu_fma.so
done
python tools/cfg5_classes.py 2000 "" > $O/classes_base.txt 2>&1; cat $O/classes_base.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_fma.so python tools/cfg5_classes.py 2000 "" > $O/classes_fma.txt 2>&1; cat $O/classes_fma.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_fma.so python tools/cfg5_map.py 48 > $O/cfg5_map_fma.txt 2>&1
