#!/bin/bash
# round 2 session 6: library built with nvcc --split-compile 0 (86 s instead of ~4 min) -- same speed?
O=gpurun_out/s6i; mkdir -p $O
one() {  # config label env...
  c=$1; l=$2; shift; shift
  env "$@" python bench.py --config $c --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c $l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
for c in cfg2 cfg3 cfg4 cfg1; do
one $c base X=1
one $c split CS_LIB_PATH=$PWD/tools/libcountgpu_split.so
done
python tools/cfg5_classes.py 2000 "" > $O/classes_base.txt 2>&1; cat $O/classes_base.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_split.so python tools/cfg5_classes.py 2000 "" > $O/classes_split.txt 2>&1; cat $O/classes_split.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_split.so timeout 2400 python -m pytest tests -x -q -m gpu > $O/tests_split.txt 2>&1; tail -2 $O/tests_split.txt
