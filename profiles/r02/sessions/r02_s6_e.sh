#!/bin/bash
# round 2 session 6: digits combined in byte lanes in groups of three (one 16-bit split per group)
O=gpurun_out/s6e; mkdir -p $O
one() {  # config label env...
  c=$1; l=$2; shift; shift
  env "$@" python bench.py --config $c --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c $l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
one cfg2 base X=1
one cfg2 g3 CS_LIB_PATH=$PWD/tools/libcountgpu_g3.so
one cfg3 base X=1
one cfg3 g3 CS_LIB_PATH=$PWD/tools/libcountgpu_g3.so
python tools/cfg5_classes.py 2000 "" > $O/classes_base.txt 2>&1; cat $O/classes_base.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_g3.so python tools/cfg5_classes.py 2000 "" > $O/classes_g3.txt 2>&1; cat $O/classes_g3.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_g3.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > $O/tests_g3.txt 2>&1; tail -2 $O/tests_g3.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_g3.so python tools/cfg5_map.py 48 > $O/cfg5_map_g3.txt 2>&1
