#!/bin/bash
# round 2 session 6: IDP.4A per-row offsets when every digit fits the byte lanes (C <= 256)
O=gpurun_out/s6d; mkdir -p $O
one() {  # config label env...
  c=$1; l=$2; shift; shift
  env "$@" python bench.py --config $c --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c $l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
for c in cfg2 cfg3 cfg1; do
one $c idp2 X=1
one $c idp4 CS_LIB_PATH=$PWD/tools/libcountgpu_idp4.so
done
CS_LIB_PATH=$PWD/tools/libcountgpu_idp4.so python tools/cfg5_classes.py 2000 "" > $O/classes_idp4.txt 2>&1; cat $O/classes_idp4.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_idp4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > $O/tests_idp4.txt 2>&1; tail -2 $O/tests_idp4.txt
