#!/bin/bash
# round 2 session 6: groups of two as the fallback of groups of three
O=gpurun_out/s6f; mkdir -p $O
CS_LIB_PATH=$PWD/tools/libcountgpu_g3.so python tools/cfg5_classes.py 2000 "" > $O/classes_g3.txt 2>&1; cat $O/classes_g3.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_g32.so python tools/cfg5_classes.py 2000 "" > $O/classes_g32.txt 2>&1; cat $O/classes_g32.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_g3.so python tools/cfg5_classes.py 2000 "" >> $O/classes_g3.txt 2>&1; tail -1 $O/classes_g3.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_g32.so python tools/cfg5_classes.py 2000 "" >> $O/classes_g32.txt 2>&1; tail -1 $O/classes_g32.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_g32.so python bench.py --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2 g32', d['ms_per_step'], d['e2e']['ms_per_step'])"
CS_LIB_PATH=$PWD/tools/libcountgpu_g32.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_narrow.py -x -q -m gpu > $O/tests_g32.txt 2>&1; tail -2 $O/tests_g32.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_g32.so python tools/cfg5_map.py 48 > $O/cfg5_map_g32.txt 2>&1
