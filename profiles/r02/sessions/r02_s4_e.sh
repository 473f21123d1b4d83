#!/bin/bash
# round 2 session 4: lean spill class, 512-thread CTAs (128 registers), HBM read ceiling
O=gpurun_out/s4e; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb8 tools/microbench8.cu && /tmp/mb8 > $O/microbench8.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_spill.py tests/test_gpu_narrow.py -x -q -m gpu > $O/tests.txt 2>&1
tail -3 $O/tests.txt
python tools/cfg5_classes.py 2000 "" CS_SPILL=0 CS_SPILL_GROUPS=1 CS_SPILL_GROUPS=4 > $O/cfg5_classes.txt 2>&1
CS_LIB_PATH=$PWD/tools/libcountgpu_t512.so python tools/cfg5_classes.py 2000 "" CS_SPILL=0 > $O/cfg5_classes_t512.txt 2>&1
CFG5_MAP_KS=7,8 python tools/cfg5_map.py 48 > $O/cfg5_map_k78.txt 2>&1
CS_LIB_PATH=$PWD/tools/libcountgpu_t512.so python tools/cfg5_map.py 48 > $O/cfg5_map_t512.txt 2>&1
cat $O/microbench8.txt $O/cfg5_classes.txt $O/cfg5_classes_t512.txt
