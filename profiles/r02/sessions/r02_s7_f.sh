#!/bin/bash
# round 2 session 7: partition class, direct form (no histogram pass) -- tests, timing against the sorted form
O=gpurun_out/s7f; mkdir -p $O
export CS_LIB_PATH=$PWD/tools/libcountgpu_rd.so
timeout 1500 python -m pytest tests/test_gpu_spill.py tests/test_gpu_narrow.py tests/test_gpu_parity.py -x -q -m gpu > $O/tests.txt 2>&1; tail -3 $O/tests.txt
python tools/cfg5_classes.py 2000 "" CS_RADIX_DIRECT=0 CS_SPILL=0 CS_SPILL=0,CS_RADIX_DIRECT=0 CS_SPILL_GROUPS=1 > $O/classes.txt 2>&1; cat $O/classes.txt
CFG5_MAP_KS=7,8 python tools/cfg5_map.py 48 CS_SPILL=0 2>&1 | grep -E '"cells": \[(225280|450560|901120|2097152)' > $O/map_direct.txt; cat $O/map_direct.txt
