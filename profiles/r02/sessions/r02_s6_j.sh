#!/bin/bash
# round 2 session 6: optimistic passes in the spill class
O=gpurun_out/s6j; mkdir -p $O
export CS_LIB_PATH=$PWD/tools/libcountgpu_spopt.so
timeout 1500 python -m pytest tests/test_gpu_spill.py tests/test_gpu_narrow.py tests/test_gpu_parity.py tests/test_gpu_multiproc.py -x -q -m gpu > $O/tests.txt 2>&1; tail -2 $O/tests.txt
python tools/cfg5_classes.py 2000 "" CS_NARROW_FAST=0 > $O/classes_opt.txt 2>&1; cat $O/classes_opt.txt
unset CS_LIB_PATH
python tools/cfg5_classes.py 2000 "" > $O/classes_base.txt 2>&1; cat $O/classes_base.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_spopt.so CFG5_MAP_KS=7,8 python tools/cfg5_map.py 48 2>&1 | grep -E '"cells": \[(225280|450560)' > $O/map_opt.txt; cat $O/map_opt.txt
