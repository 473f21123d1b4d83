#!/bin/bash
# round 2 session 5: partition kernel with 128-thread CTAs (8 per SM) against 256-thread (4 per SM)
O=gpurun_out/s5g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "partition or threads_identical" > $O/tests_256.txt 2>&1; tail -2 $O/tests_256.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_rx128.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_narrow.py tests/test_gpu_spill.py -x -q -m gpu > $O/tests_128.txt 2>&1; tail -2 $O/tests_128.txt
CFG5_MAP_KS=7,8 python tools/cfg5_map.py 48 CS_SPILL=0 2>&1 | grep -E '"cells": \[(225280|450560|901120|2097152)' > $O/map_256.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_rx128.so CFG5_MAP_KS=7,8 python tools/cfg5_map.py 48 CS_SPILL=0 2>&1 | grep -E '"cells": \[(225280|450560|901120|2097152)' > $O/map_128.txt
paste -d'|' <(grep -o '"k": [0-9], "cells": \[[0-9, ]*\]' $O/map_256.txt) <(grep -o '"us_per_query": [0-9.]*' $O/map_256.txt) <(grep -o '"us_per_query": [0-9.]*' $O/map_128.txt)
python tools/cfg5_classes.py 2000 "" > $O/classes_256.txt 2>&1; cat $O/classes_256.txt
CS_LIB_PATH=$PWD/tools/libcountgpu_rx128.so python tools/cfg5_classes.py 2000 "" > $O/classes_128.txt 2>&1; cat $O/classes_128.txt
