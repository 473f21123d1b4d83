#!/bin/bash
# round 2 session 6: groups-of-three joint index with dot products in the narrow and spill classes
O=gpurun_out/s6h; mkdir -p $O
export CS_LIB_PATH=$PWD/tools/libcountgpu_jg3.so
timeout 1500 python -m pytest tests/test_gpu_narrow.py tests/test_gpu_spill.py tests/test_gpu_parity.py -x -q -m gpu > $O/tests.txt 2>&1; tail -2 $O/tests.txt
python tools/cfg5_classes.py 2000 "" > $O/classes_g3.txt 2>&1; cat $O/classes_g3.txt
CS_JOINT_G3=0 python tools/cfg5_classes.py 2000 "" > $O/classes_pair.txt 2>&1; cat $O/classes_pair.txt
CFG5_MAP_KS=6,7,8 python tools/cfg5_map.py 48 2>&1 | grep -E '"cells": \[(56320|112640|225280)' > $O/map_g3.txt
CS_JOINT_G3=0 CFG5_MAP_KS=6,7,8 python tools/cfg5_map.py 48 2>&1 | grep -E '"cells": \[(56320|112640|225280)' > $O/map_pair.txt
paste -d'|' <(grep -o '"k": [0-9], "cells": \[[0-9, ]*\]' $O/map_g3.txt) <(grep -o '"frac": [0-9.]*' $O/map_g3.txt) <(grep -o '"frac": [0-9.]*' $O/map_pair.txt)
