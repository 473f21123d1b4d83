#!/bin/bash
# round 2 session 5: optimistic narrow pass (red.shared, verified by the counter sum), 128-thread partition CTAs
O=gpurun_out/s5h; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_narrow.py tests/test_gpu_spill.py tests/test_gpu_parity.py -x -q -m gpu > $O/tests.txt 2>&1
tail -3 $O/tests.txt
python tools/cfg5_classes.py 2000 "" CS_NARROW_FAST=0 > $O/cfg5_classes.txt 2>&1; cat $O/cfg5_classes.txt
CFG5_MAP_KS=6,7,8 python tools/cfg5_map.py 48 2>&1 | grep -E '"cells": \[(56320|112640)' > $O/map_fast.txt
CFG5_MAP_KS=6,7,8 python tools/cfg5_map.py 48 CS_NARROW_FAST=0 2>&1 | grep -E '"cells": \[(56320|112640)' > $O/map_exact.txt
paste -d'|' <(grep -o '"k": [0-9], "cells": \[[0-9, ]*\]' $O/map_fast.txt) <(grep -o '"frac": [0-9.]*' $O/map_fast.txt) <(grep -o '"frac": [0-9.]*' $O/map_exact.txt)
