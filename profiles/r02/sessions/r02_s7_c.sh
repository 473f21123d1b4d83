#!/bin/bash
# round 2 session 7: per-group spill streams (match.any routing) -- tests, group-count sweep
O=gpurun_out/s7c; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_spill.py tests/test_gpu_narrow.py -x -q -m gpu > $O/tests.txt 2>&1; tail -3 $O/tests.txt
python tools/cfg5_classes.py 2000 "" CS_SPILL_GROUPS=1 CS_SPILL_GROUPS=3 CS_SPILL_GROUPS=4 CS_SPILL_GROUPS=6 CS_SPILL_GROUPS=8 > $O/classes.txt 2>&1; cat $O/classes.txt
CFG5_MAP_KS=7,8 python tools/cfg5_map.py 48 CS_SPILL_GROUPS=4 2>&1 | grep -E '"cells": \[(225280|450560|901120)' > $O/map_g4.txt; cat $O/map_g4.txt
