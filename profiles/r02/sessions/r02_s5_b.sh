#!/bin/bash
# round 2 session 5: PTX spill slot (tests, map), cfg5 ncu launch list including the spill kernels
O=gpurun_out/s5b; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_spill.py tests/test_gpu_narrow.py -x -q -m gpu > $O/tests.txt 2>&1
tail -3 $O/tests.txt
CFG5_MAP_KS=7,8 python tools/cfg5_map.py 48 > $O/cfg5_map_k78.txt 2>&1
grep -E '"cells": \[(225280|450560)' $O/cfg5_map_k78.txt
python tools/cfg5_classes.py 2000 "" CS_SPILL_GROUPS=1 CS_SPILL_GROUPS=3 CS_SPILL_GROUPS=4 > $O/cfg5_classes.txt 2>&1; cat $O/cfg5_classes.txt
OUT=$O/ncu tools/ncu_traffic.sh cfg5 --nq 2000
python tools/ncu_step_traffic.py $O/ncu/cfg5_launches.csv cfg5 > $O/ncu/cfg5_step.txt 2>&1; cat $O/ncu/cfg5_step.txt
