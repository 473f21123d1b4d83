#!/bin/bash
# round 2 session 4: hand-scheduled narrow bump (tests, map), ncu of the dominant small-k variants
O=gpurun_out/s4h; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_narrow.py tests/test_gpu_spill.py -x -q -m gpu > $O/tests.txt 2>&1
tail -3 $O/tests.txt
CFG5_MAP_KS=6,7,8 python tools/cfg5_map.py 48 > $O/cfg5_map_k678.txt 2>&1
grep -E '"cells": \[(56320|112640|225280)' $O/cfg5_map_k678.txt
python tools/cfg5_classes.py 2000 "" > $O/cfg5_classes.txt 2>&1; cat $O/cfg5_classes.txt
run() {  # name k lo hi regex count
  ncu --set full --clock-control none -k "regex:$5" -c $6 -o /tmp/$1 -f \
      python tools/cfg5_one.py $2 $3 $4 48 > $O/$1.ncu.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
run k3_small 3 41 1760 k_hist 6
run k4_small 4 41 1760 k_hist 6
run k5_small 5 41 1760 k_hist 6
du -sh $O
