#!/bin/bash
# round 2 session 4: spill class tests + cfg5 map/knobs, then ncu --set full of single classes
# (raw CSV pages exported on the box; the .ncu-rep files are too big to bring back)
O=gpurun_out/s4d; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_spill.py tests/test_gpu_narrow.py tests/test_gpu_parity.py -x -q -m gpu > $O/tests.txt 2>&1
tail -5 $O/tests.txt
python tools/cfg5_classes.py 2000 "" CS_STREAMS=1 CS_SPILL=0 CS_SPILL=0,CS_STREAMS=1 CS_SPILL_RANGES=4 CS_SPILL_RANGES=16 CS_SPILL_SEG_ROWS=4194304 CS_SPILL_SEG_ROWS=16777216 > $O/cfg5_classes.txt 2>&1
cat $O/cfg5_classes.txt
python tools/cfg5_map.py 48 > $O/cfg5_map.txt 2>&1
run() {  # name k lo hi regex
  python tools/cfg5_one.py $2 $3 $4 12 > $O/$1.txt 2>&1 || return
  ncu --set full --clock-control none -k "regex:$5" --launch-skip 1 -c 1 -o /tmp/$1 -f \
      python tools/cfg5_one.py $2 $3 $4 12 > $O/$1.ncu.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
run k2_pack 2 0 41 k_hist
run k5_small 5 41 1760 k_hist
run k7_rows 7 28160 56320 k_hist
run k7_narrow16 7 56320 112640 k_hist
run k8_narrow8 8 112640 225280 k_hist
run k8_spill_hist 8 225280 450560 k_spill_hist
run k8_spill_count 8 225280 450560 k_spill_count
du -sh $O
