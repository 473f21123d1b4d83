#!/bin/bash
# round 2 session 4: cfg5 roofline map by (k, table size), class knob comparison
O=gpurun_out/s4b; mkdir -p $O
python tools/cfg5_map.py 48 > $O/cfg5_map.txt 2>&1
python tools/cfg5_classes.py 2000 "" CS_NARROW_MAX_PASSES=2 CS_NARROW_MAX_PASSES=4 CS_NARROW=0 CS_SEG_MAX_ROWS=8388608 CS_SEG_MAX_ROWS=2097152 > $O/cfg5_classes.txt 2>&1
tail -5 $O/cfg5_classes.txt
