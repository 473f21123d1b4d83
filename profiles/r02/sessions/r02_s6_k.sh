#!/bin/bash
# round 2 session 6: spill group count with the optimistic count kernel
O=gpurun_out/s6k; mkdir -p $O
python tools/cfg5_classes.py 2000 "" CS_SPILL_GROUPS=1 CS_SPILL_GROUPS=3 CS_SPILL_GROUPS=4 CS_SPILL_SEG_ROWS=4194304 CS_SPILL_SEG_ROWS=16777216 > $O/classes.txt 2>&1; cat $O/classes.txt
