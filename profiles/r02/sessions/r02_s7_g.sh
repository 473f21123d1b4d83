#!/bin/bash
# round 2 session 7: would 16-bit replica counters (CS_HALF, R doubled) pay on cfg5's 1760..3520-cell tables?
O=gpurun_out/s7g; mkdir -p $O
CFG5_MAP_KS=5,6,7 python tools/cfg5_map.py 48 CS_SEG_MAX_ROWS=1048576 2>&1 | grep -E '"cells": \[(1760|3520),' > $O/map_seg1m.txt
CFG5_MAP_KS=5,6,7 python tools/cfg5_map.py 48 CS_SEG_MAX_ROWS=1048576,CS_HALF=1 2>&1 | grep -E '"cells": \[(1760|3520),' > $O/map_seg1m_half.txt
paste -d'|' <(grep -o '"k": [0-9], "cells": \[[0-9, ]*\]' $O/map_seg1m.txt) <(grep -o '"frac": [0-9.]*' $O/map_seg1m.txt) <(grep -o '"frac": [0-9.]*' $O/map_seg1m_half.txt)
