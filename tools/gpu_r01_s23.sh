#!/bin/bash
mkdir -p gpurun_out/s23; O=gpurun_out/s23
B="--steps 1 --warmup 1 --no-cpu-baseline"
ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_hist<.int.4, .int.0, .int.2>" -c 1 -o /tmp/s23_c3 python bench.py --config cfg3 $B > $O/ncu_c3.log 2>&1
ncu -i /tmp/s23_c3.ncu-rep --page raw --csv > $O/full_cfg3_khist402.csv 2>&1
ncu -i /tmp/s23_c3.ncu-rep --page details --csv > $O/details_cfg3_khist402.csv 2>&1
ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_hist<.int.6, .int.3, .int.1>" -c 1 -o /tmp/s23_c2 python bench.py $B > $O/ncu_c2.log 2>&1
ncu -i /tmp/s23_c2.ncu-rep --page raw --csv > $O/full_cfg2_khist631.csv 2>&1
ncu -i /tmp/s23_c2.ncu-rep --page details --csv > $O/details_cfg2_khist631.csv 2>&1
