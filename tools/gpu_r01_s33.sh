#!/bin/bash
mkdir -p gpurun_out/s33; O=gpurun_out/s33
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $O/cfg2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_cfg2.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/cfg4_launches.csv python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_cfg4.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/cfg3_launches.csv python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_cfg3.log 2>&1
ncu -f --set full --import-source on --clock-control none -k regex:k_sel_gram -c 1 -o /tmp/s33_selg python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f.log 2>&1
ncu -i /tmp/s33_selg.ncu-rep --page raw --csv > $O/full_k_sel_gram.csv 2>&1
ncu -i /tmp/s33_selg.ncu-rep --page details --csv > $O/details_k_sel_gram.csv 2>&1
