#!/bin/bash
mkdir -p gpurun_out/s7; O=gpurun_out/s7
B="--steps 1 --warmup 3 --no-cpu-baseline"
ncu -f --set full --import-source on --clock-control none -k regex:k_sel_gram -c 1 -o /tmp/s7_selg python bench.py --config cfg4 $B > $O/ncu_f.log 2>&1
ncu -i /tmp/s7_selg.ncu-rep --page raw --csv > $O/full_k_sel_gram.csv 2>&1
ncu -i /tmp/s7_selg.ncu-rep --page details --csv > $O/details_k_sel_gram.csv 2>&1
ncu -i /tmp/s7_selg.ncu-rep --page source --csv > $O/source_k_sel_gram.csv 2>&1
ncu -f --set full --import-source on --clock-control none -k regex:"k_txt_parse_thr|k_txt_lines" -c 2 -o /tmp/s7_txt python tools/bench_ingest.py --steps 1 --warmup 0 --cpu-rows 1000 > $O/ncu_txt.log 2>&1
ncu -i /tmp/s7_txt.ncu-rep --page details --csv > $O/details_txt.csv 2>&1
ncu -i /tmp/s7_txt.ncu-rep --page raw --csv > $O/full_txt.csv 2>&1
