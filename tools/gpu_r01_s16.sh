#!/bin/bash
mkdir -p gpurun_out/s16; O=gpurun_out/s16
python -m pytest tests/test_cli.py -m gpu -q > $O/pytest_cli.log 2>&1; echo rc=$? >> $O/pytest_cli.log
B="--steps 1 --warmup 3 --no-cpu-baseline"
ncu -f --set full --import-source on --clock-control none -k regex:k_sel_gram -c 1 -o /tmp/s16_selg python bench.py --config cfg4 $B > $O/ncu_f.log 2>&1
ncu -i /tmp/s16_selg.ncu-rep --page raw --csv > $O/full_k_sel_gram.csv 2>&1
ncu -i /tmp/s16_selg.ncu-rep --page details --csv > $O/details_k_sel_gram.csv 2>&1
ncu -i /tmp/s16_selg.ncu-rep --page source --csv > $O/source_k_sel_gram.csv 2>&1
