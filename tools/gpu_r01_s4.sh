#!/bin/bash
mkdir -p gpurun_out/s4; O=gpurun_out/s4
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "itemset or cfg4" > $O/pytest_itemsets.log 2>&1; echo rc=$? >> $O/pytest_itemsets.log
python bench.py --config cfg4 --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
CS_ITEMSETS_SEL=0 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg4_tc.json 2> $O/bench_cfg4_tc.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
ncu --metrics $M --clock-control none -k regex:"k_sel" --csv --log-file $O/cfg4_sel_launches.csv python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_l.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sel_count -c 1 -o /tmp/selc python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f.log 2>&1
ncu -i /tmp/selc.ncu-rep --page raw --csv > $O/full_k_sel_count.csv 2>&1
ncu -i /tmp/selc.ncu-rep --page details --csv > $O/details_k_sel_count.csv 2>&1
ncu -i /tmp/selc.ncu-rep --page source --csv > $O/source_k_sel_count.csv 2>&1
