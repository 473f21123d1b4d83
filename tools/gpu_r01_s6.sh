#!/bin/bash
mkdir -p gpurun_out/s6; O=gpurun_out/s6
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "itemset or cfg4" > $O/pytest_itemsets.log 2>&1; echo rc=$? >> $O/pytest_itemsets.log
python -m pytest tests/test_ingest.py -m gpu -x -q > $O/pytest_ingest.log 2>&1; echo rc=$? >> $O/pytest_ingest.log
python bench.py --config cfg4 --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python tools/bench_ingest.py > $O/bench_ingest.json 2> $O/bench_ingest.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
ncu --metrics $M --clock-control none -k regex:"k_sel" --csv --log-file $O/cfg4_sel_launches.csv python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_l.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/ingest_launches.csv python tools/bench_ingest.py --steps 1 --warmup 0 --cpu-rows 1000 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sel_gram -c 1 -o /tmp/selg python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f.log 2>&1
ncu -i /tmp/selg.ncu-rep --page raw --csv > $O/full_k_sel_gram.csv 2>&1
ncu -i /tmp/selg.ncu-rep --page details --csv > $O/details_k_sel_gram.csv 2>&1
