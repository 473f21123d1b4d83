#!/bin/bash
mkdir -p gpurun_out/s27; O=gpurun_out/s27
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "itemset or cfg4" > $O/pytest_itemsets.log 2>&1; echo rc=$? >> $O/pytest_itemsets.log
python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
B="--steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sel" --csv --log-file $O/cfg4_sel_launches.csv python bench.py --config cfg4 $B > $O/ncu_l.log 2>&1
