#!/bin/bash
mkdir -p gpurun_out/s22; O=gpurun_out/s22
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
CS_CRUMB=0 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3_nocrumb.json 2> $O/bench_cfg3_nocrumb.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"k_hist" --csv --log-file $O/cfg3_launches.csv python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_l.log 2>&1
