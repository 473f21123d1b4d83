#!/bin/bash
# round-1 session-3 GPU call: ingest parity + bench, then ncu evidence for cfg4/cfg5 (exported
# to CSV on the box; .ncu-rep files removed so gpurun_out stays under the copy-back limit)
mkdir -p gpurun_out/s3
O=gpurun_out/s3
python -m pytest tests/test_ingest.py -m gpu -x -q > $O/pytest_ingest.log 2>&1; echo rc=$? >> $O/pytest_ingest.log
python tools/bench_ingest.py > $O/bench_ingest.json 2> $O/bench_ingest.err
B="--steps 1 --warmup 3 --no-cpu-baseline"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $O/ingest_launches.csv python tools/bench_ingest.py --steps 1 --warmup 0 --cpu-rows 1000 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:"k_radix|k_hist|k_score" --csv --log-file $O/cfg5_launches.csv python bench.py --config cfg5 $B > $O/ncu_cfg5_l.log 2>&1
ncu --metrics $M --clock-control none -k regex:"k_itemsets|k_pmt" --csv --log-file $O/cfg4_launches.csv python bench.py --config cfg4 $B > $O/ncu_cfg4_l.log 2>&1
for spec in "cfg4 k_itemsets_tc" "cfg5 k_radix_part" "cfg5 k_radix_count"; do
  set -- $spec
  ncu --set full --import-source on --clock-control none -k regex:$2 -c 1 -o /tmp/$1_$2 python bench.py --config $1 $B > $O/ncu_$1_$2.log 2>&1
  ncu -i /tmp/$1_$2.ncu-rep --page raw --csv > $O/full_$1_$2.csv 2>&1
  ncu -i /tmp/$1_$2.ncu-rep --page details --csv > $O/details_$1_$2.csv 2>&1
done
ls -la $O
