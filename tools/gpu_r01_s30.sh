#!/bin/bash
mkdir -p gpurun_out/s30; O=gpurun_out/s30
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "itemset or cfg4" > $O/pytest_itemsets.log 2>&1; echo rc=$? >> $O/pytest_itemsets.log
for dbg in 0 7; do
  CS_SEL_DEBUG=$dbg python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_dbg$dbg.json 2> $O/bench_dbg$dbg.err
done
