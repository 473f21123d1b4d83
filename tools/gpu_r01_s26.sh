#!/bin/bash
mkdir -p gpurun_out/s26; O=gpurun_out/s26
python -m pytest tests/test_gpu_parity.py tests/test_ingest.py -m gpu -q -k "edge or itemset or cfg4 or ingest or loader" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python tools/bench_ingest.py > $O/bench_ingest.json 2> $O/bench_ingest.err
