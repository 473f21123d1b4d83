#!/bin/bash
mkdir -p gpurun_out/s14; O=gpurun_out/s14
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pinned or edges or golden or sweep or cfg1" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
CS_TRACE=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
CS_ZEROCOPY=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg2_nozc.json 2> $O/bench_cfg2_nozc.err
python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
