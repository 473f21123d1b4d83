#!/bin/bash
# round 2 session 3: re-verification of the restored tree on a fresh box
mkdir -p gpurun_out/s3a
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3a/smoke.txt 2>&1
python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/s3a/gpu_tests.txt 2>&1
python bench.py > gpurun_out/s3a/bench_cfg2.json 2> gpurun_out/s3a/bench_cfg2.err
python bench.py --impl reference > gpurun_out/s3a/bench_ref_cfg2.json 2> gpurun_out/s3a/bench_ref_cfg2.err
for c in cfg1 cfg3 cfg4; do python bench.py --config $c > gpurun_out/s3a/bench_$c.json 2> gpurun_out/s3a/bench_$c.err; done
python bench.py --config cfg5 --nq 4000 --steps 3 --warmup 3 > gpurun_out/s3a/bench_cfg5_4k.json 2> gpurun_out/s3a/bench_cfg5_4k.err
tail -3 gpurun_out/s3a/gpu_tests.txt
