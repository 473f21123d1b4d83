#!/bin/bash
# round 2 session 4: re-verification of the restored tree on a fresh box
O=gpurun_out/s4a; mkdir -p $O
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q --durations=25 > $O/gpu_tests.txt 2>&1
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --impl reference > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
for c in cfg1 cfg3 cfg4; do python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --config cfg5 --nq 4000 --steps 3 --warmup 3 > $O/bench_cfg5_4k.json 2> $O/bench_cfg5_4k.err
python tools/cfg5_classes.py > $O/cfg5_classes.txt 2>&1
tail -3 $O/gpu_tests.txt
