#!/bin/bash
# full verification: GPU tests, smoke, every config's bench line, the reference arm
O=gpurun_out/full; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in cfg1 cfg3 cfg4; do python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --config cfg5 --steps 3 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_cfg2.json 2> $O/ref_cfg2.err
python tools/bench_ingest.py > $O/bench_ingest.json 2> $O/bench_ingest.err
