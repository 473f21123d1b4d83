#!/bin/bash
# round 2 session 4: spill/narrow/parity tests on the lean spill build; bench-output gap
O=gpurun_out/s4f; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_spill.py tests/test_gpu_narrow.py tests/test_gpu_parity.py -x -q -m gpu > $O/tests.txt 2>&1
tail -3 $O/tests.txt
python tools/cfg5_classes.py 2000 "" CFG5_BENCH_OUTPUTS=1 CFG5_BENCH_OUTPUTS=1,CS_STREAMS=1 > $O/cfg5_outputs_2k.txt 2>&1
python tools/cfg5_classes.py 4000 "" CFG5_BENCH_OUTPUTS=1 > $O/cfg5_outputs_4k.txt 2>&1
cat $O/cfg5_outputs_2k.txt $O/cfg5_outputs_4k.txt
CS_TRACE=1 python bench.py --config cfg5 --nq 4000 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5_4k.json 2> $O/bench_cfg5_4k.err
cat $O/bench_cfg5_4k.json | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'], d['clocks'], d.get('diag'))"
