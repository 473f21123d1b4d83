#!/bin/bash
# round 2 session 4: compile-time byte-lane digit count in the lane16 / rows16 paths
O=gpurun_out/s4i; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_narrow.py tests/test_gpu_spill.py -x -q -m gpu > $O/tests.txt 2>&1
tail -3 $O/tests.txt
python tools/cfg5_classes.py 2000 "" > $O/cfg5_classes.txt 2>&1; cat $O/cfg5_classes.txt
python tools/cfg5_map.py 48 > $O/cfg5_map.txt 2>&1
python bench.py --no-cpu-baseline --no-dropin > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --config cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --config cfg1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
for f in $O/bench_*.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value']), d['ms_per_step'], 'e2e', round(d['e2e']['value']), d['e2e'].get('ms_per_step'), d['gpu_launches'])
PY
done
