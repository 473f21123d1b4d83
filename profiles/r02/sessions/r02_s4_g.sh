#!/bin/bash
# round 2 session 4: bench lines of every config on the side-stream build (and CS_STREAMS=1 for cfg2/cfg3)
O=gpurun_out/s4g; mkdir -p $O
python bench.py --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
CS_STREAMS=1 python bench.py --no-cpu-baseline --no-dropin > $O/bench_cfg2_1stream.json 2> $O/bench_cfg2_1stream.err
python bench.py --config cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
CS_STREAMS=1 python bench.py --config cfg3 --no-cpu-baseline > $O/bench_cfg3_1stream.json 2> $O/bench_cfg3_1stream.err
python bench.py --config cfg1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
for f in $O/bench_*.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value']), d['ms_per_step'], 'e2e', round(d['e2e']['value']), d['e2e'].get('ms_per_step'), d['gpu_launches'])
PY
done
