#!/bin/bash
# round 2 session 5 (final): full GPU suite, bench lines of every config, reference arm, ncu launch lists (traffic)
O=gpurun_out/s5z; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 > $O/gpu_tests.txt 2>&1
tail -3 $O/gpu_tests.txt
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --impl reference > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
for c in cfg1 cfg3 cfg4; do python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --config cfg5 --steps 3 --warmup 3 > $O/bench_cfg5_stream.json 2> $O/bench_cfg5_stream.err
OUT=$O/ncu tools/ncu_traffic.sh cfg2 --no-dropin
OUT=$O/ncu tools/ncu_traffic.sh cfg3
OUT=$O/ncu tools/ncu_traffic.sh cfg4
OUT=$O/ncu tools/ncu_traffic.sh cfg5 --nq 2000
for c in cfg2 cfg3 cfg4 cfg5; do python tools/ncu_step_traffic.py $O/ncu/${c}_launches.csv $c > $O/ncu/${c}_step.txt 2>&1; tail -1 $O/ncu/${c}_step.txt; done
for f in $O/bench_*.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value']), d.get('ms_per_step'), 'e2e', round(d['e2e']['value']), d['e2e'].get('ms_per_step'), d.get('gpu_launches'), (d.get('roofline') or {}).get('frac'))
PY
done
du -sh $O
