#!/bin/bash
# round 2 session 7 (last): smoke, full GPU suite, default bench + reference arm, torchrun and forced-sharded paths
O=gpurun_out/s7z; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 3000 python -m pytest tests -m gpu -x -q > $O/gpu_tests.txt 2>&1; tail -2 $O/gpu_tests.txt
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --impl reference > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --no-dropin > $O/bench_cfg2_torchrun.json 2> $O/bench_cfg2_torchrun.err
CS_BENCH_FORCE_SHARDED=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --config cfg5 --nq 2000 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_cfg5_sharded1.json 2> $O/bench_cfg5_sharded1.err
for f in $O/bench_*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['value']), d.get('ms_per_step'), 'e2e', round(d['e2e']['value']), d['e2e'].get('ms_per_step'), d.get('gpu_launches'), d.get('scaling'), (d.get('run') or {}).get('parallelism'))
except Exception as e:
    print(sys.argv[1], 'ERR', e)
PY
done
