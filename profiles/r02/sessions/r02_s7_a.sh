#!/bin/bash
# round 2 session 7: cfg5 e2e -- planning of a 2,000-query one-shot call exposed or chunked
O=gpurun_out/s7a; mkdir -p $O
one() {  # label env...
  l=$1; shift
  env "$@" python bench.py --config cfg5 --nq 6000 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$l', 'dev_ms %.1f'%d['ms_per_step'], 'e2e_ms %.1f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
one default X=1
one chunk_min250 CS_QB_SCORE_MIN=1 CS_QB_MIN_CHUNK=250
one chunk_min500 CS_QB_SCORE_MIN=1 CS_QB_MIN_CHUNK=500
one chunk2 CS_QB_CHUNKS=2
one bench6000 CS_BENCH_CHUNK=6000
CS_TRACE=1 python bench.py --config cfg5 --nq 2000 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "plan_build: (setup|upload)|cs_query_batch" | tail -4
