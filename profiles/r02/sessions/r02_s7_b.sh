#!/bin/bash
# round 2 session 7: work-based two-chunk rule for score-only one-shot batches (cfg5 e2e), regression checks
O=gpurun_out/s7b; mkdir -p $O
one() {  # config nq label env...
  c=$1; n=$2; l=$3; shift; shift; shift
  env "$@" python bench.py --config $c $n --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c $l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
one cfg5 "--nq 6000 --steps 2 --warmup 1" new X=1
one cfg5 "--nq 6000 --steps 2 --warmup 1" old CS_QB_SCORE_WORK_G=100000000
one cfg5 "--nq 6000 --steps 2 --warmup 1" new X=1
one cfg2 "" new X=1
one cfg3 "" new X=1
timeout 1500 python -m pytest tests/test_gpu_spill.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dropin.py -x -q -m gpu > $O/tests.txt 2>&1; tail -2 $O/tests.txt
