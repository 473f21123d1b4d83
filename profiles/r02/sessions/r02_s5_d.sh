#!/bin/bash
# round 2 session 5: chunk-share sweep for the one-shot e2e path (cfg2, cfg3); ncu of cfg2's largest variants
O=gpurun_out/s5d; mkdir -p $O
one() {  # config label env...
  c=$1; l=$2; shift; shift
  env "$@" python bench.py --config $c --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c $l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/e2e_sweep.txt
}
for c in cfg2 cfg3; do
one $c g4_min2000 CS_QB_GROWTH=4 CS_QB_MIN_CHUNK=2000
one $c g3_min2000 CS_QB_GROWTH=3 CS_QB_MIN_CHUNK=2000
one $c g3_min700 CS_QB_GROWTH=3 CS_QB_MIN_CHUNK=700
one $c g2_min3000 CS_QB_GROWTH=2 CS_QB_MIN_CHUNK=3000
one $c g2_min1400 CS_QB_GROWTH=2 CS_QB_MIN_CHUNK=1400
one $c g2_min600 CS_QB_GROWTH=2 CS_QB_MIN_CHUNK=600
done
run() {  # name skip
  ncu --set full --clock-control none --cache-control none -k k_hist --launch-skip $2 -c 1 -o /tmp/$1 -f \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dropin > $O/$1.ncu.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
run cfg2_top1 33
run cfg2_top2 34
du -sh $O
