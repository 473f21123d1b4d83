#!/bin/bash
# round 2 session 5: cfg2 e2e knob sweep; ncu --set full of cfg2's two largest K1 variants
O=gpurun_out/s5c; mkdir -p $O
one() {  # label env...
  l=$1; shift
  env "$@" python bench.py --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/e2e_sweep.txt
}
one default X=1
one chunks1 CS_QB_CHUNKS=1
one chunks2 CS_QB_CHUNKS=2
one chunks3 CS_QB_CHUNKS=3
one minchunk1000 CS_QB_MIN_CHUNK=1000
one minchunk1500 CS_QB_MIN_CHUNK=1500
one minchunk3000 CS_QB_MIN_CHUNK=3000
one growth3 CS_QB_GROWTH=3
one growth6 CS_QB_GROWTH=6
one planthreads2 CS_PLAN_THREADS=2
one streams2 CS_STREAMS=2
one streams3 CS_STREAMS=3
run() {  # name regex
  ncu --set full --clock-control none --cache-control none -k "regex:$2" --launch-skip 3 -c 1 -o /tmp/$1 -f \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dropin > $O/$1.ncu.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
run cfg2_k6_rows16 'k_hist<.int.6, .int.3, .int.1>'
run cfg2_k4_lane16 'k_hist<.int.4, .int.0, .int.1>'
du -sh $O
