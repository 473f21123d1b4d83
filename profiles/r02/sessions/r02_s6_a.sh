#!/bin/bash
# round 2 session 6: cfg2 L2 residency -- streaming table stores, warm-L2 diagnostic, DRAM bytes per launch
O=gpurun_out/s6a; mkdir -p $O
one() {  # label env...
  l=$1; shift
  env "$@" python bench.py --no-cpu-baseline --no-dropin 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$l', 'dev_ms %.3f'%d['ms_per_step'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" | tee -a $O/sweep.txt
}
one base X=1
one base_noflush CS_BENCH_NOFLUSH=1
one stcs CS_LIB_PATH=$PWD/tools/libcountgpu_stcs.so
one stcs_noflush CS_LIB_PATH=$PWD/tools/libcountgpu_stcs.so CS_BENCH_NOFLUSH=1
one base X=1
one stcs CS_LIB_PATH=$PWD/tools/libcountgpu_stcs.so
CS_LIB_PATH=$PWD/tools/libcountgpu_stcs.so OUT=$O/ncu tools/ncu_traffic.sh cfg2 --no-dropin
python tools/ncu_step_traffic.py $O/ncu/cfg2_launches.csv cfg2 | tail -3
CS_LIB_PATH=$PWD/tools/libcountgpu_stcs.so python bench.py --config cfg3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3 stcs', d['ms_per_step'], d['e2e']['ms_per_step'])"
