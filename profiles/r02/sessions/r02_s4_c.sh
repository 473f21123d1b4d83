#!/bin/bash
# round 2 session 4: ncu --set full of single cfg5 classes (after each ran clean without ncu)
O=gpurun_out/s4c; mkdir -p $O
run() {  # name k lo hi regex
  python tools/cfg5_one.py $2 $3 $4 12 > $O/$1.txt 2>&1 || return
  ncu --set full --clock-control none --import-source on -k "regex:$5" --launch-skip 1 -c 1 -o $O/$1 -f \
      python tools/cfg5_one.py $2 $3 $4 12 > $O/$1.ncu.log 2>&1
}
run k2_pack 2 0 41 k_hist
run k5_small 5 41 1760 k_hist
run k7_rows 7 28160 56320 k_hist
run k7_narrow16 7 56320 112640 k_hist
run k8_narrow8 8 112640 225280 k_hist
run k8_part 8 450560 901120 k_radix_part
run k8_count 8 450560 901120 k_radix_count
ls -la $O
