#!/bin/bash
# selected-inversion run-group size sweep on c5 / c4-shaped instances + the
# factor with smem-staged pair lists (bash tools/sel_sweep2.sh)
for cfg in 'c5 {}' 'c4 {"nt":64,"m":512000}'; do
  set -- $cfg
  for g in 8 4 3 2; do
    echo "== $1 $2 PINLA_SEL_RUN_GROUP=$g"
    PINLA_SEL_RUN_GROUP=$g python tools/prof_case.py $1 "$2" 1 1 selinv 2>&1 | grep -E "selinv|rep 0"
  done
done
