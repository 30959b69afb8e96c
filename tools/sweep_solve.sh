#!/bin/bash
# c2 solve/factor phase times under the solve tuning switches (tuning only)
mkdir -p gpurun_out
out=gpurun_out/sweep_solve.txt; : > $out
for s in "" "PINLA_SOLVE_LINKS=0" "PINLA_SOLVE_LINKS=1" "PINLA_SOLVE_LINKS=2" \
         "PINLA_SOLVE_GROUP=1" "PINLA_SOLVE_GROUP=4" "PINLA_SOLVE_GROUP=8" "PINLA_SOLVE_GROUP=16" \
         "PINLA_SOLVE_GROUP=32" "PINLA_SOLVE_GROUP=64"; do
  echo "== ${s:-default}" >> $out
  env $s timeout 300 python tools/perf_probe.py c2 2>&1 | grep -E "batch of|phases" | tail -2 >> $out
done
