#!/bin/bash
# factor/solve poll back-off threshold sweep (rebuilds libpinla.so on the box; tuning only)
mkdir -p gpurun_out
out=gpurun_out/sweep_spin.txt; : > $out
for N in 4 1000000 0 32; do
  make -s -B -C paper_2204_04678_b200/csrc EXTRA=-DPINLA_SPIN_SLEEP_AFTER=$N > /dev/null 2>&1
  for c in c2 c3; do
    echo "== spin $N $c" >> $out
    timeout 400 python tools/perf_probe.py $c 2>&1 | grep -E "batch of|factor:" | tail -2 >> $out
  done
done
