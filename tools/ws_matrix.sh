#!/bin/bash
# factor kernel A/B matrix: config x resident slots x kernel (0 = 128-thread, 2 = WS forced)
for cfg in c3 c4 c5; do
  for slots in 1 3; do
    for w in 0 2; do
      echo "== $cfg slots $slots ws $w"; PINLA_VERBOSE=1 PINLA_FACTOR_WS=$w timeout 900 python tools/big_probe.py $cfg "{}" x $slots 2>&1 | grep -o "critical path.*\|factor_ms=.*TF/s (executed flops)" | tail -2
    done
  done
done
