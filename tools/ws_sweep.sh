#!/bin/bash
# WS factor kernel: chunk-cap sweep on c3 / c4
for cfg in c3 c4; do
  for cap in 16 32 64; do
    echo "== $cfg cap $cap"; PINLA_CHUNK_CAP=$cap timeout 900 python tools/big_probe.py $cfg "{}" 2>&1 | grep -o "factor_ms=.*TF/s (executed flops)" | tail -1
  done
done
