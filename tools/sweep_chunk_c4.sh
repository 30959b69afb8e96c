#!/bin/bash
# factor chunk-size sweep on full c4, 3 resident slots (throughput-bound DAG, warp-specialised kernel)
# and on c5 x 3; PINLA_CHUNK_MODE / PINLA_CHUNK_CAP are analysis.cpp tuning switches
mkdir -p gpurun_out
OUT=gpurun_out/chunk_sweep_c4.txt
touch $OUT
for cfg in ${CFGS:-c4}; do
for mc in ${COMBOS:-"3,16 3,32 4,16 4,32 2,16 2,32"}; do
  m=${mc%,*}; c=${mc#*,}
  r=$(PINLA_CHUNK_MODE=$m PINLA_CHUNK_CAP=$c timeout 400 python tools/big_probe.py $cfg "{}" x ${SLOTS:-3} 2>&1 | grep -o "f=[0-9.]* .*factor_ms=.*TF/s (executed flops)" | tail -1)
  echo "$cfg x${SLOTS:-3} mode $m cap $c: $r" | tee -a $OUT
done
done
