#!/bin/bash
# claim-order locality sweep on full c4 x 3: PINLA_FACTOR_LOCALITY="R,C" (rows per band, columns per block; unset = bottom level only);
# factor TF/s and the DRAM bytes of the launch (single-pass ncu counters)
mkdir -p gpurun_out
OUT=gpurun_out/locality_sweep.txt
: > $OUT
for rc in ${COMBOS:-off 4,4 8,8 2,8 8,2 16,16}; do
  if [ $rc = off ]; then unset PINLA_FACTOR_LOCALITY; else export PINLA_FACTOR_LOCALITY=$rc; fi
  r=$(timeout 400 python tools/big_probe.py c4 "{}" x 3 2>&1 | grep -o "factor_ms=.*TF/s (executed flops)" | tail -1)
  timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:factor_ws_kernel -s 1 -c 1 --csv \
    --log-file /tmp/loc_dram.csv python tools/big_probe.py c4 '{}' x 3 > /dev/null 2>&1
  d=$(grep -o "dram__bytes_read.sum\",\"byte\",\"[0-9]*" /tmp/loc_dram.csv | grep -o "[0-9]*$")
  echo "locality $rc: $r; dram read bytes per launch $d" | tee -a $OUT
done
