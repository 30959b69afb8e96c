#!/bin/bash
# factor task traces (old vs WS kernel): c5 reduced (chain-bound) and c2
mkdir -p gpurun_out
OV='{"nt": 40, "m": 320000}'
for w in 0 1; do
  PINLA_FACTOR_WS=$w PINLA_TRACE=gpurun_out/tr_c5_$w.bin timeout 600 python tools/prof_case.py c5 "$OV" 1 1 > gpurun_out/tr_c5_$w.log 2>&1
  python tools/trace_analyze.py gpurun_out/tr_c5_$w.bin > gpurun_out/tr_c5_$w.txt 2>&1
  PINLA_FACTOR_WS=$w PINLA_TRACE=gpurun_out/tr_c2_$w.bin timeout 600 python tools/trace_batch.py c2 > gpurun_out/tr_c2_$w.log 2>&1
  python tools/trace_analyze.py gpurun_out/tr_c2_$w.bin > gpurun_out/tr_c2_$w.txt 2>&1
  rm -f gpurun_out/tr_c5_$w.bin gpurun_out/tr_c2_$w.bin
done
