#!/bin/bash
# c5 selected-inversion tuning sweep (one process per setting) + one traced run
# usage: bash tools/sel_sweep.sh > gpurun_out/sel_sweep.txt
CMD='python tools/prof_case.py c5 {} 1 1 selinv'
run() { echo "== $1"; env $1 $CMD 2>&1 | grep -E "selinv|rep 0"; }
run "PINLA_NONE=1"
run "PINLA_SEL_GROUP=2"
run "PINLA_SEL_GROUP=8"
run "PINLA_SEL_CHUNK_MODE=0"
run "PINLA_SELINV_NOCONT=1"
run "PINLA_SELINV_SCHED=s"
echo "== trace"
PINLA_TRACE_SELINV=gpurun_out/sel_c5.bin $CMD 2>&1 | grep selinv
python tools/sel_trace.py gpurun_out/sel_c5.bin
rm -f gpurun_out/sel_c5.bin
