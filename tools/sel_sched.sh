#!/bin/bash
for cfg in c4 c5; do
  for sch in f s; do
    echo "== $cfg selinv sched $sch"; PINLA_SELINV_SCHED=$sch timeout 900 python tools/big_probe.py $cfg "{}" selinv 2>&1 | grep -o "selinv_ms=.*TF/s"
  done
done
