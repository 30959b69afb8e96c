#!/bin/bash
# quick check of a factor-kernel change: GPU tests, then factor TF/s on the big configs, then the timeline
mkdir -p gpurun_out
OUT=gpurun_out/quick_ab.txt
: > $OUT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/quick_pytest.log 2>&1
echo "pytest exit $?: $(tail -1 gpurun_out/quick_pytest.log)" | tee -a $OUT
for cs in ${CASES:-c4,3 c3,3 c5,3 c4,1}; do
  c=${cs%,*}; n=${cs#*,}
  r=$(timeout 400 python tools/big_probe.py $c "{}" x $n 2>&1 | grep -o "f=[0-9.]* .*factor_ms=.*TF/s (executed flops)" | tail -1)
  echo "$c x$n: $r" | tee -a $OUT
done
for c in ${SELCASES:-c4 c5 c3}; do
  r=$(timeout 400 python tools/big_probe.py $c "{}" selinv 2>&1 | grep -o "selinv_ms=.*TF/s var[^ ]* *[^ ]* [^ ]*" | tail -1)
  echo "$c selinv: $r" | tee -a $OUT
  r=$(PINLA_SELINV_CONT=0 timeout 400 python tools/big_probe.py $c "{}" selinv 2>&1 | grep -o "selinv_ms=.*TF/s var[^ ]* *[^ ]* [^ ]*" | tail -1)
  echo "$c selinv (continuations off): $r" | tee -a $OUT
done
bash tools/ws_timeline.sh
