#!/bin/bash
# A/B of the software-pipelined fragment loads in the warp-specialised MMA loops
# (PINLA_WS_PREFETCH, compile-time): tools/ab/libpinla_pf0.so is the build without it.
mkdir -p gpurun_out
OUT=gpurun_out/pf_ab.txt
: > $OUT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pf_pytest.log 2>&1
echo "pytest (prefetch build) exit $?: $(tail -1 gpurun_out/pf_pytest.log)" | tee -a $OUT
cp paper_2204_04678_b200/libpinla.so /tmp/libpinla_pf1.so
for v in pf1 pf0; do
  if [ $v = pf0 ]; then cp tools/ab/libpinla_pf0.so paper_2204_04678_b200/libpinla.so; else cp /tmp/libpinla_pf1.so paper_2204_04678_b200/libpinla.so; fi
  for cfg in c4 c5; do
    r=$(timeout 400 python tools/big_probe.py $cfg "{}" x 3 2>&1 | grep -o "f=[0-9.]* .*factor_ms=.*TF/s (executed flops)" | tail -1)
    echo "$v $cfg x3: $r" | tee -a $OUT
    r=$(timeout 400 python tools/big_probe.py $cfg "{}" selinv 2>&1 | grep -o "selinv_ms=.*TF/s var[^ ]* *[^ ]* [^ ]*" | tail -1)
    echo "$v $cfg selinv: $r" | tee -a $OUT
  done
done
cp /tmp/libpinla_pf1.so paper_2204_04678_b200/libpinla.so
