#!/bin/bash
# A/B of two builds on selected inversion: in-tree vs tools/ab/$1
ALT=$1
mkdir -p gpurun_out
OUT=gpurun_out/sel_ab.txt
: > $OUT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/sel_ab_pytest.log 2>&1
echo "pytest (in-tree build) exit $?: $(tail -1 gpurun_out/sel_ab_pytest.log)" | tee -a $OUT
cp paper_2204_04678_b200/libpinla.so /tmp/libpinla_main.so
for v in main alt main alt; do
  if [ $v = alt ]; then cp tools/ab/$ALT paper_2204_04678_b200/libpinla.so; else cp /tmp/libpinla_main.so paper_2204_04678_b200/libpinla.so; fi
  for c in c4 c5 c3; do
    r=$(timeout 400 python tools/big_probe.py $c "{}" selinv 2>&1 | grep -o "selinv_ms=.*TF/s var[^ ]* *[^ ]* [^ ]*" | tail -1)
    echo "$v $c selinv: $r" | tee -a $OUT
  done
done
cp /tmp/libpinla_main.so paper_2204_04678_b200/libpinla.so
