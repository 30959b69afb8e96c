#!/bin/bash
# A/B of two builds of libpinla.so on the big configs: the in-tree build vs tools/ab/$1
# usage: bash tools/lib_ab.sh libpinla_x0.so "c4,3 c3,3 c5,3 c4,1"
ALT=$1
mkdir -p gpurun_out
OUT=gpurun_out/lib_ab.txt
: > $OUT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lib_ab_pytest.log 2>&1
echo "pytest (in-tree build) exit $?: $(tail -1 gpurun_out/lib_ab_pytest.log)" | tee -a $OUT
cp paper_2204_04678_b200/libpinla.so /tmp/libpinla_main.so
for v in main alt main alt; do
  if [ $v = alt ]; then cp tools/ab/$ALT paper_2204_04678_b200/libpinla.so; else cp /tmp/libpinla_main.so paper_2204_04678_b200/libpinla.so; fi
  for cs in ${2:-c4,3 c3,3 c5,3 c4,1}; do
    c=${cs%,*}; n=${cs#*,}
    r=$(timeout 400 python tools/big_probe.py $c "{}" x $n 2>&1 | grep -o "f=[0-9.]* .*factor_ms=.*TF/s (executed flops)" | tail -1)
    echo "$v $c x$n: $r" | tee -a $OUT
  done
done
cp /tmp/libpinla_main.so paper_2204_04678_b200/libpinla.so
