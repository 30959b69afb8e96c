#!/bin/bash
# A/B of the task-slot ring depth of the warp-specialised factor kernel (PINLA_WS_SLOTS, compile-time)
mkdir -p gpurun_out
OUT=gpurun_out/slots_ab.txt
: > $OUT
cp paper_2204_04678_b200/libpinla.so /tmp/libpinla_main.so
for v in main s3 s4 main s3; do
  if [ $v = main ]; then cp /tmp/libpinla_main.so paper_2204_04678_b200/libpinla.so; else cp tools/ab/libpinla_$v.so paper_2204_04678_b200/libpinla.so; fi
  for cs in c4,3 c5,3 c4,1 c3,1; do
    c=${cs%,*}; n=${cs#*,}
    r=$(timeout 400 python tools/big_probe.py $c "{}" x $n 2>&1 | grep -o "f=[0-9.]* .*factor_ms=.*TF/s (executed flops)" | tail -1)
    echo "$v $c x$n: $r" | tee -a $OUT
  done
done
cp /tmp/libpinla_main.so paper_2204_04678_b200/libpinla.so
# functional check of the multi-rank bench path: two ranks on this one GPU over gloo (numbers meaningless)
PINLA_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-c5-selinv > gpurun_out/bench_2rank_shared.log 2>&1
echo "2-rank shared-GPU bench exit $?"; tail -1 gpurun_out/bench_2rank_shared.log | cut -c1-300
