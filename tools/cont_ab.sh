#!/bin/bash
# A/B of the chunk continuations of the warp-specialised factor kernel (PINLA_FACTOR_CONT=0: off)
mkdir -p gpurun_out
OUT=gpurun_out/cont_ab.txt
: > $OUT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/cont_pytest.log 2>&1
echo "pytest exit $?: $(tail -1 gpurun_out/cont_pytest.log)" | tee -a $OUT
for v in 1 0; do
  for cs in "c4 3" "c5 3" "c3 3" "c4 1" "c3 1"; do
    set -- $cs
    r=$(PINLA_FACTOR_CONT=$v timeout 400 python tools/big_probe.py $1 "{}" x $2 2>&1 | grep -o "f=[0-9.]* .*factor_ms=.*TF/s (executed flops)" | tail -1)
    echo "cont=$v $1 x$2: $r" | tee -a $OUT
  done
done
r=$(timeout 300 python bench.py --config c2 --steps 10 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["phases_ms_per_step"])')
echo "c2 bench cont=1: $r" | tee -a $OUT
r=$(PINLA_FACTOR_CONT=0 timeout 300 python bench.py --config c2 --steps 10 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["phases_ms_per_step"])')
echo "c2 bench cont=0: $r" | tee -a $OUT
bash tools/ws_timeline.sh
