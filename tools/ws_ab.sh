#!/bin/bash
# A/B of the warp-specialised factor kernel (PINLA_FACTOR_WS=1, default) vs the
# 128-thread kernel (=0): GPU tests first, then factor times on c2/c3/c4/c5.
mkdir -p gpurun_out
STAGES=${1:-"tests c2 c3 c4 c5"}
for s in $STAGES; do
  case $s in
    tests)
      timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ws_pytest.log 2>&1
      echo "pytest(ws) exit $?"; tail -3 gpurun_out/ws_pytest.log;;
    c2)
      for w in 0 1; do
        PINLA_FACTOR_WS=$w timeout 600 python bench.py --config c2 --no-cpu-baseline --no-c5-selinv --steps 10 > gpurun_out/ws_c2_$w.log 2>&1
        echo "c2 ws=$w exit $?"; tail -1 gpurun_out/ws_c2_$w.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['ms_per_launch'], d['roofline']['achieved'], d.get('f_at_theta'))"
      done;;
    c3|c4|c5)
      for w in 0 1; do
        PINLA_FACTOR_WS=$w timeout 900 python tools/big_probe.py $s "{}" > gpurun_out/ws_${s}_$w.log 2>&1
        echo "$s ws=$w exit $?"; grep -o "f=[0-9.]* .*TF/s (executed flops)" gpurun_out/ws_${s}_$w.log
      done;;
  esac
done
