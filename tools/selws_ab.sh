#!/bin/bash
# selected-inversion kernel A/B (PINLA_SELINV_WS=0: 128-thread FIFO kernel, 2: warp-specialised forced)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/selws_pytest.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/selws_pytest.log
for cfg in c3 c4 c5; do
  for w in 0 2; do
    echo "== $cfg selinv ws $w"; PINLA_SELINV_WS=$w timeout 300 python tools/big_probe.py $cfg "{}" selinv 2>&1 | grep -o "selinv_ms=.*TF/s var[^ ]* *[^ ]* [^ ]*"
  done
done
echo "== c4 3 slots factor"; timeout 300 python tools/big_probe.py c4 "{}" x 3 2>&1 | grep -o "factor_ms=.*TF/s (executed flops)" | tail -1
