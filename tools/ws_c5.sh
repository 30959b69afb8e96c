#!/bin/bash
# c5 (chain-bound, critical lane) sensitivity of the WS factor kernel
mkdir -p gpurun_out
OV='{"nt": 80, "m": 640000}'
run() { echo "== $*"; env "$@" timeout 600 python tools/prof_case.py c5 "$OV" 1 2 2>&1 | tail -1; }
run PINLA_FACTOR_WS=0
run PINLA_FACTOR_WS=1
run PINLA_FACTOR_WS=1 PINLA_LANE_CTAS=4
run PINLA_FACTOR_WS=1 PINLA_LANE_CTAS=12
run PINLA_FACTOR_WS=1 PINLA_FACTOR_LANE=0
run PINLA_FACTOR_WS=0 PINLA_FACTOR_LANE=0
