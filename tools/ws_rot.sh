#!/bin/bash
OV='{"nt": 80, "m": 640000}'
echo "== rot 96 (default)"; PINLA_FACTOR_WS=1 timeout 600 python tools/prof_case.py c5 "$OV" 1 2 2>&1 | tail -1
cp paper_2204_04678_b200/libpinla.so /tmp/lib_def.so; cp gpurun_in_rot0.so paper_2204_04678_b200/libpinla.so
echo "== rot 0"; PINLA_FACTOR_WS=1 timeout 600 python tools/prof_case.py c5 "$OV" 1 2 2>&1 | tail -1
cp /tmp/lib_def.so paper_2204_04678_b200/libpinla.so
