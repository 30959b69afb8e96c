#!/bin/bash
# consumer timeline of one 3-slot warp-specialised factor launch on the c4 block shape (n_t = 16)
mkdir -p gpurun_out
OV='{"nt": 16, "m": 128000}'
for mc in ${COMBOS:-"3,16"}; do
  m=${mc%,*}; c=${mc#*,}
  PINLA_CHUNK_MODE=$m PINLA_CHUNK_CAP=$c PINLA_TRACE=/tmp/tr_ws.bin timeout 600 python tools/prof_case.py c4 "$OV" 3 2 > gpurun_out/ws_timeline_${m}_${c}.txt 2>&1
  python tools/ws_timeline.py /tmp/tr_ws.bin ${RINGWAIT:+ringwait} >> gpurun_out/ws_timeline_${m}_${c}.txt 2>&1
  rm -f /tmp/tr_ws.bin
  echo "== mode $m cap $c"; tail -14 gpurun_out/ws_timeline_${m}_${c}.txt
done
