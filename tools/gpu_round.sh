#!/bin/bash
# One GPU-box pass: smoke, GPU tests, bench (both arms), ncu launch list and a
# full ncu capture of one 3-slot factor_ws_kernel launch of the c4 bench.  Outputs in gpurun_out/.
# usage (from this container):
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [tag] [stages]'
TAG=${1:-r01}
STAGES=${2:-"smoke tests bench ref launches full"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
for s in $STAGES; do
  case $s in
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
      echo "smoke exit $?";;
    tests)
      timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
      echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu_$TAG.log;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1
      echo "bench exit $?"; tail -1 gpurun_out/bench_$TAG.log;;
    ref)
      timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1
      echo "ref exit $?"; tail -1 gpurun_out/bench_ref_$TAG.log;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
        > gpurun_out/ncu_launch_$TAG.log 2>&1
      echo "launches exit $?";;
    full)
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:factor_ws_kernel -s 2 -c 1 \
        -f -o gpurun_out/factor_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
        > gpurun_out/ncu_full_$TAG.log 2>&1
      echo "full exit $?";;
    fullsel)
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 6 -c 1 \
        -f -o gpurun_out/solve_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
        > gpurun_out/ncu_fullsolve_$TAG.log 2>&1
      echo "fullsolve exit $?";;
    fullws)
      # --set full of one warp-specialised factor launch (3 slots) and one selected-inversion launch on
      # the c4 block shape (64x64 grid, n_t = 16): replays need the kernel's state saved, so not full c4
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:factor_ws_kernel -s 1 -c 1 \
        -f -o gpurun_out/factorws_$TAG python tools/prof_case.py c4 '{"nt": 16, "m": 128000}' 3 2 \
        > gpurun_out/ncu_factorws_$TAG.log 2>&1
      echo "fullws factor exit $?"
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:selinv_ws_kernel -c 1 \
        -f -o gpurun_out/selinvws_$TAG python tools/prof_case.py c4 '{"nt": 16, "m": 128000}' 1 1 selinv \
        > gpurun_out/ncu_selinvws_$TAG.log 2>&1
      echo "fullws selinv exit $?";;
    factordram)
      # DRAM bytes of one full-size c4 3-slot factor launch (single-pass metrics, no replay)
      timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -k regex:factor_ws_kernel -s 1 -c 1 --csv --log-file gpurun_out/factor_dram_c4_$TAG.csv \
        python tools/big_probe.py c4 '{}' x 3 > gpurun_out/ncu_factordram_$TAG.log 2>&1
      echo "factordram exit $?";;
    probes)
      for c in c4 c5; do
        timeout 900 python tools/big_probe.py $c "{}" selinv > gpurun_out/${c}_probe_$TAG.txt 2>&1
        echo "probe $c exit $?"; tail -2 gpurun_out/${c}_probe_$TAG.txt
        timeout 900 python tools/big_probe.py $c "{}" x 3 > gpurun_out/${c}_probe3_$TAG.txt 2>&1
        echo "probe3 $c exit $?"; tail -1 gpurun_out/${c}_probe3_$TAG.txt
      done;;
    solvedram)
      # DRAM bytes of one c4 solve launch (single-pass metrics: no replay of the 80 GB state)
      timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -k regex:solve_kernel -c 1 --csv --log-file gpurun_out/solve_dram_c4_$TAG.csv \
        python tools/big_probe.py c4 > gpurun_out/ncu_solvedram_$TAG.log 2>&1
      echo "solvedram exit $?";;
  esac
done
# traces (not timed): single-slot and 5-slot factor launch of c2
if [[ " $STAGES " == *" trace "* ]]; then
  PINLA_TRACE=gpurun_out/trace1_$TAG.bin timeout 600 python tools/trace1.py c2 > gpurun_out/trace1_$TAG.log 2>&1
  PINLA_TRACE=gpurun_out/trace5_$TAG.bin timeout 600 python tools/trace_batch.py c2 > gpurun_out/trace5_$TAG.log 2>&1
  echo "trace exit $?"
fi
if [[ " $STAGES " == *" strace "* ]]; then
  PINLA_TRACE_SOLVE=gpurun_out/strace_c3_$TAG.bin timeout 900 python tools/big_probe.py c3 > gpurun_out/strace_c3_$TAG.log 2>&1
  PINLA_TRACE_SOLVE=gpurun_out/strace_c2_$TAG.bin timeout 600 python tools/trace_batch.py c2 > gpurun_out/strace_c2_$TAG.log 2>&1
  echo "strace exit $?"
fi
