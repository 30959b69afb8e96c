# larger-config evidence: full fits (c1, c2, c3) and one f + selinv at c5
mkdir -p gpurun_out
timeout 1500 python tools/fit_probe.py c1 c2 c3 > gpurun_out/fit_probe_r01.log 2>&1; echo "fit $?"
timeout 900 python tools/big_probe.py c5 "{}" selinv > gpurun_out/c5_probe_r01.log 2>&1; echo "c5 $?"
