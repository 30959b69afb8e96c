#!/bin/bash
# copy the outputs of `tools/gpu_round.sh TAG ...` from gpurun_out/ into profiles/ (round-2 names)
T=$1
tail -1 gpurun_out/bench_$T.log > profiles/bench_c4_r02.json
tail -1 gpurun_out/bench_ref_$T.log > profiles/bench_ref_c4_r02.json
python tools/ncu_summary.py shares gpurun_out/launches_$T.csv profiles/launch_shares_c4_r02.csv > /dev/null
cp gpurun_out/launches_$T.csv profiles/launches_c4_r02.csv
cp gpurun_out/factor_dram_c4_$T.csv profiles/factor_dram_c4_r02.csv
for f in c4_probe c4_probe3 c5_probe c5_probe3; do cp gpurun_out/${f}_$T.txt profiles/${f}_r02.txt; done
python tools/ncu_summary.py full gpurun_out/factorws_$T.ncu-rep profiles/factorws_ncu_c4nt16_r02.json > /dev/null
python tools/ncu_summary.py full gpurun_out/selinvws_$T.ncu-rep profiles/selinvws_ncu_c4nt16_r02.json > /dev/null
(cat gpurun_out/nvsmi_$T.txt; echo "pytest -m gpu:"; tail -1 gpurun_out/pytest_gpu_$T.log; tail -3 gpurun_out/smoke_$T.log) > profiles/gpu_tests_r02.txt
python - <<PY
import json
d = json.load(open('profiles/bench_c4_r02.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'factor TF/s', d['roofline']['achieved'], 'frac', d['roofline']['frac'],
      'traffic', d['roofline']['traffic'], 'solve frac', d['hbm_kernels']['solve_kernel']['frac'],
      'asm frac', d['hbm_kernels']['assembly']['frac'], 'selinv c4/c5', d['selinv']['c4']['selinv_s'], d['selinv']['c5']['selinv_s'],
      'clocks', d['clocks'], 'cpu', d['cpu_baseline']['value'], 'launches', d['gpu_launches'])
f = json.load(open('profiles/factorws_ncu_c4nt16_r02.json'))
print('ncu factor: tensor active', f['tensor_pipe_active_pct_elapsed'], 'dram/launch', f['dram_bytes_per_launch'], f['top_stalls_pct'])
s = json.load(open('profiles/selinvws_ncu_c4nt16_r02.json'))
print('ncu selinv: tensor active', s['tensor_pipe_active_pct_elapsed'])
PY
head -5 profiles/launch_shares_c4_r02.csv
grep -o "dram__bytes[a-z_.]*\",\"byte\",\"[0-9]*\"\|duration.sum\",\"ns\",\"[0-9]*\"" profiles/factor_dram_c4_r02.csv
