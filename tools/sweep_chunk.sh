mkdir -p gpurun_out
for m in 0 1 2 3; do
  PINLA_CHUNK_MODE=$m timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/sweep_chunk$m.log 2>&1
  echo "mode $m: $(tail -1 gpurun_out/sweep_chunk$m.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["phases_ms_per_step"])')"
done
