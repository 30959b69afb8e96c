mkdir -p gpurun_out
for c in c4 c5; do
PINLA_VERBOSE=1 timeout 600 python -c "
import sys,time; sys.path.insert(0,'.')
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.objective import ObjectiveEvaluator
t=time.time(); inst=make_instance('$c'); print('gen',time.time()-t,flush=True)
t=time.time(); ev=ObjectiveEvaluator(inst.spec, inst.y); print('create',time.time()-t, flush=True)
" > gpurun_out/create_$c.log 2>&1
echo "$c exit $?"
done
nproc; lscpu | grep -i "model name\|^CPU(s)\|Thread\|Core"
