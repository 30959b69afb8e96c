"""Small driver for ncu captures: one config (with overrides), `slots`
theta slots, `reps` eval_batch calls at theta_true (+ optional selinv).

    python tools/prof_case.py c4 '{"nt": 16, "m": 128000}' 1 2 [selinv]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2204_04678_b200.objective import ObjectiveEvaluator  # noqa: E402
from paper_2204_04678_b200.synth import make_instance  # noqa: E402

cfg = sys.argv[1]
over = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
slots = int(sys.argv[3]) if len(sys.argv) > 3 else 1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
do_sel = len(sys.argv) > 5 and sys.argv[5] == "selinv"
inst = make_instance(cfg, **over)
ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=slots)
st = ev.engine.stats()
th = np.array([inst.theta_true] * st["slots"])
for r in range(reps):
    ev.engine.reset_stats()
    t0 = time.time()
    res = ev.engine.eval_batch(th)
    s = ev.engine.stats()
    print(f"rep {r}: {time.time()-t0:.3f}s f={res['f'][0]:.6f} iters={res['iters'].tolist()} "
          f"factor {s['factor_ms']:.2f} ms/{s['factor_launches']} launches "
          f"({st['factor_flops_limited']*s['factor_slot_runs']/(s['factor_ms']*1e-3)/1e12:.2f} TF/s exec), "
          f"solve kernel {s['solve_kernel_ms']:.2f} ms "
          f"({st['solve_bytes']*s['solve_slot_runs']/(s['solve_kernel_ms']*1e-3)/1e9:.0f} GB/s)", flush=True)
if do_sel:
    ev.engine.reset_stats()
    var, _ = ev.marginal_variances(inst.theta_true)
    s = ev.engine.stats()
    print(f"selinv {s['selinv_ms']:.2f} ms ({st['selinv_flops']/(s['selinv_ms']*1e-3)/1e12:.2f} TF/s)")
