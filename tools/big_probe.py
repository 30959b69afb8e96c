"""Full-size probe: create + one f(theta) (+ optional selinv) for a big config,
with nvidia-smi clocks sampled over each timed call (bench.ClockSampler).

    python tools/big_probe.py c5 '{}' selinv [slots]
"""
import json
import resource
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402
from paper_2204_04678_b200.objective import ObjectiveEvaluator  # noqa: E402
from paper_2204_04678_b200.synth import make_instance  # noqa: E402

cfg = sys.argv[1]
over = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
do_selinv = len(sys.argv) > 3 and sys.argv[3] == "selinv"
slots = int(sys.argv[4]) if len(sys.argv) > 4 else 1
t0 = time.time()
inst = make_instance(cfg, **over)
t1 = time.time()
print(f"{cfg} n={inst.n} m={inst.spec.m} gen {t1-t0:.1f}s", flush=True)
ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=slots)
t2 = time.time()
st = ev.engine.stats()
print(f"create {t2-t1:.1f}s (engine analyze {st['analyze_s']:.1f}s) slots {st['slots']} device "
      f"{st['device_bytes']/1e9:.1f} GB tiles {st['n_tiles']} NT {st['n_tile_rows']} factor_flops "
      f"{st['factor_flops']:.3e} exec {st['factor_flops_limited']:.3e} host maxrss "
      f"{resource.getrusage(resource.RUSAGE_SELF).ru_maxrss/1e6:.1f} GB", flush=True)
thetas = np.array([inst.theta_true] * st["slots"])
for rep in range(2):
    ev.engine.reset_stats()
    clk = ClockSampler(0).start()
    t3 = time.time()
    r = ev.engine.eval_batch(thetas, want_modes=False)
    t4 = time.time()
    clocks = clk.stop()
    s = ev.engine.stats()
    fl = st["factor_flops_limited"] * s["factor_slot_runs"]
    print(f"eval {t4-t3:.3f}s ({len(thetas)} slots) f={r['f'][0]:.6f} status={r['status'].tolist()} "
          f"iters={r['iters'].tolist()} factor_ms={s['factor_ms']:.1f} ({s['factor_launches']} launches) "
          f"-> {fl/(s['factor_ms']*1e-3)/1e12:.2f} TF/s (executed flops); solve_kernel_ms="
          f"{s['solve_kernel_ms']:.1f} -> {st['solve_bytes']*s['solve_slot_runs']/(s['solve_kernel_ms']*1e-3)/1e9:.0f} GB/s "
          f"({st['solve_bytes']/1e9:.1f} GB per slot-solve); assemble_ms={s['assemble_ms']:.2f} "
          f"({s['assemble_bytes_done']/(s['assemble_ms']*1e-3)/1e9:.0f} GB/s); clocks {json.dumps(clocks)}",
          flush=True)
if do_selinv:
    clk = ClockSampler(0).start()
    t5 = time.time()
    var, _ = ev.marginal_variances(inst.theta_true)
    t6 = time.time()
    clocks = clk.stop()
    s = ev.engine.stats()
    print(f"selinv+mode {t6-t5:.2f}s selinv_ms={s['selinv_ms']:.1f} -> "
          f"{st['selinv_flops']/(s['selinv_ms']*1e-3)/1e12:.2f} TF/s var[:3]={var[:3]} clocks "
          f"{json.dumps(clocks)}", flush=True)
