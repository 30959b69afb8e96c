"""Full-size probe: create + one f(theta) (+ optional selinv) for a big config."""
import sys, time, json, resource
import numpy as np
sys.path.insert(0, ".")
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.objective import ObjectiveEvaluator

cfg = sys.argv[1]
over = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
do_selinv = len(sys.argv) > 3 and sys.argv[3] == "selinv"
t0 = time.time(); inst = make_instance(cfg, **over); t1 = time.time()
print(f"{cfg} n={inst.n} m={inst.spec.m} gen {t1-t0:.1f}s", flush=True)
ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=1)
t2 = time.time()
st = ev.engine.stats()
print(f"create {t2-t1:.1f}s (engine analyze {st['analyze_s']:.1f}s) device {st['device_bytes']/1e9:.1f} GB tiles {st['n_tiles']} NT {st['n_tile_rows']} factor_flops {st['factor_flops']:.3e} host maxrss {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss/1e6:.1f} GB", flush=True)
for rep in range(2):
    ev.engine.reset_stats()
    t3 = time.time(); r = ev.engine.eval_batch(np.array([inst.theta_true]), want_modes=False); t4 = time.time()
    s = ev.engine.stats()
    ph = ev.engine.phase_times()
    print(f"eval {t4-t3:.3f}s f={r['f'][0]:.6f} status={r['status'][0]} iters={r['iters'][0]} factor_ms={s['factor_ms']:.1f} ({s['factor_launches']} launches) solve_ms={s['solve_ms']:.1f} -> {st['factor_flops']*s['factor_slot_runs']/(s['factor_ms']*1e-3)/1e12:.2f} TF/s (dense-tile flops); "
          f"solve {st['solve_bytes']*s['n_solves']/(s['solve_ms']*1e-3)/1e9:.0f} GB/s ({st['solve_bytes']/1e9:.1f} GB per solve); assemble_ms={ph['assemble_ms']:.2f} other_ms={ph['other_ms']:.2f} nnz_cond={st['nnz_cond']}", flush=True)
if do_selinv:
    t5 = time.time(); var, _ = ev.marginal_variances(inst.theta_true); t6 = time.time()
    s = ev.engine.stats()
    print(f"selinv+mode {t6-t5:.2f}s selinv_ms={s['selinv_ms']:.1f} -> {st['selinv_flops']/(s['selinv_ms']*1e-3)/1e12:.2f} TF/s var[:3]={var[:3]}", flush=True)
