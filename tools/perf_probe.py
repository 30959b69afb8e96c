"""Dev perf probe: create + batched f(theta) timings on full-size configs."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.objective import ObjectiveEvaluator

cfg = sys.argv[1]
over = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
slots = int(sys.argv[3]) if len(sys.argv) > 3 else None
t0 = time.time(); inst = make_instance(cfg, **over); t1 = time.time()
ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=slots); t2 = time.time()
d = inst.theta_true.size
eps = 5e-3
pts = [inst.theta_true] + [inst.theta_true + s * eps * np.eye(d)[i] for i in range(d) for s in (1, -1)]
print(f"{cfg} n={inst.n} m={inst.spec.m} gen {t1-t0:.1f}s create {t2-t1:.1f}s", ev.engine.stats(), flush=True)
x, its, st, bc, ld = ev.engine.mode(inst.theta_true)
print("mode its", its, "status", st, flush=True)
for rep in range(3):
    ev.engine.reset_stats()
    t3 = time.time(); r = ev.engine.eval_batch(np.array(pts), warm=x); t4 = time.time()
    print(f"batch of {len(pts)}: {t4-t3:.3f}s -> {len(pts)/(t4-t3):.2f} evals/s iters {r['iters'].tolist()} status {r['status'].tolist()}", flush=True)
    st = ev.engine.stats()
    print("   phases", ev.engine.phase_times(), "launches", st["kernel_launches"], "factorizations", st["n_factorizations"], flush=True)
    print(f"   factor: {st['factor_launches']} launches, {st['factor_slot_runs']} slot-runs, {st['factor_ms']/max(1,st['factor_launches']):.3f} ms/launch, {st['factor_ms']/max(1,st['factor_slot_runs']):.3f} ms/slot-run", flush=True)
t5 = time.time(); var, _ = ev.marginal_variances(inst.theta_true, x); t6 = time.time()
print(f"selinv (incl. mode) {t6-t5:.3f}s", ev.engine.phase_times(), flush=True)
