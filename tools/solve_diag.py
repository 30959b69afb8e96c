"""Solve-accuracy diagnostic on c2: FD stencil batch (as bench.py) -> per-slot
f, Newton iterations, launches; plus mode residual ||Q_c x - rhs|| through the
generic factorize/solve drop-ins on the conditional precision at theta_true."""
import os, sys, json
import numpy as np
sys.path.insert(0, ".")
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.engine import Engine
sys.path.insert(0, "tools")

inst = make_instance("c2")
eng = Engine(inst.spec, inst.y, max_slots=5)
theta = inst.theta_true
d = theta.size
pts = [theta.copy()]
for j in range(d):
    e = np.zeros(d); e[j] = 5e-3
    pts += [theta + e, theta - e]
pts = np.array(pts)
warm, its, st, _, _ = eng.mode(theta)
eng.reset_stats()
res = eng.eval_batch(pts, warm, want_modes=True)
s = eng.stats()
out = {"G": os.environ.get("PINLA_SOLVE_GROUP", "default"), "f": [float(v) for v in res["f"]],
       "iters": [int(v) for v in res["iters"]], "launches": int(s["kernel_launches"]),
       "mode_its": int(its)}
np.save(f"gpurun_out/diag_modes_{out['G']}.npy", res["modes"])
print(json.dumps(out))
rng = np.random.default_rng(0)
b = rng.normal(size=eng.n)
xs = [eng.solve_resident(b) for _ in range(10)]
ndiff = sum(int(np.any(x != xs[0])) for x in xs)
np.save(f"gpurun_out/diag_x_{out['G']}.npy", xs[0])
print(json.dumps({"G": out["G"], "solve_runs_differing": ndiff,
                  "max_rel_spread": float(max(np.max(np.abs(x - xs[0])) for x in xs) / np.max(np.abs(xs[0])))}))
