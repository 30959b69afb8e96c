"""GPU time of f(theta) / selinv on a reference-kind model vs the ND tile
height cap (PINLA_ND_TILE_MAX), one process per setting."""
import json
import os
import subprocess
import sys

CODE = r'''
import sys, time, json
sys.path.insert(0, ".")
import numpy as np
from paper_2204_04678_b200.objective import ObjectiveEvaluator
from paper_2204_04678_b200.synth import reference_kind_instance
kind, side, m, slots = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
inst = reference_kind_instance(kind, side=side, m=m)
ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=slots)
th = np.array([inst.theta_true] * ev.engine.max_slots)
for _ in range(3):
    ev.engine.eval_batch(th)
ev.engine.reset_stats()
t0 = time.perf_counter()
for _ in range(10):
    ev.engine.eval_batch(th)
dt = (time.perf_counter() - t0) / 10
s = ev.engine.stats()
ev.engine.reset_stats()
var, _ = ev.marginal_variances(inst.theta_true)
s2 = ev.engine.stats()
print(json.dumps(dict(slots=int(s["slots"]), batch_ms=dt * 1e3, factor_ms=s["factor_ms"] / 10,
                      exec_flops=s["factor_flops_limited"], nT=s["n_tiles"], NT=s["n_tile_rows"],
                      selinv_ms=s2["selinv_ms"])))
'''
for tm in (64, 48, 32, 24):
    for slots in (1, 7):
        env = dict(os.environ, PINLA_ND_TILE_MAX=str(tm))
        out = subprocess.run([sys.executable, "-c", CODE, "leukemia-like", "63", "6174", str(slots)],
                             env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(f"tile_max {tm} slots {slots}: {line}", flush=True)
