"""Trace the first all-slots-active factor launch of a c2 FD batch
(PINLA_TRACE=<file> set by the caller); analyze with tools/trace_analyze.py."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.objective import ObjectiveEvaluator
inst = make_instance(sys.argv[1] if len(sys.argv) > 1 else "c2")
d = inst.theta_true.size
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2 * d + 1
ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=k)
x, its, st, _, _ = ev.engine.mode(inst.theta_true)
pts = [inst.theta_true] + [inst.theta_true + s * 5e-3 * np.eye(d)[i] for i in range(d) for s in (1, -1)]
r = ev.engine.eval_batch(np.array(pts[:k]), warm=x)
print("iters", r["iters"].tolist(), ev.engine.stats()["factor_ms"])
