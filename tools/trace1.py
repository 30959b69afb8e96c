"""Trace one single-slot factor launch of c2 (PINLA_TRACE set by the caller)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.objective import ObjectiveEvaluator
inst = make_instance(sys.argv[1] if len(sys.argv) > 1 else "c2")
ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=1)
r = ev.engine.eval_batch(np.array([inst.theta_true]), want_modes=False)
print("f", r["f"][0], ev.engine.stats()["factor_ms"])
