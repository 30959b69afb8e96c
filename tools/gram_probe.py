import sys, numpy as np
sys.path.insert(0, ".")
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.objective import ObjectiveEvaluator
inst = make_instance("c5", nt=60, m=480000)
ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=1)
r = ev.engine.eval_batch(np.array([inst.theta_true]), want_modes=False)
print("f", r["f"][0])
