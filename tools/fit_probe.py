"""Full-optimisation wall time through the public fit() on the GPU engine
(optimize -> explore_grid -> latent_marginals), per config.

    python tools/fit_probe.py c1 c2 [--slots K]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402
from paper_2204_04678_b200.fit import FitConfig, fit
from paper_2204_04678_b200.objective import ObjectiveEvaluator
from paper_2204_04678_b200.optimizer import FDConfig, LineSearchConfig
from paper_2204_04678_b200.synth import make_instance

for cfg in [a for a in sys.argv[1:] if not a.startswith("--")]:
    inst = make_instance(cfg)
    t0 = time.perf_counter()
    ev = ObjectiveEvaluator(inst.spec, inst.y)
    t1 = time.perf_counter()
    fc = FitConfig(fd=FDConfig("central"), line_search=LineSearchConfig(candidates=6))
    clk = ClockSampler(0).start()
    res = fit(inst.spec, inst.y, fc, evaluator=ev)
    t2 = time.perf_counter()
    clocks = clk.stop()
    s = res.summary()
    st = ev.engine.stats()
    print(json.dumps({"config": cfg, "n": inst.n, "m": inst.spec.m, "create_s": t1 - t0,
                      "fit_s": t2 - t1, "total_s": t2 - t0, "theta_mode": s["theta_mode"],
                      "theta_true": inst.theta_true.tolist(), "f_mode": s["f_mode"],
                      "iterations": s["iterations"], "n_fn_evals": s["n_fn_evals"],
                      "status": s["status"], "kernel_launches": st["kernel_launches"],
                      "phases": ev.engine.phase_times(), "slots": st["slots"],
                      "clocks": clocks}), flush=True)
    ev.close()
