"""Compare orderings by their tile structure (host only)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.ordering import choose_order, conditional_graph
from paper_2204_04678_b200.model import build_design
from paper_2204_04678_b200 import _lib
import scipy.sparse as sp

cfg = sys.argv[1]
import json
over = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
inst = make_instance(cfg, **over)
spec = inst.spec
A = build_design(spec)
plan = spec._prior_plan
G = conditional_graph(spec, A, plan.indptr, plan.indices)
L = sp.tril(G).tocsc(); L.sort_indices()
for ordering in sys.argv[3:] or ["band", "structured"]:
    t0 = time.time()
    perm, nd, b = choose_order(spec, A, plan.indptr, plan.indices, ordering)
    t1 = time.time()
    info = _lib.analyze_pattern(L.indptr, L.indices, perm, nd, b)
    t2 = time.time()
    print(ordering, f"order {t1-t0:.2f}s analyze {t2-t1:.2f}s", {k: (f"{v:.3e}" if v > 1e6 else v) for k, v in info.items()})
