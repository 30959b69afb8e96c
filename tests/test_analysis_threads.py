"""The host build/analysis runs its per-column / per-task loops on host
threads (analysis.hpp par_for); every index writes its own outputs, so the
tile analysis must not depend on the thread count (PINLA_BUILD_THREADS)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, sys
import numpy as np
import scipy.sparse as sp
sys.path.insert(0, ROOT)
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.ordering import choose_order, conditional_graph
from paper_2204_04678_b200.model import build_design
from paper_2204_04678_b200 import _lib
out = {}
for cfg, over in (("c2", dict()), ("c3", dict(nt=8, m=80000))):
    inst = make_instance(cfg, **over)
    spec = inst.spec
    A = build_design(spec)
    plan = spec._prior_plan
    G = conditional_graph(spec, A, plan.indptr, plan.indices)
    L = sp.tril(G).tocsc(); L.sort_indices()
    perm, nd, b = choose_order(spec, A, plan.indptr, plan.indices, "structured")
    info = _lib.analyze_pattern(L.indptr, L.indices, perm, nd, b, want_tiles=True)
    rows, cols = info.pop("tile_rows"), info.pop("tile_cols")
    out[cfg] = dict(info={k: float(v) for k, v in info.items()},
                    tiles=[int(np.asarray(rows, np.int64) @ np.arange(len(rows))),
                           int(np.asarray(cols, np.int64) @ np.arange(len(cols)))])
print(json.dumps(out))
""".replace("ROOT", repr(ROOT))


def _run(threads):
    env = dict(os.environ, PINLA_BUILD_THREADS=str(threads))
    r = subprocess.run([sys.executable, "-c", PROBE], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_analysis_independent_of_build_threads():
    one, many = _run(1), _run(8)
    assert one == many
