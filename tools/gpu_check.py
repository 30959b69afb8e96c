"""Quick GPU parity check against tests/golden fixtures (dev tool)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_2204_04678_b200.synth import make_instance
from paper_2204_04678_b200.objective import ObjectiveEvaluator

cases = sys.argv[1:] or ["c1", "c2r", "c3r", "c4r", "c5r"]
for case in cases:
    G = np.load(f"tests/golden/{case}.npz")
    inst = make_instance(str(G["config"]), **json.loads(str(G["overrides"])))
    t0 = time.time()
    ev = ObjectiveEvaluator(inst.spec, inst.y, inner_tol=float(G["inner_tol"]))
    t1 = time.time()
    res = ev.engine.eval_batch(G["thetas"], want_modes=True)
    t2 = time.time()
    fr = G["f_components"][:, 0]
    rel = np.abs(res["f"] - fr) / np.abs(fr)
    ldrel = np.abs(res["logdets"] - G["logdets"]) / np.abs(G["logdets"])
    moderr = np.max(np.abs(res["modes"][0] - G["mode"])) / max(1e-300, np.max(np.abs(G["mode"])))
    print(f"{case}: n={inst.n} create {t1-t0:.2f}s eval {t2-t1:.3f}s status={res['status'].tolist()} iters={res['iters'].tolist()} ref_its={G['f_components'][:,5].tolist()}")
    print(f"   f rel err max {rel.max():.3e}  logdet rel {ldrel.max():.3e}  mode rel {moderr:.3e}")
    print(f"   comps gpu {res['comps'][0]}\n   comps ref {G['f_components'][0,:5]}")
    if "variances" in G.files:
        t3 = time.time()
        var, x = ev.marginal_variances(G["thetas"][0])
        t4 = time.time()
        vr = np.max(np.abs(var - G["variances"]) / np.abs(G["variances"]))
        print(f"   selinv {t4-t3:.3f}s var rel err max {vr:.3e}")
    print("   stats", {k: v for k, v in ev.engine.stats().items()})
    ev.close()
