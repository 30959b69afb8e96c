"""GPU parity against the reference (golden vectors) and the CPU oracle.

Tolerances (BASELINE.json north_star): f(theta) and log det within 1e-9
relative; marginal variances within 1e-8 relative; theta* within 1e-5
absolute.  All compute goes through libpinla.so (C-ABI)."""

import numpy as np
import pytest

from conftest import golden_instance, load_golden

pytestmark = pytest.mark.gpu

CASES = ["c1", "c2r", "c3r", "c4r", "c5r", "c3g", "c4g", "c5g"]
# c3g / c4g / c5g: the FULL BASELINE spatial grids (n_s = 3600 / 4096 / 2048,
# 57 / 64 / 32 tiles per time block) at n_t = 4: the chain-lane, fused-link,
# product-group and partial-group features of the tile DAG run at their
# real block sizes, compared with the reference itself
F_TOL = 1e-9
VAR_TOL = 1e-8


def evaluator(G, **kw):
    from paper_2204_04678_b200.objective import ObjectiveEvaluator

    inst = golden_instance(G)
    return inst, ObjectiveEvaluator(inst.spec, inst.y, inner_tol=float(G["inner_tol"]), **kw)


@pytest.mark.parametrize("case", CASES)
def test_f_logdets_mode_vs_reference(case):
    G = load_golden(case)
    inst, ev = evaluator(G)
    res = ev.engine.eval_batch(G["thetas"], want_modes=True)
    assert np.all(res["status"] == 0)
    ref = G["f_components"][:, :5]
    rel = np.abs(res["comps"] - ref) / np.maximum(1.0, np.abs(ref))
    assert rel.max() <= F_TOL, rel
    ldrel = np.abs(res["logdets"] - G["logdets"]) / np.abs(G["logdets"])
    assert ldrel.max() <= F_TOL, ldrel
    m = G["mode"]
    assert np.max(np.abs(res["modes"][0] - m)) <= 1e-7 * max(1.0, np.max(np.abs(m)))
    check_iterations(inst, G, res["iters"])
    ev.close()


def check_iterations(inst, G, iters):
    """Newton iteration counts.  Gaussian: 1, the reference's.  Poisson: the
    count is decided at the arithmetic floor, where the reference's ascent
    test compares two rounded totals (~1e4-1e6) whose true difference is
    below their rounding: a coin flip.  Even the oracle, running the same
    numpy-level rule with other summation kernels, does not reproduce it
    (grid2d: reference [7, 6, 8, 7], oracle [7, 6, 7, 7]; DESIGN s1.3).  The
    engine decides the ascent on the sum of per-term differences, so it
    never needs the extra floor iterations the reference's lottery can
    cost; asserted: at most two more iterations than the reference, with f,
    log dets and the mode at parity (checked by the caller)."""
    ref = G["f_components"][:, 5].astype(int)
    if inst.spec.family == "gaussian":
        assert np.all(np.asarray(iters) == 1) and np.all(ref == 1)
        return
    print(f"Newton iterations: engine {list(map(int, iters))} reference {list(ref)}")
    assert np.all(np.asarray(iters) <= ref + 2), (list(iters), list(ref))


@pytest.mark.parametrize("case", CASES)
def test_marginal_variances_vs_reference(case):
    G = load_golden(case)
    inst, ev = evaluator(G)
    var, mode = ev.marginal_variances(G["thetas"][0])
    ref = G["variances"]
    assert np.max(np.abs(var - ref) / ref) <= VAR_TOL
    ev.close()


def test_full_c2_vs_reference():
    G = load_golden("c2")
    inst, ev = evaluator(G)
    res = ev.engine.eval_batch(G["thetas"], want_modes=False)
    ref = G["f_components"][:, :5]
    assert np.max(np.abs(res["comps"] - ref) / np.maximum(1.0, np.abs(ref))) <= F_TOL
    var, _ = ev.marginal_variances(G["thetas"][0])
    assert np.max(np.abs(var - G["variances"]) / G["variances"]) <= VAR_TOL
    ev.close()


@pytest.mark.parametrize("cfg,over", [
    ("c1", dict(nx=13, ny=11, m=300)),           # n = 145: ragged last tile
    ("c2", dict(nx=9, ny=7, m=250)),             # poisson, tiny
    ("c3", dict(nx=7, ny=9, nt=5, m=400)),       # ST gaussian, p = 4
    ("c4", dict(nx=10, ny=10, nt=3, m=500)),     # p = 8 arrow
    ("c5", dict(nx=6, ny=5, nt=7, m=300)),       # ST poisson + temporal effect
])
def test_random_theta_vs_oracle(cfg, over):
    from oracle.oracle import OracleEvaluator
    from paper_2204_04678_b200.objective import ObjectiveEvaluator
    from paper_2204_04678_b200.synth import make_instance

    inst = make_instance(cfg, seed=3, **over)
    ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=3)
    orc = OracleEvaluator(inst.spec, inst.y)
    rng = np.random.default_rng(7)
    pts = [inst.theta_true + rng.normal(0, 0.4, inst.theta_true.size) for _ in range(7)]
    got = ev.eval_batch(pts)  # 7 points through 3 slots: chunked batches
    want = [orc.eval(p)["f"] for p in pts]
    for g, w in zip(got, want):
        assert abs(g - w) <= F_TOL * abs(w)
    var, _ = ev.marginal_variances(pts[0])
    assert np.max(np.abs(var - orc.variances(pts[0])) / orc.variances(pts[0])) <= VAR_TOL
    ev.close()


def test_deterministic_and_slot_independent():
    from paper_2204_04678_b200.objective import ObjectiveEvaluator
    from paper_2204_04678_b200.synth import make_instance

    inst = make_instance("c5", nx=8, ny=8, nt=4, m=500)
    pts = [inst.theta_true + 0.01 * k for k in range(5)]
    a = ObjectiveEvaluator(inst.spec, inst.y, max_slots=5)
    b = ObjectiveEvaluator(inst.spec, inst.y, max_slots=1)
    fa1 = a.eval_batch(pts)
    fa2 = a.eval_batch(pts)
    fb = b.eval_batch(pts)
    assert fa1 == fa2 == fb  # bitwise: fixed-order tile accumulation and reductions
    va, _ = a.marginal_variances(pts[0])
    vb, _ = b.marginal_variances(pts[0])
    assert np.array_equal(va, vb)


def test_prior_logdet_kronecker_identity_small():
    from gpu_util import prior_logdet
    from paper_2204_04678_b200.objective import ObjectiveEvaluator
    from paper_2204_04678_b200.synth import make_instance

    for cfg, over in (("c1", dict(nx=30, ny=20, m=400)), ("c3", dict(nx=12, ny=10, nt=7, m=600)),
                      ("c5", dict(nx=8, ny=6, nt=9, m=500))):
        inst = make_instance(cfg, **over)
        ev = ObjectiveEvaluator(inst.spec, inst.y, analytic_prior_logdet=False)
        res = ev.engine.eval_batch([inst.theta_true])
        want = prior_logdet(inst, inst.theta_true)
        assert abs(res["logdets"][0, 1] - want) <= 1e-11 * abs(want)
        ev.close()


@pytest.mark.parametrize("cfg,over", [("c1", dict(nx=30, ny=20, m=400)), ("c2", dict(nx=25, ny=19, m=600)),
                                      ("c4", dict(nx=12, ny=10, nt=5, m=800)),
                                      ("c5", dict(nx=8, ny=6, nt=9, m=500))])
def test_analytic_prior_logdet_equals_factorized(cfg, over):
    """The closed-form log det Q_prior (engine default for lattice / AR(1)
    models) reproduces the reference's factorized value: same f to 1e-12."""
    from paper_2204_04678_b200.objective import ObjectiveEvaluator
    from paper_2204_04678_b200.synth import make_instance

    inst = make_instance(cfg, **over)
    pts = [inst.theta_true, inst.theta_true + 0.2]
    a = ObjectiveEvaluator(inst.spec, inst.y, analytic_prior_logdet=True)
    b = ObjectiveEvaluator(inst.spec, inst.y, analytic_prior_logdet=False)
    assert a.engine.analytic_prior_logdet and not b.engine.analytic_prior_logdet
    ra, rb = a.engine.eval_batch(pts), b.engine.eval_batch(pts)
    assert np.max(np.abs(ra["logdets"][:, 1] - rb["logdets"][:, 1]) / np.abs(rb["logdets"][:, 1])) <= 1e-12
    assert np.max(np.abs(ra["f"] - rb["f"]) / np.abs(rb["f"])) <= 1e-12
    assert a.engine.stats()["n_factorizations"] < b.engine.stats()["n_factorizations"]


def test_fit_c1_theta_star_vs_reference():
    """Full quasi-Newton fit on the GPU (central FD, candidates=6 pinned on
    both sides, SURVEY s7 hard part 3) vs the reference's fit."""
    from paper_2204_04678_b200.fit import FitConfig, fit
    from paper_2204_04678_b200.optimizer import FDConfig, LineSearchConfig
    from paper_2204_04678_b200.runtime import ThreadBudget

    G = load_golden("c1")
    inst = golden_instance(G)
    res = fit(inst.spec, inst.y, FitConfig(budget=ThreadBudget(7, 1), fd=FDConfig(scheme="central"),
                                           line_search=LineSearchConfig(candidates=6)))
    assert np.max(np.abs(res.theta_mode.theta - G["fit_theta"])) <= 1e-5
    assert abs(res.f_mode - float(G["fit_f"])) <= 1e-9 * abs(float(G["fit_f"]))
    mu = G["fit_latent_mean"]
    sd = G["fit_latent_sd"]
    assert np.max(np.abs(res.marginals.latent_mean - mu)) <= 1e-6 * max(1.0, np.max(np.abs(mu)))
    assert np.max(np.abs(res.marginals.latent_sd - sd) / sd) <= 1e-6


def test_fit_c2r_poisson_theta_star_vs_reference():
    from paper_2204_04678_b200.fit import FitConfig, fit
    from paper_2204_04678_b200.optimizer import FDConfig, LineSearchConfig
    from paper_2204_04678_b200.runtime import ThreadBudget

    G = load_golden("c2r")
    inst = golden_instance(G)
    res = fit(inst.spec, inst.y, FitConfig(budget=ThreadBudget(7, 1), fd=FDConfig(scheme="central"),
                                           line_search=LineSearchConfig(candidates=6),
                                           inner_tol=float(G["inner_tol"])))
    assert np.max(np.abs(res.theta_mode.theta - G["fit_theta"])) <= 1e-5


@pytest.mark.parametrize("case", ["c2fit", "c2fitd"])
def test_fit_full_c2_vs_reference(case):
    """Full c2 (Poisson, n = 40 003) fits: the pinned optimizer settings
    (theta* <= 1e-5) and the reference defaults (mixed FD, 5 candidates: the
    reference itself runs into max-iters there, see below)."""
    import json

    from paper_2204_04678_b200.fit import FitConfig, fit
    from paper_2204_04678_b200.optimizer import FDConfig, LineSearchConfig
    from paper_2204_04678_b200.runtime import ThreadBudget

    G = load_golden(case)
    inst = golden_instance(G)
    cfg = json.loads(str(G["fit_config"]))
    res = fit(inst.spec, inst.y, FitConfig(budget=ThreadBudget(7, 1), fd=FDConfig(scheme=cfg["fd"]),
                                           line_search=LineSearchConfig(candidates=cfg["candidates"])))
    if case == "c2fitd":
        # With its own defaults the REFERENCE does not converge on full c2: 200
        # iterations ("max-iters", 2 598 evaluations), f = 133 454.49 -- 10.7
        # above the optimum the pinned settings reach (c2fit: 133 443.81) --
        # with a near-singular Hessian (hyper sds 324 / 9 995).  Forward
        # differences at inner_tol 1e-8 in the flat kappa valley follow rounding
        # noise, so the path is implementation-noise driven on both sides and
        # the end points are not comparable at 1e-5 (the engine stops "stalled"
        # at f = 133 458.60).  What is pinned instead: neither side reports
        # convergence, both end above the pinned-settings optimum, and the
        # objective itself agrees at the reference's end point.
        from paper_2204_04678_b200.objective import ObjectiveEvaluator

        assert str(G["fit_status"]) != "converged" and res.optimization.status != "converged"
        f_opt = float(load_golden("c2fit")["fit_f"])
        assert float(G["fit_f"]) > f_opt + 1.0 and res.f_mode > f_opt + 1.0
        ev = ObjectiveEvaluator(inst.spec, inst.y, inner_tol=1e-12)
        val, _ = ev.eval_objective(np.asarray(G["fit_theta"]))
        assert abs(val.f - float(G["fit_f"])) <= 1e-9 * abs(float(G["fit_f"]))
        return
    assert res.optimization.status == str(G["fit_status"])
    assert np.max(np.abs(res.theta_mode.theta - G["fit_theta"])) <= 1e-5
    assert abs(res.f_mode - float(G["fit_f"])) <= 1e-9 * abs(float(G["fit_f"]))


def test_fit_c1_grid_strategy_vs_reference():
    """strategy="grid": explore_grid waves on the Hessian eigen-axes + one
    selected inversion per integration point, mixture marginals."""
    from paper_2204_04678_b200.fit import FitConfig, fit
    from paper_2204_04678_b200.optimizer import FDConfig, LineSearchConfig
    from paper_2204_04678_b200.runtime import ThreadBudget

    G = load_golden("c1grid")
    inst = golden_instance(G)
    res = fit(inst.spec, inst.y, FitConfig(budget=ThreadBudget(7, 1), fd=FDConfig(scheme="central"),
                                           line_search=LineSearchConfig(candidates=6),
                                           strategy="grid"))
    assert np.max(np.abs(res.theta_mode.theta - G["fit_theta"])) <= 1e-5
    assert res.marginals.n_points == int(G["fit_n_points"])
    mu, sd = G["fit_latent_mean"], G["fit_latent_sd"]
    assert np.max(np.abs(res.marginals.latent_mean - mu)) <= 1e-6 * max(1.0, np.max(np.abs(mu)))
    assert np.max(np.abs(res.marginals.latent_sd - sd) / sd) <= 1e-6
    hsd = np.array([h.sd for h in res.marginals.hyper])
    assert np.max(np.abs(hsd - G["fit_hyper_sd"]) / G["fit_hyper_sd"]) <= 1e-4
