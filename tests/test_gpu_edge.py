"""Failure semantics and edge cases on the device path."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def small(cfg="c1", **over):
    from paper_2204_04678_b200.synth import make_instance

    base = dict(c1=dict(nx=10, ny=9, m=200), c2=dict(nx=8, ny=8, m=300),
                c5=dict(nx=6, ny=5, nt=4, m=200))[cfg]
    base.update(over)
    return make_instance(cfg, **base)


def test_one_bad_slot_does_not_poison_the_batch():
    from paper_2204_04678_b200.errors import BatchError, NotPositiveDefinite
    from paper_2204_04678_b200.fit import FitObjective
    from paper_2204_04678_b200.objective import ObjectiveEvaluator

    inst = small("c2")
    ev = ObjectiveEvaluator(inst.spec, inst.y, max_slots=3)
    good = inst.theta_true
    bad = np.array([800.0, -3.0])  # exp overflow -> inf precision -> not PD
    vals = ev.eval_values([good, bad, good + 0.1])
    assert isinstance(vals[1], NotPositiveDefinite)
    ref = ev.eval_values([good, good + 0.1])
    assert vals[0].f == ref[0].f and vals[2].f == ref[1].f
    with pytest.raises(BatchError) as info:
        ev.eval_batch([good, bad, bad])
    assert info.value.slot == 1
    fo = FitObjective(ev)
    out = fo.eval_batch([good, bad])
    assert math.isfinite(out[0]) and out[1] == math.inf
    with pytest.raises(NotPositiveDefinite):
        ev.eval_objective(bad)


def test_inner_divergence():
    from paper_2204_04678_b200.errors import InnerDivergence
    from paper_2204_04678_b200.objective import ObjectiveEvaluator

    inst = small("c2")
    ev = ObjectiveEvaluator(inst.spec, inst.y, max_inner=1, inner_tol=1e-14)
    with pytest.raises(InnerDivergence):
        ev.eval_objective(inst.theta_true)


def test_warm_start_and_gaussian_ignores_it():
    from paper_2204_04678_b200.errors import DimensionMismatch
    from paper_2204_04678_b200.objective import ObjectiveEvaluator

    inst = small("c5")
    ev = ObjectiveEvaluator(inst.spec, inst.y)
    v0, a0 = ev.eval_objective(inst.theta_true)
    v1, a1 = ev.eval_objective(inst.theta_true, warm_start=a0.mode)
    assert a1.iterations <= a0.iterations
    assert abs(v1.f - v0.f) <= 1e-9 * abs(v0.f)
    with pytest.raises(DimensionMismatch):
        ev.eval_objective(inst.theta_true, warm_start=np.zeros(3))
    g = small("c1")
    evg = ObjectiveEvaluator(g.spec, g.y)
    f0 = evg.objective(g.theta_true)
    f1 = evg.objective(g.theta_true, warm_start=np.ones(g.n))
    assert f0 == f1 and evg.gaussian_approx(g.theta_true).iterations == 1


def test_component_identity_and_empty_batch():
    from paper_2204_04678_b200.objective import ObjectiveEvaluator

    inst = small("c1")
    ev = ObjectiveEvaluator(inst.spec, inst.y)
    val, _ = ev.eval_objective(inst.theta_true + 0.2)
    recon = -(val.log_prior_hyper + val.log_prior_latent + val.log_likelihood - val.log_gaussian_approx)
    assert abs(val.f - recon) <= 1e-12 * abs(val.f)
    assert ev.eval_batch([]) == []


def test_reference_kinds_model_on_device():
    """The reference's own iid/rw1/besag components run through the RCM
    tile path; f equals the oracle's."""
    from oracle.oracle import OracleEvaluator
    from paper_2204_04678_b200.model import Component, ModelSpec
    from paper_2204_04678_b200.objective import ObjectiveEvaluator

    rng = np.random.default_rng(11)
    m = 400
    side = 6
    idx = np.arange(side * side).reshape(side, side)
    u = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
    v = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
    import scipy.sparse as sp

    W = sp.coo_matrix((np.ones(u.size), (u, v)), shape=(36, 36))
    W = (W + W.T).tocsr()
    comps = [
        Component("trend", "rw1", 30, 1, obs_index=rng.integers(0, 30, m)),
        Component("space", "besag", 36, 2, obs_index=rng.integers(0, 36, m),
                  graph=(W.indptr.astype(np.int64), W.indices.astype(np.int64))),
        Component("u", "iid", 50, 3, obs_index=rng.integers(0, 50, m)),
    ]
    from paper_2204_04678_b200.model import ModelSpec as MS

    spec = MS(m, "gaussian", comps, Z=rng.normal(size=(m, 2)))
    y = rng.normal(size=m)
    ev = ObjectiveEvaluator(spec, y)
    orc = OracleEvaluator(spec, y)
    for th in ([0.2, 0.1, -0.3, 0.5], [1.0, 2.0, 0.0, -1.0]):
        g = ev.objective(th)
        w = orc.eval(np.array(th))["f"]
        assert abs(g - w) <= 1e-9 * abs(w)
