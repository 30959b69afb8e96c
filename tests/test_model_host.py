"""Host-side model logic: prior plan vs the oracle's independent assembler,
hyper prior / likelihood KATs (reference test_model.py), design, orderings."""

import math

import numpy as np
import pytest

from paper_2204_04678_b200.model import (
    Component, LatticeGraph, ModelSpec, assemble_prior_precision, build_design, likelihood_terms,
    log_prior_hyper,
)
from paper_2204_04678_b200.synth import make_instance


@pytest.mark.parametrize("cfg,over", [
    ("c1", {}), ("c2", dict(nx=20, ny=20, m=500)), ("c3", dict(nx=8, ny=8, nt=5, m=400)),
    ("c5", dict(nx=8, ny=8, nt=5, m=400)),
])
def test_prior_plan_matches_independent_assembly(cfg, over):
    from oracle.oracle import OracleModel

    inst = make_instance(cfg, **over)
    om = OracleModel(inst.spec, inst.y)
    plan = inst.spec._prior_plan
    assert np.array_equal(plan.indptr, om.p_indptr)
    assert np.array_equal(plan.indices, om.p_indices)
    rng = np.random.default_rng(1)
    for _ in range(3):
        th = inst.theta_true + rng.normal(0, 0.3, inst.theta_true.size)
        a = assemble_prior_precision(inst.spec, th).data
        b = om.prior_values(th)
        assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(b))


def test_reference_kinds_bitwise_plan():
    """iid/rw1/rw2/besag: value = base * exp(theta) + jitter exactly."""
    m = 30
    rng = np.random.default_rng(0)
    g_indptr = np.array([0, 1, 3, 4], dtype=np.int64)
    g_indices = np.array([1, 0, 2, 1], dtype=np.int64)
    comps = [
        Component("a", "rw1", 6, 1, obs_index=rng.integers(0, 6, m)),
        Component("b", "rw2", 5, 2, obs_index=rng.integers(0, 5, m)),
        Component("c", "besag", 3, 3, obs_index=rng.integers(0, 3, m), graph=(g_indptr, g_indices)),
        Component("d", "iid", 4, 4, obs_index=rng.integers(0, 4, m)),
    ]
    spec = ModelSpec(m, "gaussian", comps, Z=rng.normal(size=(m, 2)))
    th = np.array([0.1, 0.3, -0.2, 0.7, 1.1])
    Q = assemble_prior_precision(spec, th).to_dense()
    from oracle.oracle import OracleModel

    om = OracleModel(spec, np.zeros(m))
    Qo = np.zeros_like(Q)
    vals = om.prior_values(th)
    cols = np.repeat(np.arange(spec.latent_dim), np.diff(om.p_indptr))
    Qo[om.p_indices, cols] = vals
    Qo = Qo + np.tril(Qo, -1).T
    assert np.array_equal(Q, Qo)


def test_hyper_prior_kats():
    spec = ModelSpec(3, "gaussian", [Component("u", "iid", 2, 0, obs_index=np.zeros(3, int),
                                               hyper_shape=1.0, hyper_rate=1.0)],
                     noise_precision=1.0, intercept=False)
    assert abs(log_prior_hyper(spec, [0.0]) - (-1.0)) < 1e-14
    assert abs(log_prior_hyper(spec, [math.log(2.0)]) - (math.log(2.0) - 2.0)) < 1e-14


def test_likelihood_kats():
    spec = ModelSpec(1, "poisson", [Component("u", "iid", 1, 0, obs_index=np.zeros(1, int))],
                     intercept=False)
    ll, d1, d2 = likelihood_terms(spec, np.array([0.0]), np.array([3.0]), [0.0])
    assert d1[0] == 2.0 and d2[0] == -1.0
    assert abs(ll - (0.0 - 1.0 - math.lgamma(4.0))) < 1e-12
    spec = ModelSpec(3, "gaussian", [Component("u", "iid", 3, 0, obs_index=np.arange(3))],
                     noise_precision=2.0, intercept=False)
    y = np.array([0.5, -1.0, 2.0])
    ll, d1, d2 = likelihood_terms(spec, y.copy(), y, [0.0])
    assert np.all(d1 == 0.0) and np.all(d2 == -2.0)
    assert abs(ll - 1.5 * (math.log(2.0) - math.log(2 * math.pi))) < 1e-12


def test_theta_layout_noise_first():
    inst = make_instance("c3", nx=6, ny=6, nt=3, m=100)
    assert inst.spec.theta_names[0] == "log_prec_noise"
    assert inst.spec.theta_dim == 4
    inst = make_instance("c5", nx=6, ny=6, nt=3, m=100)
    assert inst.spec.theta_dim == 5


def test_bilinear_design_rows():
    inst = make_instance("c1", nx=10, ny=10, m=300)
    A = build_design(inst.spec)
    assert A.shape == (300, inst.n)
    field = A[:, inst.spec.n_fixed:]
    assert np.allclose(np.asarray(field.sum(axis=1)).ravel(), 1.0)
    assert np.all(np.diff(field.indptr) <= 4)


def test_structured_order_is_time_major_bta():
    from paper_2204_04678_b200.ordering import structured_order

    inst = make_instance("c5", nx=4, ny=4, nt=3, m=50)
    perm, nd, bounds = structured_order(inst.spec)
    assert bounds is None
    spec = inst.spec
    assert nd == spec.n_fixed
    assert sorted(perm.tolist()) == list(range(spec.latent_dim))
    # block t = 16 field nodes then the temporal node of t
    ofs_f = spec.component_offset(spec.components[0])
    ofs_t = spec.component_offset(spec.components[1])
    assert perm[16] == ofs_t + 0 and perm[0] == ofs_f
    assert list(perm[-nd:]) == list(range(spec.n_fixed))
