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
    perm, nd, bounds = structured_order(inst.spec, two_sided=False)
    assert bounds is None
    spec = inst.spec
    assert nd == spec.n_fixed
    assert sorted(perm.tolist()) == list(range(spec.latent_dim))
    # block t = 16 field nodes then the temporal node of t
    ofs_f = spec.component_offset(spec.components[0])
    ofs_t = spec.component_offset(spec.components[1])
    assert perm[16] == ofs_t + 0 and perm[0] == ofs_f
    assert list(perm[-nd:]) == list(range(spec.n_fixed))


def test_two_sided_time_order_is_fill_free_and_splits_the_chain():
    """Blocks 0..h-1 forward, nt-1..h+1 backward, separator h last: the
    symbolic factor has no more nonzeros than the one-sided BTA order, and
    no tile couples the two segments except through the separator."""
    from paper_2204_04678_b200.model import build_design
    from paper_2204_04678_b200.ordering import conditional_graph, structured_order

    inst = make_instance("c5", nx=4, ny=4, nt=7, m=80)
    spec = inst.spec
    A = build_design(spec)
    plan = spec._prior_plan
    G = conditional_graph(spec, A, plan.indptr, plan.indices).toarray() != 0
    ns1 = 17  # 16 field nodes + the temporal node of each block

    p1, nd1, _ = structured_order(spec, two_sided=False)
    p2, nd2, b2 = structured_order(spec)
    assert nd1 == nd2 == spec.n_fixed
    assert sorted(p2.tolist()) == list(range(spec.latent_dim))
    # segment boundaries are tile boundaries: A = 3 blocks, B = 3 blocks, sep = 1
    cuts = set(b2.tolist())
    assert 3 * ns1 in cuts and 6 * ns1 in cuts and 7 * ns1 in cuts
    # block order: 0,1,2 | 6,5,4 | 3
    ofs_t = spec.component_offset(spec.components[1])
    tnode = [int(p2[k * ns1 + 16]) - ofs_t for k in range(7)]
    assert tnode == [0, 1, 2, 6, 5, 4, 3]
    # symbolic fill of the two-sided order does not exceed the one-sided BTA
    rng = np.random.default_rng(0)
    W = rng.uniform(0.1, 1.0, G.shape) * G
    S = (W + W.T) / 2 + np.eye(G.shape[0]) * G.shape[0]

    def nnz_l(perm):
        L = np.linalg.cholesky(S[np.ix_(perm, perm)])
        return np.count_nonzero(np.abs(L) > 1e-14)

    assert nnz_l(p2) <= nnz_l(p1)
