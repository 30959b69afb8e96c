"""Pin the CPU oracle (oracle/) before trusting it as the checker.

(a) the reference's own known-answer tests, restated
    (/root/reference/pkg/tests/test_cholesky.py:30-34, 98-101, 146-151,
     159-171; test_model.py:127-162)
(b) golden vectors from the UNMODIFIED reference run through the SURVEY
    Appendix-B adapter (tests/golden/make_golden.py).
"""

import math

import numpy as np
import pytest

from conftest import golden_instance, load_golden

TWO = np.array([[4.0, 2.0], [2.0, 3.0]])


def _lower(M):
    import scipy.sparse as sp

    L = sp.tril(sp.csc_matrix(M)).tocsc()
    L.sort_indices()
    return L.indptr.astype(np.int64), L.indices.astype(np.int64), L.data.astype(np.float64)


def test_hand_2x2_factor_solve_selinv(oracle_lib):
    o = oracle_lib
    ip, ix, v = _lower(TWO)
    s = o.analyze(2, ip, ix, "natural")
    Lx, ld = o.factorize(s, v)
    np.testing.assert_allclose(Lx, [2.0, 1.0, math.sqrt(2.0)])  # test_cholesky.py:30-34
    assert abs(ld - math.log(8.0)) < 1e-14
    np.testing.assert_allclose(o.solve(s, Lx, np.array([8.0, 7.0])), [1.25, 1.5], atol=1e-14)
    Sx, var = o.selected_inverse(s, Lx)
    np.testing.assert_allclose(var, [0.375, 0.5], atol=1e-14)  # test_cholesky.py:146-151
    assert abs(Sx[1] - (-0.25)) < 1e-14


def test_not_positive_definite_column(oracle_lib):
    o = oracle_lib
    ip, ix, v = _lower(np.array([[1.0, 2.0], [2.0, 1.0]]))
    s = o.analyze(2, ip, ix, "natural")
    with pytest.raises(o.NotPD) as info:
        o.factorize(s, v)
    assert info.value.column == 1  # test_cholesky.py:50-55


def test_rw2_selinv_vs_dense(oracle_lib):
    o = oracle_lib
    n = 300
    D = np.diff(np.eye(n), 2, axis=0)
    R = 1.7 * D.T @ D + 1e-3 * np.eye(n)  # test_cholesky.py:159-171
    ip, ix, v = _lower(R)
    s = o.analyze(n, ip, ix, "nested-dissection", leaf_cutoff=32)
    Lx, ld = o.factorize(s, v)
    _, var = o.selected_inverse(s, Lx)
    dense = np.linalg.inv(R)
    assert np.max(np.abs(var - np.diag(dense)) / np.diag(dense)) <= 1e-9
    sign, ref = np.linalg.slogdet(R)
    assert abs(ld - ref) <= 1e-9 * abs(ref)


def test_hyper_prior_and_likelihood_kats():
    from oracle.oracle import OracleModel
    from paper_2204_04678_b200.model import Component, ModelSpec

    spec = ModelSpec(1, "poisson", [Component("u", "iid", 1, 0, obs_index=np.zeros(1, int),
                                              hyper_shape=1.0, hyper_rate=1.0)], intercept=False)
    om = OracleModel(spec, np.array([3.0]))
    assert abs(om.log_prior_hyper([0.0]) - (-1.0)) < 1e-14  # test_model.py:127-132
    assert abs(om.log_prior_hyper([math.log(2.0)]) - (math.log(2.0) - 2.0)) < 1e-14
    ll, d1, d2 = om.lik(np.array([0.0]), [0.0])  # test_model.py:158-162
    assert d1[0] == 2.0 and d2[0] == -1.0
    assert abs(ll - (0.0 - 1.0 - math.lgamma(4.0))) < 1e-12


@pytest.mark.parametrize("case", ["c1", "c2r", "c3r", "c4r", "c5r"])
def test_oracle_matches_reference_goldens(case):
    from oracle.oracle import OracleEvaluator

    G = load_golden(case)
    inst = golden_instance(G)
    ev = OracleEvaluator(inst.spec, inst.y, inner_tol=float(G["inner_tol"]))
    for k, th in enumerate(G["thetas"]):
        r = ev.eval(th)
        ref = G["f_components"][k]
        got = [r["f"], r["log_prior_hyper"], r["log_prior_latent"], r["log_likelihood"],
               r["log_gaussian_approx"]]
        for g, w in zip(got, ref[:5]):
            assert abs(g - w) <= 1e-11 * max(1.0, abs(w)), (case, k, got, ref)
        assert r["iterations"] == int(ref[5])
        assert abs(r["logdet_cond"] - G["logdets"][k, 0]) <= 1e-12 * abs(G["logdets"][k, 0])
        assert abs(r["logdet_prior"] - G["logdets"][k, 1]) <= 1e-12 * abs(G["logdets"][k, 1])
        if k == 0:
            m = G["mode"]
            assert np.max(np.abs(r["mode"] - m)) <= 1e-9 * max(1.0, np.max(np.abs(m)))
            if "variances" in G.files:
                from oracle.oracle import selected_inverse

                _, var = selected_inverse(ev.sym_cond, r["Lcond"])
                assert np.max(np.abs(var - G["variances"]) / G["variances"]) <= 1e-10


def test_golden_data_not_drifted():
    """The generator must still produce the data the goldens were made from."""
    import hashlib

    for case in ("c1", "c2r", "c3r", "c4r", "c5r"):
        G = load_golden(case)
        inst = golden_instance(G)
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(inst.y).tobytes())
        h.update(np.ascontiguousarray(inst.spec.Z).tobytes())
        for c in inst.spec.components:
            if c.design is not None:
                h.update(c.design.data.tobytes())
                h.update(c.design.indices.astype(np.int64).tobytes())
        assert h.hexdigest() == str(G["data_hash"]), case


def test_level2_tree_factorization_bitwise(oracle_lib):
    """cholesky.py:282-322: the level-2 schedule (sibling subtrees of the ND
    separator tree as parallel tasks, pruned by _pruned_tasks :217-258, run by
    run_tree_tasks runtime.py:180-268) gives the serial factor bit for bit."""
    import scipy.sparse as sp

    o = oracle_lib
    side = 70
    e = np.ones(side)
    T = sp.diags([-e[:-1], 2 * e, -e[:-1]], [-1, 0, 1])
    G = sp.kron(sp.eye(side), T) + sp.kron(T, sp.eye(side))
    Q = (G @ G + 0.3 * G + 0.01 * sp.eye(side * side)).tocsc()
    ip, ix, v = _lower(Q)
    s = o.analyze(Q.shape[0], ip, ix, "nested-dissection")
    nodes, root = s.tree
    assert nodes[root]["end"] == s.n and min(nd["span_start"] for nd in nodes) == 0
    parents, children, ranges = o.pruned_tasks(s, 4)
    assert len(ranges) > 4
    cover = np.zeros(s.n, np.int64)
    for a, b in ranges:
        cover[a:b] += 1
    assert np.all(cover == 1)  # every column in exactly one task
    for t, p in enumerate(parents):
        if p >= 0:
            assert ranges[t][1] <= ranges[p][0]  # a child's span precedes its parent
    L1, ld1 = o.factorize(s, v)
    for w in (2, 4):
        Lw, ldw = o.factorize(s, v, workers=w)
        assert np.array_equal(L1, Lw) and ld1 == ldw
