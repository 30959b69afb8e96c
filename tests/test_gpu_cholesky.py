"""Generic device factorize / solve / selected_inverse drop-ins against the
reference's known answers (test_cholesky.py) and dense numpy."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TWO = np.array([[4.0, 2.0], [2.0, 3.0]])


def mats():
    from paper_2204_04678_b200.sparse import SparseSymMatrix

    return SparseSymMatrix


def test_hand_2x2():
    from paper_2204_04678_b200.cholesky import analyze, factorize, selected_inverse, solve

    Q = mats().from_dense(TWO)
    fac = factorize(analyze(Q, "natural"), Q)
    assert abs(fac.log_det - math.log(8.0)) < 1e-14  # test_cholesky.py:30-34
    np.testing.assert_allclose(solve(fac, np.array([8.0, 7.0])), [1.25, 1.5], atol=1e-14)
    si = selected_inverse(fac)
    np.testing.assert_allclose(si.marginal_variances, [0.375, 0.5], atol=1e-14)


def test_identity_and_not_pd():
    from paper_2204_04678_b200.cholesky import analyze, factorize
    from paper_2204_04678_b200.errors import NotPositiveDefinite

    Q = mats().from_dense(np.eye(7))
    assert factorize(analyze(Q, "natural"), Q).log_det == 0.0
    Q = mats().from_dense(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(NotPositiveDefinite) as info:
        factorize(analyze(Q, "natural"), Q)
    assert info.value.column == 1  # test_cholesky.py:50-55


@pytest.mark.parametrize("n", [1, 63, 64, 65, 300])
def test_rw2_vs_dense(n):
    from paper_2204_04678_b200.cholesky import analyze, factorize, selected_inverse, solve

    if n < 3:
        R = np.array([[2.5]])
    else:
        D = np.diff(np.eye(n), 2, axis=0)
        R = 1.7 * D.T @ D + 1e-3 * np.eye(n)  # test_cholesky.py:159-171
    Q = mats().from_dense(R)
    for ordering in ("natural", "nested-dissection"):
        fac = factorize(analyze(Q, ordering), Q)
        sign, ref = np.linalg.slogdet(R)
        assert abs(fac.log_det - ref) <= 1e-9 * max(1.0, abs(ref))
        dense = np.linalg.inv(R)
        var = selected_inverse(fac).marginal_variances
        assert np.max(np.abs(var - np.diag(dense)) / np.diag(dense)) <= 1e-9
        b = np.random.default_rng(n).standard_normal(n)
        x = solve(fac, b)
        assert np.max(np.abs(R @ x - b)) / np.max(np.abs(b)) <= 1e-10


def test_random_gmrf_vs_dense():
    from paper_2204_04678_b200.cholesky import analyze, factorize, selected_inverse

    rng = np.random.default_rng(4)
    n = 500
    M = np.zeros((n, n))
    for _ in range(4 * n):
        i, j = rng.integers(0, n, 2)
        if i != j:
            M[i, j] = M[j, i] = rng.normal()
    np.fill_diagonal(M, np.abs(M).sum(1) + 0.5)
    Q = mats().from_dense(M)
    fac = factorize(analyze(Q), Q)
    assert abs(fac.log_det - np.linalg.slogdet(M)[1]) <= 1e-9 * abs(np.linalg.slogdet(M)[1])
    var = selected_inverse(fac).marginal_variances
    assert np.max(np.abs(var - np.diag(np.linalg.inv(M))) / np.diag(np.linalg.inv(M))) <= 1e-9
