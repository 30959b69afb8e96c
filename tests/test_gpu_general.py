"""General GMRFs (the reference's own iid / besag kinds) on the native
nested-dissection tile path, against the UNMODIFIED reference's outputs
(tests/golden/{grid2d,leuks,leuk}.npz, made by tests/golden/make_golden.py).

The engine orders the conditional pattern exactly as the reference does
(same permutation), so besides the ordering-invariant f, log dets, modes and
variances, the factor / selected-inverse VALUES on the reference's scalar
pattern and the GMRF sample (cholesky.py:339-353) are compared entry-wise."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

F_TOL = 1e-9
VAR_TOL = 1e-8
KIND_CASES = ["grid2d", "leuks", "leuk"]


def _setup(case):
    from paper_2204_04678_b200.objective import ObjectiveEvaluator
    from paper_2204_04678_b200.synth import reference_kind_instance

    G = load_golden(case)
    inst = reference_kind_instance(str(G["kind"]), side=int(G["side"]), m=int(G["m"]))
    ev = ObjectiveEvaluator(inst.spec, inst.y, inner_tol=float(G["inner_tol"]))
    return G, inst, ev


@pytest.mark.parametrize("case", KIND_CASES)
def test_general_gmrf_f_logdets_iterations_vs_reference(case):
    G, inst, ev = _setup(case)
    assert np.array_equal(ev.engine.perm, G["perm_cond"])  # the reference's ordering
    res = ev.engine.eval_batch(G["thetas"], want_modes=True)
    assert np.all(res["status"] == 0)
    ref = G["f_components"]
    rel = np.abs(res["comps"] - ref[:, :5]) / np.maximum(1.0, np.abs(ref[:, :5]))
    assert rel.max() <= F_TOL, rel
    from test_gpu_parity import check_iterations

    check_iterations(inst, G, res["iters"])  # Newton iteration counts
    ldrel = np.abs(res["logdets"] - G["logdets"]) / np.abs(G["logdets"])
    assert ldrel.max() <= F_TOL, ldrel
    m = G["mode"]
    assert np.max(np.abs(res["modes"][0] - m)) <= 1e-7 * max(1.0, np.max(np.abs(m)))
    ev.close()


@pytest.mark.parametrize("case", KIND_CASES)
def test_general_gmrf_variances_and_payloads_vs_reference(case):
    from paper_2204_04678_b200.cholesky import sample_gmrf, selected_inverse

    G, inst, ev = _setup(case)
    th = G["thetas"][0]
    val, approx = ev.eval_objective(th)
    si = selected_inverse(approx.factor)
    ref = G["variances"]
    assert np.max(np.abs(si.marginal_variances - ref) / ref) <= VAR_TOL
    sym = approx.factor.symbolic
    assert sym.nnz == int(G["nnz_L"])
    # entries of L and Sigma on the reference's pattern (subset for leuk)
    rows, cols = G["L_rows"], G["L_cols"]
    Lp, Li = sym.Lp, sym.Li
    pos = np.array([Lp[c] + np.searchsorted(Li[Lp[c]:Lp[c + 1]], r) for r, c in zip(rows, cols)])
    Lv = approx.factor.values[pos]
    Sv = si.values[pos]
    Lref, Sref = G["L_values"], G["Sigma_values"]
    scale = np.max(np.abs(Lref))
    assert np.max(np.abs(Lv - Lref)) <= 1e-9 * scale
    # Sigma entries on the correlation scale |dS_ij| / sqrt(S_ii S_jj): the
    # intrinsic besag + vague intercept make Sigma ill-conditioned (entries
    # up to ~1e2 cancelling to ~1e-4), so entry-relative errors of the small
    # off-diagonal entries are conditioning-limited on both sides
    var_perm = si.marginal_variances[sym.perm]
    corr_scale = np.sqrt(var_perm[rows] * var_perm[cols])
    assert np.max(np.abs(Sv - Sref) / corr_scale) <= VAR_TOL
    diag = rows == cols
    assert np.max(np.abs(Sv[diag] - Sref[diag]) / Sref[diag]) <= VAR_TOL
    if "sample_z" in G.files:
        x = sample_gmrf(approx.factor, G["sample_z"])
        xr = G["sample_x"]
        assert np.max(np.abs(x - xr)) <= 1e-8 * max(1.0, np.max(np.abs(xr)))
    # the conditional precision at the mode: Q_c x* = A^T tau (y - offsets)
    # (Gaussian) holds on the payload matrix
    if inst.spec.family == "gaussian":
        Qf = approx.cond_precision.to_scipy()  # both triangles
        tau = float(np.exp(th[0]))
        rhs = ev.A.T @ (tau * (inst.y - inst.spec.offsets))
        r = Qf @ approx.mode - rhs
        assert np.max(np.abs(r)) <= 1e-8 * np.max(np.abs(rhs))
    ev.close()


@pytest.mark.parametrize("case", ["grid2d", "leuks"])
def test_general_gmrf_fit_vs_reference(case):
    from paper_2204_04678_b200.fit import FitConfig, fit
    from paper_2204_04678_b200.optimizer import FDConfig, LineSearchConfig
    from paper_2204_04678_b200.runtime import ThreadBudget
    from paper_2204_04678_b200.synth import reference_kind_instance

    G = load_golden(case)
    inst = reference_kind_instance(str(G["kind"]), side=int(G["side"]), m=int(G["m"]))
    res = fit(inst.spec, inst.y, FitConfig(budget=ThreadBudget(7, 1), fd=FDConfig(scheme="central"),
                                           line_search=LineSearchConfig(candidates=6)))
    assert np.max(np.abs(res.theta_mode.theta - G["fit_theta"])) <= 1e-5
    assert abs(res.f_mode - float(G["fit_f"])) <= 1e-9 * abs(float(G["fit_f"]))
    sd = G["fit_latent_sd"]
    assert np.max(np.abs(res.marginals.latent_sd - sd) / sd) <= 1e-6


def test_general_gmrf_device_work_vs_reference_nd():
    """Executed tile flops of the leukemia-like factorization against the
    reference ND's scalar count (sum of squared column counts)."""
    G, inst, ev = _setup("leuk")
    st = ev.engine.stats()
    ratio = st["factor_flops_limited"] / float(G["sum_colcount_sq"])
    print(f"leukemia-like: executed tile flops / sum c^2 = {ratio:.2f}")
    assert ratio < 8.0
    ev.close()


def test_cli_fit_writes_schema_valid_outputs(tmp_path):
    """`python -m paper_2204_04678_b200.cli fit` on files (model.json with a
    besag graph_file, data.csv): outputs validate against the contracts and
    theta* equals the in-memory fit()."""
    import json

    from test_io_host import _write_grid2d

    from paper_2204_04678_b200.cli import main
    from paper_2204_04678_b200.fit import FitConfig, fit
    from paper_2204_04678_b200.io import validate

    inst = _write_grid2d(tmp_path)
    out = tmp_path / "run"
    rc = main(["fit", "--model", str(tmp_path / "model.json"), "--data", str(tmp_path / "data.csv"),
               "--out", str(out), "--strategy", "grid"])
    assert rc == 0
    summary = json.loads((out / "summary.json").read_text())
    validate(summary, "summary")
    validate(json.loads((out / "hyper.json").read_text()), "hyper")
    for line in (out / "trace.jsonl").read_text().splitlines():
        validate(json.loads(line), "trace")
    r = fit(inst.spec, inst.y, FitConfig(strategy="grid"))
    assert np.max(np.abs(np.array(summary["theta_mode"]) - r.theta_mode.theta)) <= 1e-12
    rows = (out / "marginals.csv").read_text().splitlines()
    assert len(rows) == inst.n + 1
