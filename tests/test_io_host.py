"""Model / data / graph readers and the run-output writers (host only)."""

import json
from types import SimpleNamespace

import numpy as np
import pytest


def _write_grid2d(tmp_path):
    from paper_2204_04678_b200.io import write_graph_file
    from paper_2204_04678_b200.synth import reference_kind_instance

    inst = reference_kind_instance("grid2d", side=6)
    c = inst.spec.components[0]
    write_graph_file(tmp_path / "graph.txt", *c.graph)
    (tmp_path / "model.json").write_text(json.dumps({
        "likelihood": {"family": "poisson"}, "fixed": [],
        "components": [{"name": "spatial", "kind": "besag", "graph_file": "graph.txt",
                        "hyper": {"shape": 1.0, "rate": 5e-5}}],
        "options": {"intercept": True}}))
    lines = ["y,exposure,spatial"] + [f"{float(y)!r},{float(e)!r},{float(i)!r}" for y, e, i in
                                      zip(inst.y, inst.spec.exposures, c.obs_index)]
    (tmp_path / "data.csv").write_text("\n".join(lines) + "\n")
    return inst


def test_load_model_round_trip(tmp_path):
    from paper_2204_04678_b200.io import load_model

    inst = _write_grid2d(tmp_path)
    spec, y = load_model(tmp_path / "model.json", tmp_path / "data.csv")
    assert np.array_equal(y, inst.y)
    assert spec.theta_names == inst.spec.theta_names and spec.latent_dim == inst.n
    a, b = spec._prior_plan, inst.spec._prior_plan
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.term_coef, b.term_coef)


def test_config_errors(tmp_path):
    from paper_2204_04678_b200.errors import ConfigError
    from paper_2204_04678_b200.io import read_model_file

    p = tmp_path / "m.json"
    p.write_text(json.dumps({"likelihood": {"family": "binomial"}}))
    with pytest.raises(ConfigError) as e:
        read_model_file(p)
    assert e.value.key == "likelihood.family"
    p.write_text(json.dumps({"likelihood": {"family": "gaussian"},
                             "components": [{"name": "s", "kind": "besag"}]}))
    with pytest.raises(ConfigError) as e:
        read_model_file(p)
    assert "graph_file" in e.value.key


def test_outputs_validate_against_schemas(tmp_path):
    from paper_2204_04678_b200.io import validate, write_fit_outputs
    from paper_2204_04678_b200.marginals import HyperMarginal, MarginalResult
    from paper_2204_04678_b200.runtime import ThreadBudget

    marg = MarginalResult(np.array([0.1, 0.2]), np.array([1.0, 2.0]), ["a", "b"],
                          hyper=[HyperMarginal("log_prec_s", 0.5, 0.1,
                                               [(0.3, 0.1), (0.5, 1.0), (0.7, 0.1)])], n_points=3)
    trace = [{"iter": 0, "f": 10.0, "grad_norm": 1.0, "step": 0.0, "n_evals": 3, "wall_ms": 1.0},
             {"iter": 1, "f": 9.0, "grad_norm": 0.1, "step": 0.5, "n_evals": 9, "wall_ms": 2.0}]
    summary = {"theta_mode": [0.5], "theta_names": ["log_prec_s"], "f_mode": 9.0,
               "status": "converged", "iterations": 1, "n_fn_evals": 9, "time_per_fn_s": 0.01,
               "analyze_s": 0.1, "total_s": 0.3, "budget": "1:1", "n_latent": 2, "n_obs": 4,
               "n_integration_points": 3}
    res = SimpleNamespace(marginals=marg, optimization=SimpleNamespace(trace=trace, status="converged"),
                          budget=ThreadBudget(1, 1), summary=lambda: summary)
    write_fit_outputs(tmp_path, res)
    validate(json.loads((tmp_path / "summary.json").read_text()), "summary")
    validate(json.loads((tmp_path / "hyper.json").read_text()), "hyper")
    for line in (tmp_path / "trace.jsonl").read_text().splitlines():
        validate(json.loads(line), "trace")
    rows = (tmp_path / "marginals.csv").read_text().splitlines()
    assert rows[0] == "index,component,mean,sd" and len(rows) == 3
