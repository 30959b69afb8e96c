"""File formats of the fit pipeline (reference model.py:363-534 readers,
marginals.py:241-265 / cli.py:64-78 writers): the model JSON document, the
data CSV, the besag graph file, and the run outputs marginals.csv,
hyper.json, trace.jsonl and summary.json (contracts in
``paper_2204_04678_b200/schemas/``).  Host-side glue around the device
pipeline; nothing here touches the GPU."""

from __future__ import annotations

import csv
import json
from pathlib import Path

import numpy as np

from .errors import ConfigError
from .model import COMPONENT_KINDS, DEFAULT_FIXED_PRIOR_PREC, DEFAULT_HYPER_RATE, \
    DEFAULT_HYPER_SHAPE, DEFAULT_JITTER, Component, ModelSpec

SCHEMA_DIR = Path(__file__).parent / "schemas"


def read_graph_file(path):
    """Adjacency list: first token n, then per vertex "i deg j1 .. jdeg"
    (0-based).  Returns (indptr, indices) of the symmetric graph."""
    tok = Path(path).read_text().split()
    if not tok:
        raise ConfigError("graph_file", f"{path}: empty graph file")
    vals = [int(t) for t in tok]
    n, pos = vals[0], 1
    nbrs = [[] for _ in range(n)]
    while pos < len(vals):
        i, deg = vals[pos], vals[pos + 1]
        if not 0 <= i < n:
            raise ConfigError("graph_file", f"{path}: vertex {i} out of range")
        js = vals[pos + 2: pos + 2 + deg]
        if len(js) != deg:
            raise ConfigError("graph_file", f"{path}: truncated neighbour list of {i}")
        for j in js:
            if not 0 <= j < n or j == i:
                raise ConfigError("graph_file", f"{path}: bad neighbour {j} of {i}")
            nbrs[i].append(j)
            nbrs[j].append(i)
        pos += 2 + deg
    indptr = np.zeros(n + 1, dtype=np.int64)
    lists = [np.unique(np.asarray(b, dtype=np.int64)) for b in nbrs]
    indptr[1:] = np.cumsum([x.size for x in lists])
    indices = np.concatenate(lists) if n else np.empty(0, np.int64)
    return indptr, indices


def write_graph_file(path, indptr, indices):
    n = indptr.size - 1
    lines = [str(n)]
    for v in range(n):
        nb = indices[indptr[v]: indptr[v + 1]]
        lines.append(" ".join(str(int(x)) for x in [v, nb.size, *nb]))
    Path(path).write_text("\n".join(lines) + "\n")


def _hyper(obj, key):
    if obj is None:
        return DEFAULT_HYPER_SHAPE, DEFAULT_HYPER_RATE
    if not isinstance(obj, dict) or "shape" not in obj or "rate" not in obj:
        raise ConfigError(key, "hyper prior needs {shape, rate}")
    a, b = float(obj["shape"]), float(obj["rate"])
    if a <= 0 or b <= 0:
        raise ConfigError(key, "hyper prior shape and rate must be positive")
    return a, b


def read_model_file(path) -> dict:
    try:
        doc = json.loads(Path(path).read_text())
    except json.JSONDecodeError as exc:
        raise ConfigError("model", f"{path}: invalid JSON ({exc})") from exc
    if not isinstance(doc, dict):
        raise ConfigError("model", "top level must be an object")
    lik = doc.get("likelihood")
    if not isinstance(lik, dict) or lik.get("family") not in ("gaussian", "poisson"):
        raise ConfigError("likelihood.family", "missing or unknown likelihood.family")
    comps = doc.get("components", [])
    if not isinstance(comps, list):
        raise ConfigError("components", "must be a list")
    for i, c in enumerate(comps):
        if not isinstance(c, dict) or "kind" not in c or "name" not in c:
            raise ConfigError(f"components[{i}]", "needs name and kind")
        if c["kind"] not in COMPONENT_KINDS:
            raise ConfigError(f"components[{i}].kind", f"unknown kind {c['kind']!r}")
        if c["kind"] == "besag" and "graph_file" not in c:
            raise ConfigError(f"components[{i}].graph_file", "besag needs graph_file")
        if c["kind"] != "besag" and "size" not in c:
            raise ConfigError(f"components[{i}].size", "needs size")
    fixed = doc.get("fixed", [])
    if not isinstance(fixed, list) or not all(isinstance(s, str) for s in fixed):
        raise ConfigError("fixed", "must be a list of covariate names")
    if not isinstance(doc.get("options", {}), dict):
        raise ConfigError("options", "must be an object")
    return doc


def read_data_file(path) -> dict:
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    if not rows:
        raise ConfigError("data", f"{path}: empty file")
    head, body = rows[0], rows[1:]
    for k, r in enumerate(body, start=2):
        if len(r) != len(head):
            raise ConfigError("data", f"{path}:{k}: wrong column count")
    try:
        cols = np.array(body, dtype=np.float64).reshape(len(body), len(head))
    except ValueError:
        raise ConfigError("data", f"{path}: non-numeric value") from None
    return {name: cols[:, j].copy() for j, name in enumerate(head)}


def build_model(doc: dict, data: dict, base_dir=".", graphs: dict | None = None):
    """(ModelSpec, y) from a validated model document and data columns."""
    if "y" not in data:
        raise ConfigError("data.y", "data file needs a y column")
    y = data["y"]
    m = y.shape[0]
    if m == 0:
        raise ConfigError("data", "no observations")
    lik = doc["likelihood"]
    family = lik["family"]
    opts = doc.get("options", {})
    fixed = doc.get("fixed", [])
    for nm in fixed:
        if nm not in data:
            raise ConfigError(f"fixed.{nm}", "covariate column missing from data")
    Z = np.column_stack([data[nm] for nm in fixed]) if fixed else None
    k = 1 if (family == "gaussian" and "precision" not in lik) else 0
    comps = []
    for i, c in enumerate(doc.get("components", [])):
        nm = c["name"]
        if nm not in data:
            raise ConfigError(f"components[{i}].{nm}", "index column missing from data")
        graph = None
        if c["kind"] == "besag":
            graph = (graphs or {}).get(nm) or read_graph_file(Path(base_dir) / c["graph_file"])
            size = graph[0].size - 1
        else:
            size = int(c["size"])
        a, b = _hyper(c.get("hyper"), f"components[{i}].hyper")
        comps.append(Component(nm, c["kind"], size, k, obs_index=data[nm].astype(np.int64),
                               graph=graph, hyper_shape=a, hyper_rate=b))
        k += 1
    spec = ModelSpec(m, family, comps, Z=Z, fixed_names=list(fixed),
                     intercept=bool(opts.get("intercept", True)), offsets=data.get("offset"),
                     exposures=data.get("exposure"),
                     noise_precision=float(lik["precision"]) if "precision" in lik else None,
                     noise_hyper=_hyper(lik.get("hyper"), "likelihood.hyper"),
                     fixed_prior_prec=float(opts.get("fixed_prior_precision", DEFAULT_FIXED_PRIOR_PREC)),
                     jitter=float(opts.get("jitter", DEFAULT_JITTER)))
    if family == "poisson" and np.any(y < 0):
        raise ConfigError("data.y", "poisson counts must be non-negative")
    return spec, y


def load_model(model_path, data_path):
    return build_model(read_model_file(model_path), read_data_file(data_path),
                       base_dir=Path(model_path).parent)


# ---------------------------------------------------------------- outputs
def write_marginals_csv(path, result):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["index", "component", "mean", "sd"])
        for i, (lab, mu, sd) in enumerate(zip(result.labels, result.latent_mean, result.latent_sd)):
            w.writerow([i, lab, repr(float(mu)), repr(float(sd))])


def write_hyper_json(path, result, meta: dict | None = None):
    doc = {"hyperparameters": [{"name": h.name, "mode": float(h.mode), "sd": float(h.sd),
                                "table": ([[float(a), float(b)] for a, b in h.table]
                                          if h.table else None)} for h in result.hyper],
           "n_integration_points": int(result.n_points), "meta": meta or {}}
    Path(path).write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def write_fit_outputs(out_dir, result):
    """marginals.csv, hyper.json, trace.jsonl, summary.json (cli.py:64-78)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    write_marginals_csv(out / "marginals.csv", result.marginals)
    write_hyper_json(out / "hyper.json", result.marginals,
                     meta={"budget": str(result.budget), "status": result.optimization.status})
    with open(out / "trace.jsonl", "w") as fh:
        for e in result.optimization.trace:
            fh.write(json.dumps({k: e[k] for k in ("iter", "f", "grad_norm", "step", "n_evals",
                                                   "wall_ms") if k in e}, sort_keys=True) + "\n")
    (out / "summary.json").write_text(json.dumps(result.summary(), indent=2, sort_keys=True) + "\n")


def validate(doc, schema_name: str):
    """Check a document against one of the output contracts (jsonschema)."""
    import jsonschema

    schema = json.loads((SCHEMA_DIR / f"{schema_name}.schema.json").read_text())
    jsonschema.validate(doc, schema)
