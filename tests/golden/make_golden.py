"""Generate golden vectors by running the UNMODIFIED reference package.

Runs only in the build container (needs /root/reference, read-only):

    NUMBA_CACHE_DIR=/tmp/numba_golden python tests/golden/make_golden.py [names...]

The reference has no SPDE / AR(1) components, so it is
driven through the three-patch adapter of SURVEY.md Appendix B: in the
``parinla.objective`` namespace, ``assemble_prior_precision`` returns the
BASELINE prior on one fixed pattern (computed by the oracle's independent
scipy assembler), ``log_prior_hyper`` applies the reference log-gamma formula
to every theta_j, and ``build_design`` returns [Z | A_field].  Everything
numerical after that — ordering, Cholesky, solves, Newton loop, f assembly,
optimizer, selected inversion — is reference code.

Output: ``tests/golden/<case>.npz`` with the instance parameters, a hash of
the generated data (drift detector), f(theta) and its components at a few
theta points, log-determinants, the conditional mode and the marginal
variances at theta_true, and (for fit cases) the reference fit result.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")

import parinla  # noqa: E402
import parinla.objective as ref_objective  # noqa: E402
from parinla.model import Component as RefComponent, ModelSpec as RefSpec  # noqa: E402
from parinla.sparse import SparseSymMatrix as RefSSM  # noqa: E402

from oracle.oracle import OracleModel  # noqa: E402
from paper_2204_04678_b200.synth import make_instance  # noqa: E402

# case -> (config, overrides, do_fit, do_selinv[, options])
# do_fit: False | True (pinned: central FD, 6 candidates) | "defaults" (the
# reference FitConfig defaults: mixed FD, candidates = max(l1, 5) = 5 pinned)
# options: evals (False: fit only), strategy ("eb" | "grid")
CASES = {
    "c1": ("c1", {}, True, True),
    "c2r": ("c2", dict(nx=40, ny=40, m=4000), True, True),
    "c2": ("c2", {}, False, True),
    "c3r": ("c3", dict(nx=12, ny=12, nt=6, m=3000), False, True),
    "c4r": ("c4", dict(nx=16, ny=16, nt=4, m=4000), False, True),
    "c5r": ("c5", dict(nx=16, ny=8, nt=6, m=3000), False, True),
    # full spatial grids at reduced n_t: the BASELINE block sizes (n_s = 3600,
    # 4096, 2048: 57 / 64 / 32 tiles per time block), m scaled with n_t
    "c3g": ("c3", dict(nt=4, m=40_000), False, True),
    "c4g": ("c4", dict(nt=4, m=32_000), False, True),
    "c5g": ("c5", dict(nt=4, m=32_000), False, True),
    # full c2 fits: pinned optimizer settings and the reference defaults
    "c2fit": ("c2", {}, True, False, dict(evals=False)),
    "c2fitd": ("c2", {}, "defaults", False, dict(evals=False)),
    # c1 with the grid integration strategy (explore_grid waves + K selinvs)
    "c1grid": ("c1", {}, True, False, dict(evals=False, strategy="grid")),
}
OFFSETS = [0.0, 0.1, -0.1, 0.3]
# the reference's own model kinds (no adapter: iid / besag are native there),
# instances from synth.reference_kind_instance; general-GMRF ND path
KIND_CASES = {
    "leuk": dict(kind="leukemia-like", fit=False, sample=False, values_subset=4000),
    "grid2d": dict(kind="grid2d", fit=True, sample=True, values_subset=None),
    "leuks": dict(kind="leukemia-like", side=20, m=900, fit=True, sample=True, values_subset=None),
}


def data_hash(inst) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(inst.y).tobytes())
    h.update(np.ascontiguousarray(inst.spec.Z).tobytes())
    for c in inst.spec.components:
        if c.design is not None:
            h.update(c.design.data.tobytes())
            h.update(c.design.indices.astype(np.int64).tobytes())
    return h.hexdigest()


class Adapter:
    """Installs the three patches and builds the reference ModelSpec."""

    def __init__(self, inst):
        self.inst = inst
        spec = inst.spec
        self.om = OracleModel(spec, inst.y)
        n_comp = spec.latent_dim - spec.n_fixed
        comp = RefComponent("field", "iid", n_comp, 1 if spec.family == "gaussian" else 0,
                            obs_index=np.zeros(spec.m, dtype=np.int64))
        rs = RefSpec(spec.m, spec.family, [comp], Z=spec.Z, intercept=False)
        rs.theta_names = tuple(spec.theta_names)
        rs.theta_dim = spec.theta_dim
        self.rs = rs
        self.indptr = self.om.p_indptr
        self.indices = self.om.p_indices

    def install(self):
        om, indptr, indices = self.om, self.indptr, self.indices

        def assemble(spec, theta):
            th = spec.hyper_params(theta).theta
            out = RefSSM.__new__(RefSSM)
            out.n = om.n
            out.indptr = indptr
            out.indices = indices
            out.data = om.prior_values(th)
            return out

        ref_objective.assemble_prior_precision = assemble
        ref_objective.log_prior_hyper = lambda spec, theta: om.log_prior_hyper(
            spec.hyper_params(theta).theta)
        ref_objective.build_design = lambda spec: om.A


def make_case(name):
    cfg, over, do_fit, do_selinv = CASES[name][:4]
    opts = CASES[name][4] if len(CASES[name]) > 4 else {}
    inst = make_instance(cfg, **over)
    ad = Adapter(inst)
    ad.install()
    out = dict(case=name, config=cfg, overrides=json.dumps(over), data_hash=data_hash(inst),
               theta_true=inst.theta_true)
    t0 = time.time()
    inner_tol = 1e-12 if inst.spec.family == "poisson" else 1e-8
    ev = ref_objective.ObjectiveEvaluator(ad.rs, inst.y, inner_tol=inner_tol)
    out["analyze_s"] = time.time() - t0
    out["inner_tol"] = inner_tol
    thetas, comps, lds = [], [], []
    offsets = OFFSETS if cfg in ("c1", "c2") and name != "c2" else OFFSETS[:2]
    if not opts.get("evals", True):
        offsets = []
    for k, off in enumerate(offsets):
        th = inst.theta_true + off * np.cos(np.arange(inst.theta_true.size) + k)
        val, approx = ev.eval_objective(th)
        fac_prior = parinla.factorize(ev.sym_prior, ref_objective.assemble_prior_precision(ad.rs, th))
        thetas.append(th)
        comps.append([val.f, val.log_prior_hyper, val.log_prior_latent, val.log_likelihood,
                      val.log_gaussian_approx, approx.iterations])
        lds.append([approx.factor.log_det, fac_prior.log_det])
        if k == 0:
            out["mode"] = approx.mode
            if do_selinv:
                t1 = time.time()
                si = parinla.selected_inverse(approx.factor)
                out["selinv_s"] = time.time() - t1
                out["variances"] = si.marginal_variances
                out["factor_nnz"] = approx.factor.symbolic.nnz
        print(f"  {name} theta[{k}] f={val.f:.12g} its={approx.iterations}", flush=True)
    if thetas:
        out["thetas"] = np.array(thetas)
        out["f_components"] = np.array(comps)
        out["logdets"] = np.array(lds)
    if do_fit:
        if do_fit == "defaults":
            fd = parinla.FDConfig()
            ls = parinla.LineSearchConfig(candidates=5)
        else:
            fd = parinla.FDConfig(scheme="central")
            ls = parinla.LineSearchConfig(candidates=6)
        strategy = opts.get("strategy", "eb")
        out["fit_config"] = json.dumps(dict(fd=fd.scheme, candidates=ls.candidates,
                                            strategy=strategy))
        t1 = time.time()
        res = parinla.fit(ad.rs, inst.y, parinla.FitConfig(budget=parinla.ThreadBudget(7, 1),
                                                            fd=fd, line_search=ls,
                                                            strategy=strategy))
        out["fit_s"] = time.time() - t1
        out["fit_theta"] = res.theta_mode.theta
        out["fit_f"] = res.f_mode
        out["fit_status"] = res.optimization.status
        out["fit_iterations"] = res.optimization.iterations
        out["fit_n_evals"] = res.optimization.n_evals
        out["fit_hessian"] = res.hessian
        out["fit_latent_mean"] = res.marginals.latent_mean
        out["fit_latent_sd"] = res.marginals.latent_sd
        out["fit_n_points"] = res.marginals.n_points
        out["fit_hyper_sd"] = np.array([h.sd for h in res.marginals.hyper])
        print(f"  {name} fit theta*={res.theta_mode.theta} status={res.optimization.status} "
              f"its={res.optimization.iterations} {out['fit_s']:.1f}s", flush=True)
    np.savez_compressed(os.path.join(os.path.dirname(__file__), f"{name}.npz"), **out)


_ORIGINALS = {k: getattr(ref_objective, k) for k in
              ("assemble_prior_precision", "log_prior_hyper", "build_design")}


def make_kind_case(name):
    """Reference-kind model through the unmodified reference (no patches)."""
    from parinla.ordering import AdjacencyGraph

    from paper_2204_04678_b200.synth import reference_kind_instance

    for k, v in _ORIGINALS.items():
        setattr(ref_objective, k, v)
    opt = KIND_CASES[name]
    inst = reference_kind_instance(opt["kind"], side=opt.get("side"), m=opt.get("m"))
    spec = inst.spec
    comps = []
    for c in spec.components:
        g = None
        if c.graph is not None:
            ip, ix = c.graph
            g = AdjacencyGraph(c.size, ip, ix)
        comps.append(RefComponent(c.name, c.kind, c.size, c.theta_index,
                                  obs_index=np.asarray(c.obs_index, dtype=np.int64), graph=g))
    rs = RefSpec(spec.m, spec.family, comps, Z=spec.Z, fixed_names=spec.fixed_names,
                 intercept=spec.intercept, exposures=spec.exposures)
    assert rs.theta_names == spec.theta_names, (rs.theta_names, spec.theta_names)
    out = dict(case=name, kind=opt["kind"], side=inst.params["side"],
               m=int(spec.m), data_hash=data_hash(inst), theta_true=inst.theta_true)
    inner_tol = 1e-8  # the reference default (fit() uses it too)
    t0 = time.time()
    ev = ref_objective.ObjectiveEvaluator(rs, inst.y, inner_tol=inner_tol)
    out["analyze_s"] = time.time() - t0
    out["inner_tol"] = inner_tol
    sym = ev.sym_cond
    out["perm_cond"] = sym.permutation.perm
    out["perm_prior"] = ev.sym_prior.permutation.perm
    cc = np.diff(sym.Lp).astype(np.float64)
    out["nnz_L"] = sym.nnz
    out["sum_colcount_sq"] = float(np.sum(cc * cc))
    thetas, comps_v, lds = [], [], []
    for k, off in enumerate(OFFSETS):
        th = inst.theta_true + off * np.cos(np.arange(inst.theta_true.size) + k)
        val, approx = ev.eval_objective(th)
        fac_prior = parinla.factorize(ev.sym_prior, ref_objective.assemble_prior_precision(rs, th))
        thetas.append(th)
        comps_v.append([val.f, val.log_prior_hyper, val.log_prior_latent, val.log_likelihood,
                        val.log_gaussian_approx, approx.iterations])
        lds.append([approx.factor.log_det, fac_prior.log_det])
        if k == 0:
            out["mode"] = approx.mode
            t1 = time.time()
            si = parinla.selected_inverse(approx.factor)
            out["selinv_s"] = time.time() - t1
            out["variances"] = si.marginal_variances
            fv, sv = approx.factor.values, si.values
            Lp, Li = sym.Lp, sym.Li
            cols = np.repeat(np.arange(sym.n, dtype=np.int64), np.diff(Lp))
            if opt["values_subset"]:
                rng = np.random.default_rng(0)
                pick = np.sort(rng.choice(fv.size, opt["values_subset"], replace=False))
                pick = np.union1d(pick, Lp[:-1][:: max(1, sym.n // 500)])  # some diagonals
            else:
                pick = np.arange(fv.size)
            out["L_rows"], out["L_cols"] = Li[pick], cols[pick]
            out["L_values"], out["Sigma_values"] = fv[pick], sv[pick]
            if opt["sample"]:
                z = np.random.default_rng(1).standard_normal(sym.n)
                out["sample_z"] = z
                out["sample_x"] = parinla.cholesky.sample_gmrf(approx.factor, z)
        print(f"  {name} theta[{k}] f={val.f:.12g} its={approx.iterations}", flush=True)
    out["thetas"] = np.array(thetas)
    out["f_components"] = np.array(comps_v)
    out["logdets"] = np.array(lds)
    if opt["fit"]:
        fd = parinla.FDConfig(scheme="central")
        ls = parinla.LineSearchConfig(candidates=6)
        t1 = time.time()
        res = parinla.fit(rs, inst.y, parinla.FitConfig(budget=parinla.ThreadBudget(7, 1),
                                                        fd=fd, line_search=ls))
        out["fit_s"] = time.time() - t1
        out["fit_theta"] = res.theta_mode.theta
        out["fit_f"] = res.f_mode
        out["fit_status"] = res.optimization.status
        out["fit_iterations"] = res.optimization.iterations
        out["fit_latent_mean"] = res.marginals.latent_mean
        out["fit_latent_sd"] = res.marginals.latent_sd
        print(f"  {name} fit theta*={res.theta_mode.theta} status={res.optimization.status} "
              f"{out['fit_s']:.1f}s", flush=True)
    np.savez_compressed(os.path.join(os.path.dirname(__file__), f"{name}.npz"), **out)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES) + list(KIND_CASES)
    for nm in names:
        print("case", nm, flush=True)
        if nm in KIND_CASES:
            make_kind_case(nm)
        else:
            make_case(nm)
