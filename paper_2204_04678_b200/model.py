"""Latent Gaussian model: theta layout, prior precision plan, likelihood.

Mirrors the reference model surface (`/root/reference/pkg/src/parinla/
model.py:31-356`: ``HyperParams``, ``Component``, ``ModelSpec``,
``assemble_prior_precision``, ``log_prior_hyper``, ``likelihood_terms``,
``build_design``) and extends the component kinds with the fields the
BASELINE configurations need:

* ``spde2d``      Q = tau (kappa^4 I + 2 kappa^2 G + G^2), G = lattice graph
                  Laplacian D - W; theta = (log tau, log kappa).
* ``ar1``         Q = tau Q_AR1(rho); theta = (log tau, logit rho).
* ``ar1_spde2d``  Q = Q_AR1(rho) (x) Q_spde(tau, kappa), time-major;
                  theta = (log tau, log kappa, logit rho).

The prior precision is a fixed pattern whose values are a short sum of
theta-gains times constant basis coefficients (``PriorPlan``):
``value[e] = sum_t coef[t] * gain[gain_id[t]] + const[e]`` over the terms
``t`` of entry ``e``.  For the reference kinds every entry has exactly one
term (gain exp(theta_c)) and ``const`` holds the diagonal jitter / the fixed
block precision, which reproduces reference `model.py:263-282` bit for bit.
The same plan is uploaded once to the device and evaluated there per theta.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .errors import ConfigError, DimensionMismatch, StructureError
from .sparse import SparseSymMatrix

COMPONENT_KINDS = ("iid", "rw1", "rw2", "besag", "spde2d", "ar1", "ar1_spde2d")
THETA_PER_KIND = {"iid": 1, "rw1": 1, "rw2": 1, "besag": 1, "spde2d": 2, "ar1": 2, "ar1_spde2d": 3}

DEFAULT_FIXED_PRIOR_PREC = 1e-3
DEFAULT_JITTER = 1e-5
DEFAULT_HYPER_SHAPE = 1.0
DEFAULT_HYPER_RATE = 5e-5
LOG_2PI = math.log(2.0 * math.pi)


@dataclass(frozen=True)
class HyperParams:
    """Log-scale hyperparameters with their labels (reference `model.py:31-47`)."""

    theta: np.ndarray
    names: tuple

    def __post_init__(self):
        th = np.atleast_1d(np.asarray(self.theta, dtype=np.float64))
        object.__setattr__(self, "theta", th)
        if not np.all(np.isfinite(th)):
            raise StructureError("hyperparameters must be finite")
        if len(self.names) != th.shape[0]:
            raise DimensionMismatch("names and theta disagree")

    @property
    def dim(self) -> int:
        return int(self.theta.shape[0])


class LatticeGraph:
    """4-neighbour nx-by-ny lattice, vertex id = row * nx + col (row-major)."""

    def __init__(self, nx: int, ny: int):
        self.nx, self.ny = int(nx), int(ny)
        self.n = self.nx * self.ny

    def laplacian(self) -> sp.csr_matrix:
        """Graph Laplacian D - W with natural boundary degrees (2..4)."""
        idx = np.arange(self.n).reshape(self.ny, self.nx)
        u = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
        v = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
        W = sp.coo_matrix((np.ones(u.size), (u, v)), shape=(self.n, self.n))
        W = (W + W.T).tocsr()
        deg = np.asarray(W.sum(axis=1)).ravel()
        return (sp.diags(deg) - W).tocsr()

    def adjacency_lists(self):
        L = self.laplacian().tocsr()
        L.setdiag(0)
        L.eliminate_zeros()
        return L.indptr.astype(np.int64), L.indices.astype(np.int64)


@dataclass
class Component:
    """One latent block (reference `model.py:50-61`, extended).

    ``obs_index`` maps each observation to one level with coefficient 1
    (reference design); alternatively ``design`` gives an explicit m-by-size
    sparse projection (bilinear SPDE projection).  ``graph`` is an adjacency
    (indptr, indices) pair for ``besag`` or a :class:`LatticeGraph` for the
    lattice kinds; ``nt`` is the number of time points for the AR(1) kinds.
    """

    name: str
    kind: str
    size: int
    theta_index: int
    obs_index: np.ndarray | None = None
    graph: object = None
    hyper_shape: float = DEFAULT_HYPER_SHAPE
    hyper_rate: float = DEFAULT_HYPER_RATE
    design: object = None
    nt: int = 1

    @property
    def n_theta(self) -> int:
        return THETA_PER_KIND[self.kind]


class ModelSpec:
    """Structure, data bindings and priors of one latent Gaussian model.

    Same constructor and theta layout as reference `model.py:64-185`: the
    gaussian noise log-precision comes first when it is free, then every
    component's hyperparameters in order.
    """

    def __init__(
        self,
        m: int,
        family: str,
        components: list,
        Z=None,
        fixed_names=None,
        intercept: bool = True,
        offsets=None,
        exposures=None,
        noise_precision=None,
        noise_hyper=(DEFAULT_HYPER_SHAPE, DEFAULT_HYPER_RATE),
        fixed_prior_prec: float = DEFAULT_FIXED_PRIOR_PREC,
        jitter: float = DEFAULT_JITTER,
    ):
        if family not in ("gaussian", "poisson"):
            raise ConfigError("likelihood.family", f"unknown family {family!r}")
        self.m = int(m)
        self.family = family
        self.components = list(components)
        self.Z = np.zeros((m, 0)) if Z is None else np.asarray(Z, dtype=np.float64)
        if self.Z.shape[0] != m:
            raise DimensionMismatch("covariate matrix row count differs from m")
        self.fixed_names = list(fixed_names or [f"x{i}" for i in range(self.Z.shape[1])])
        if len(self.fixed_names) != self.Z.shape[1]:
            raise DimensionMismatch("fixed effect names do not match covariates")
        self.intercept = bool(intercept)
        self.offsets = np.zeros(m) if offsets is None else np.asarray(offsets, dtype=np.float64)
        self.exposures = np.ones(m) if exposures is None else np.asarray(exposures, dtype=np.float64)
        if self.offsets.shape != (m,) or self.exposures.shape != (m,):
            raise DimensionMismatch("offsets/exposures must have length m")
        if family == "poisson" and np.any(self.exposures <= 0):
            raise ConfigError("exposure", "poisson exposures must be positive")
        self.noise_precision = noise_precision
        self.noise_hyper = noise_hyper
        self.fixed_prior_prec = float(fixed_prior_prec)
        self.jitter = float(jitter)

        names: list[str] = []
        self.noise_theta = None
        if family == "gaussian" and noise_precision is None:
            self.noise_theta = 0
            names.append("log_prec_noise")
        for comp in self.components:
            if comp.kind not in COMPONENT_KINDS:
                raise ConfigError(f"components.{comp.name}.kind", f"unknown kind {comp.kind!r}")
            if comp.theta_index != len(names):
                raise ConfigError(
                    f"components.{comp.name}.theta_index",
                    f"expected {len(names)}, got {comp.theta_index}",
                )
            names.extend(_theta_labels(comp))
            _validate_component(comp, m)
        self.theta_names = tuple(names)
        self.theta_dim = len(names)
        self.n_fixed = self.Z.shape[1] + (1 if self.intercept else 0)
        self.latent_dim = self.n_fixed + sum(c.size for c in self.components)
        if self.latent_dim < 1:
            raise ConfigError("model", "latent field is empty")
        self._prior_plan = build_prior_plan(self)
        self._labels = None

    # ------------------------------------------------------------------
    def block_slices(self):
        out, ofs = [], 0
        if self.intercept:
            out.append(("intercept", slice(0, 1)))
            ofs = 1
        for nm in self.fixed_names:
            out.append((f"beta:{nm}", slice(ofs, ofs + 1)))
            ofs += 1
        for comp in self.components:
            out.append((comp.name, slice(ofs, ofs + comp.size)))
            ofs += comp.size
        return out

    def component_offset(self, comp: Component) -> int:
        for nm, sl in self.block_slices():
            if nm == comp.name:
                return sl.start
        raise KeyError(comp.name)

    def latent_labels(self):
        if self._labels is None:
            labels = []
            for nm, sl in self.block_slices():
                if nm == "intercept" or nm.startswith("beta:"):
                    labels.append(nm)
                else:
                    labels.extend(f"{nm}[{i}]" for i in range(sl.stop - sl.start))
            self._labels = labels
        return list(self._labels)

    def hyper_params(self, theta) -> HyperParams:
        theta = np.atleast_1d(np.asarray(theta, dtype=np.float64))
        if theta.shape[0] != self.theta_dim:
            raise DimensionMismatch(
                f"theta has dimension {theta.shape[0]}, model needs {self.theta_dim}"
            )
        return HyperParams(theta=theta, names=self.theta_names)

    def hyper_shapes_rates(self):
        shapes = np.empty(self.theta_dim)
        rates = np.empty(self.theta_dim)
        if self.noise_theta is not None:
            shapes[self.noise_theta], rates[self.noise_theta] = self.noise_hyper
        for comp in self.components:
            k = comp.theta_index
            shapes[k : k + comp.n_theta] = comp.hyper_shape
            rates[k : k + comp.n_theta] = comp.hyper_rate
        return shapes, rates

    def prior_logdet_terms(self):
        """Closed-form log det Q_prior(theta) as engine terms, or None when a
        component has no closed form (reference kinds: factorize instead)."""
        kinds, thetas, dims, values = [], [], [], []
        if self.n_fixed:
            kinds.append(0)
            thetas.append(0)
            dims.append((0, 0, 0))
            values.append(self.n_fixed * math.log(self.fixed_prior_prec))
        for c in self.components:
            if c.kind == "spde2d":
                kinds.append(1)
                dims.append((c.graph.nx, c.graph.ny, 1))
            elif c.kind == "ar1_spde2d":
                kinds.append(2)
                dims.append((c.graph.nx, c.graph.ny, c.nt))
            elif c.kind == "ar1":
                kinds.append(3)
                dims.append((0, 0, c.nt))
            else:
                return None
            thetas.append(c.theta_index)
            values.append(0.0)
        return kinds, thetas, dims, values

    def noise_tau(self, theta) -> float:
        if self.noise_theta is not None:
            return float(np.exp(np.asarray(theta, dtype=np.float64)[self.noise_theta]))
        return float(self.noise_precision)

    def __repr__(self):
        return (
            f"ModelSpec(m={self.m}, family={self.family!r}, latent={self.latent_dim}, "
            f"theta={self.theta_dim})"
        )


def _theta_labels(comp):
    if comp.kind in ("iid", "rw1", "rw2", "besag"):
        return [f"log_prec_{comp.name}"]
    if comp.kind == "spde2d":
        return [f"log_tau_{comp.name}", f"log_kappa_{comp.name}"]
    if comp.kind == "ar1":
        return [f"log_prec_{comp.name}", f"logit_rho_{comp.name}"]
    return [f"log_tau_{comp.name}", f"log_kappa_{comp.name}", f"logit_rho_{comp.name}"]


def _validate_component(comp, m):
    if comp.design is None:
        if comp.obs_index is None:
            raise ConfigError(f"components.{comp.name}", "needs obs_index or design")
        comp.obs_index = np.asarray(comp.obs_index, dtype=np.int64)
        if comp.obs_index.shape != (m,):
            raise DimensionMismatch(f"component {comp.name} index column must have length m")
        if comp.obs_index.min(initial=0) < 0 or comp.obs_index.max(initial=0) >= comp.size:
            raise ConfigError(f"components.{comp.name}", "observation index out of range")
    else:
        comp.design = sp.csr_matrix(comp.design)
        if comp.design.shape != (m, comp.size):
            raise DimensionMismatch(f"component {comp.name} design must be m x size")
    if comp.kind == "rw1" and comp.size < 2:
        raise ConfigError(f"components.{comp.name}.size", "rw1 needs size >= 2")
    if comp.kind == "rw2" and comp.size < 3:
        raise ConfigError(f"components.{comp.name}.size", "rw2 needs size >= 3")
    if comp.kind == "besag":
        g = comp.graph
        if g is None:
            raise ConfigError(f"components.{comp.name}.graph", "besag needs a graph")
        n_g = g.n if hasattr(g, "n") else len(g[0]) - 1
        if n_g != comp.size:
            raise ConfigError(f"components.{comp.name}.graph", "besag needs a graph of matching size")
    if comp.kind in ("spde2d", "ar1_spde2d"):
        if not isinstance(comp.graph, LatticeGraph):
            raise ConfigError(f"components.{comp.name}.graph", "lattice kinds need a LatticeGraph")
        expect = comp.graph.n * (comp.nt if comp.kind == "ar1_spde2d" else 1)
        if expect != comp.size:
            raise ConfigError(f"components.{comp.name}.size", f"expected {expect}")
    if comp.kind == "ar1" and comp.size != comp.nt:
        raise ConfigError(f"components.{comp.name}.nt", "ar1 size must equal nt")


# ----------------------------------------------------------------------
# structure matrices (lower-triangle COO)


def _tril_coo(M):
    T = sp.tril(sp.coo_matrix(M)).tocoo()
    T.eliminate_zeros()
    return T.row.astype(np.int64), T.col.astype(np.int64), T.data.astype(np.float64)


def structure_matrix(kind: str, size: int, graph=None):
    """Lower COO of the unit-precision roughness structure (reference kinds,
    reference `model.py:192-219`)."""
    if kind == "iid":
        i = np.arange(size, dtype=np.int64)
        return i, i, np.ones(size)
    if kind == "rw1":
        D = sp.diags([-np.ones(size - 1), np.ones(size - 1)], [0, 1], shape=(size - 1, size))
        return _tril_coo(D.T @ D)
    if kind == "rw2":
        D = sp.diags(
            [np.ones(size - 2), -2.0 * np.ones(size - 2), np.ones(size - 2)],
            [0, 1, 2],
            shape=(size - 2, size),
        )
        return _tril_coo(D.T @ D)
    if kind == "besag":
        indptr, indices = (graph.indptr, graph.indices) if hasattr(graph, "indptr") else graph
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int64)
        deg = np.diff(indptr).astype(np.float64)
        cols = np.repeat(np.arange(size, dtype=np.int64), np.diff(indptr))
        low = indices > cols
        rows = np.concatenate([np.arange(size, dtype=np.int64), indices[low]])
        cs = np.concatenate([np.arange(size, dtype=np.int64), cols[low]])
        return rows, cs, np.concatenate([deg, -np.ones(int(low.sum()))])
    raise ConfigError("kind", f"unknown component kind {kind!r}")


def ar1_bases(nt: int):
    """E0 = I, E1 = interior-diagonal indicator, E2 = first off-diagonals:
    Q_AR1(rho) = (E0 + rho^2 E1 - rho E2) / (1 - rho^2)."""
    E0 = sp.identity(nt, format="csr")
    d1 = np.ones(nt)
    d1[0] = 0.0
    d1[-1] = 0.0
    E1 = sp.diags(d1, 0, format="csr")
    off = np.ones(nt - 1)
    E2 = sp.diags([off, off], [-1, 1], shape=(nt, nt), format="csr")
    return [E0, E1, E2]


def spde_bases(graph: LatticeGraph):
    G = graph.laplacian()
    return [sp.identity(graph.n, format="csr"), G, (G @ G).tocsr()]


def spde_gains(log_tau, log_kappa):
    tau = np.exp(log_tau)
    k2 = np.exp(2.0 * log_kappa)
    return np.array([tau * k2 * k2, 2.0 * tau * k2, tau])


def ar1_gains(logit_rho):
    rho = 1.0 / (1.0 + np.exp(-logit_rho))
    s = 1.0 / (1.0 - rho * rho)
    return np.array([s, rho * rho * s, -rho * s])


def dense_vertex_cut(n: int) -> int:
    """Degree at which a vertex is treated as dense (reference ND peel,
    `ordering.py:221-226`)."""
    return max(16, (n - 1) // 2)


# ----------------------------------------------------------------------
# prior plan


@dataclass
class PriorPlan:
    """Q_prior(theta) on a fixed lower-CSC pattern (original latent order).

    Terms sorted by (entry, gain id).  ``gain_index`` lists, per gain id, how
    the gain is computed from theta: (kind, theta_offset, sub) triples
    evaluated by :func:`prior_gains`.
    """

    n: int
    indptr: np.ndarray
    indices: np.ndarray
    term_entry: np.ndarray  # int64 [T]
    term_gain: np.ndarray  # int32 [T]
    term_coef: np.ndarray  # float64 [T]
    const: np.ndarray  # float64 [nnz]
    gain_spec: list = field(default_factory=list)

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    @property
    def n_gains(self) -> int:
        return len(self.gain_spec)


def build_prior_plan(spec: ModelSpec) -> PriorPlan:
    n = spec.latent_dim
    rows, cols, coefs, gids, consts_r, consts_c, consts_v = [], [], [], [], [], [], []
    gain_spec: list = []
    if spec.n_fixed:
        i = np.arange(spec.n_fixed, dtype=np.int64)
        consts_r.append(i)
        consts_c.append(i)
        consts_v.append(np.full(spec.n_fixed, spec.fixed_prior_prec))
    for comp in spec.components:
        ofs = spec.component_offset(comp)
        k = comp.theta_index
        if comp.kind in ("iid", "rw1", "rw2", "besag"):
            r, c, v = structure_matrix(comp.kind, comp.size, comp.graph)
            g = len(gain_spec)
            gain_spec.append(("exp", k, 0))
            rows.append(r + ofs)
            cols.append(c + ofs)
            coefs.append(v)
            gids.append(np.full(r.size, g, dtype=np.int32))
            d = np.arange(comp.size, dtype=np.int64) + ofs
            consts_r.append(d)
            consts_c.append(d)
            consts_v.append(np.full(comp.size, spec.jitter))
        elif comp.kind == "spde2d":
            for b, B in enumerate(spde_bases(comp.graph)):
                r, c, v = _tril_coo(B)
                g = len(gain_spec)
                gain_spec.append(("spde", k, b))
                rows.append(r + ofs)
                cols.append(c + ofs)
                coefs.append(v)
                gids.append(np.full(r.size, g, dtype=np.int32))
        elif comp.kind == "ar1":
            for a, E in enumerate(ar1_bases(comp.nt)):
                r, c, v = _tril_coo(E)
                g = len(gain_spec)
                gain_spec.append(("ar1", k, a))
                rows.append(r + ofs)
                cols.append(c + ofs)
                coefs.append(v)
                gids.append(np.full(r.size, g, dtype=np.int32))
        else:  # ar1_spde2d, time-major kron(E_a, B_b)
            Es = ar1_bases(comp.nt)
            Bs = spde_bases(comp.graph)
            for a, E in enumerate(Es):
                for b, B in enumerate(Bs):
                    r, c, v = _tril_coo(sp.kron(E, B, format="coo"))
                    if r.size == 0:
                        continue
                    g = len(gain_spec)
                    gain_spec.append(("st", k, 3 * a + b))
                    rows.append(r + ofs)
                    cols.append(c + ofs)
                    coefs.append(v)
                    gids.append(np.full(r.size, g, dtype=np.int32))
    R = np.concatenate(rows + consts_r)
    C = np.concatenate(cols + consts_c)
    key = C * n + R
    ukey = np.unique(key)
    pc, pr = ukey // n, ukey % n
    # every column needs its diagonal
    if not np.array_equal(np.unique(pc[pr == pc]), np.arange(n)):
        missing = np.setdiff1d(np.arange(n), pc[pr == pc])
        ukey = np.unique(np.concatenate([ukey, missing * n + missing]))
        pc, pr = ukey // n, ukey % n
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, pc + 1, 1)
    np.cumsum(indptr, out=indptr)
    if rows:
        tr = np.concatenate(rows)
        tc = np.concatenate(cols)
        tcoef = np.concatenate(coefs)
        tg = np.concatenate(gids)
        te = np.searchsorted(ukey, tc * n + tr)
        order = np.lexsort((tg, te))
        te, tg, tcoef = te[order], tg[order], tcoef[order]
    else:
        te = np.zeros(0, np.int64)
        tg = np.zeros(0, np.int32)
        tcoef = np.zeros(0)
    const = np.zeros(ukey.size)
    if consts_r:
        cr = np.concatenate(consts_r)
        cc = np.concatenate(consts_c)
        np.add.at(const, np.searchsorted(ukey, cc * n + cr), np.concatenate(consts_v))
    return PriorPlan(n, indptr, pr.astype(np.int64), te.astype(np.int64), tg.astype(np.int32),
                     tcoef.astype(np.float64), const, gain_spec)


def prior_gains(plan: PriorPlan, theta) -> np.ndarray:
    """Gain vector for one theta (host scalar work; uploaded per slot)."""
    th = np.asarray(theta, dtype=np.float64)
    out = np.empty(plan.n_gains)
    with np.errstate(over="ignore"):
        for g, (kind, k, sub) in enumerate(plan.gain_spec):
            if kind == "exp":
                out[g] = np.exp(th[k])
            elif kind == "spde":
                out[g] = spde_gains(th[k], th[k + 1])[sub]
            elif kind == "ar1":
                out[g] = np.exp(th[k]) * ar1_gains(th[k + 1])[sub]
            else:
                a, b = divmod(sub, 3)
                out[g] = ar1_gains(th[k + 2])[a] * spde_gains(th[k], th[k + 1])[b]
    return out


def assemble_prior_precision(spec: ModelSpec, theta) -> SparseSymMatrix:
    """Q_prior(theta) on the theta-invariant pattern (host reference path,
    used for diagnostics and tests; the device evaluates the same plan)."""
    hp = spec.hyper_params(theta)
    plan = spec._prior_plan
    gains = prior_gains(plan, hp.theta)
    vals = np.zeros(plan.nnz)
    with np.errstate(over="ignore", invalid="ignore"):
        np.add.at(vals, plan.term_entry, plan.term_coef * gains[plan.term_gain])
        vals = vals + plan.const
    out = SparseSymMatrix.__new__(SparseSymMatrix)
    out.n, out.indptr, out.indices, out.data = plan.n, plan.indptr, plan.indices, vals
    return out


def log_prior_hyper(spec: ModelSpec, theta) -> float:
    """Sum over j of the log-gamma(a_j, b_j) density of exp(theta_j) plus the
    log-scale Jacobian theta_j (reference `model.py:285-299`)."""
    hp = spec.hyper_params(theta)
    a, b = spec.hyper_shapes_rates()
    th = hp.theta
    terms = a * np.log(b) + a * th - b * np.exp(th)
    terms -= np.array([math.lgamma(v) for v in a])
    return float(np.sum(terms))


def likelihood_terms(spec: ModelSpec, eta, y, theta):
    """(loglik, d1, d2) in the linear predictor (reference `model.py:302-331`).

    Host version, used by tests and diagnostics; the device kernels compute the
    same quantities (`csrc/lik.cu`)."""
    eta = np.asarray(eta, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if eta.shape != (spec.m,) or y.shape != (spec.m,):
        raise DimensionMismatch("eta and y must have length m")
    full = eta + spec.offsets
    if spec.family == "gaussian":
        tau = spec.noise_tau(theta)
        r = y - full
        ll = 0.5 * spec.m * (math.log(tau) - LOG_2PI) - 0.5 * tau * float(r @ r)
        return ll, tau * r, np.full(spec.m, -tau)
    from scipy.special import gammaln

    if np.any(y < 0) or not np.all(np.isfinite(y)):
        raise StructureError("poisson observations must be finite and non-negative")
    mu = spec.exposures * np.exp(full)
    ll = float(np.sum(y * full + y * np.log(spec.exposures)) - np.sum(mu) - np.sum(gammaln(y + 1.0)))
    return ll, y - mu, -mu


def build_design(spec: ModelSpec) -> sp.csr_matrix:
    """m x n design A with eta = A x (reference `model.py:334-356`, plus
    explicit projection designs for the lattice kinds)."""
    blocks = []
    if spec.intercept:
        blocks.append(sp.csr_matrix(np.ones((spec.m, 1))))
    if spec.Z.shape[1]:
        blocks.append(sp.csr_matrix(spec.Z))
    rows = np.arange(spec.m, dtype=np.int64)
    for comp in spec.components:
        if comp.design is not None:
            blocks.append(sp.csr_matrix(comp.design))
        else:
            blocks.append(
                sp.csr_matrix((np.ones(spec.m), (rows, comp.obs_index)), shape=(spec.m, comp.size))
            )
    A = sp.hstack(blocks, format="csr") if blocks else sp.csr_matrix((spec.m, 0))
    if A.shape[1] != spec.latent_dim:
        raise StructureError("design width disagrees with the latent dimension")
    if np.any(np.diff(A.indptr) < 1):
        raise StructureError("every observation needs at least one design entry")
    A.sort_indices()
    return A
