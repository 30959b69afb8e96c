"""Negative log hyper-posterior f(theta) on the B200 engine.

Drop-in for the reference ``ObjectiveEvaluator`` (`/root/reference/pkg/src/
parinla/objective.py:104-354`): same constructor arguments, same
``eval_objective`` / ``objective`` / ``gaussian_approx`` / ``stats`` /
``cache_*`` surface, same exceptions (``NotPositiveDefinite`` with the column
in original order, ``InnerDivergence``), same f decomposition

    f = -(log_prior_hyper + log_prior_latent + log_likelihood
          - log_gaussian_approx)

with every term carrying its full constants.  The arithmetic runs in
libpinla (assembly, tile-DAG factorizations, solves, Newton loop); this module
only marshals.  New: :meth:`ObjectiveEvaluator.eval_batch`, which the
optimizer's batch hook uses to put a whole FD stencil / line-search batch on
the device in one call (all slots concurrently).
"""

from __future__ import annotations

import math
import threading
import time
from collections import OrderedDict
from dataclasses import dataclass, field  # noqa: F401

import numpy as np

from .engine import Engine
from .errors import BatchError, DimensionMismatch, InnerDivergence, NotPositiveDefinite
from .model import HyperParams, ModelSpec
from .runtime import SERIAL, ThreadBudget

LOG_2PI = math.log(2.0 * math.pi)
STATUS_OK, STATUS_NOT_PD, STATUS_INNER = 0, 1, 2


@dataclass
class DeviceFactor:
    """Handle to the conditional factor of one theta (the reference's
    CholeskyFactor of Q_c, cholesky.py:168-190).

    The tiles live on the device only while their slot is not reused; the
    factor is re-derived from (theta, warm start) when needed, which is a
    pure function of both (reference contract, objective.py:104-110):
    ``values`` (on ``symbolic``'s scalar pattern, the engine's ordering) and
    ``sample_gmrf`` make it resident first."""

    evaluator: "ObjectiveEvaluator"
    theta: np.ndarray
    warm_start: np.ndarray | None
    log_det: float

    @property
    def n(self) -> int:
        return self.evaluator.n

    @property
    def symbolic(self):
        return self.evaluator.sym_cond

    def make_resident(self):
        """Factor of Q_c(theta) at the mode (from this warm start) in slot 0."""
        self.evaluator._make_resident(self.theta, self.warm_start)

    @property
    def values(self) -> np.ndarray:
        self.make_resident()
        s = self.symbolic
        return self.evaluator.engine.tile_entries(0, 0, s.Li, s.entry_columns())

    def factor_diagonal(self) -> np.ndarray:
        return self.values[self.symbolic.Lp[:-1]]


class GaussianApprox:
    """Gaussian match to p(x | theta, y) (reference objective.py:39-50).
    ``cond_precision`` (Q_c at the mode, a SparseSymMatrix on the
    conditional pattern, original order) is read from the device on first
    access when it was not given."""

    def __init__(self, theta: HyperParams, mode, cond_precision, factor: DeviceFactor,
                 iterations: int, inner_trace=None):
        self.theta = theta
        self.mode = mode
        self._cond = cond_precision
        self.factor = factor
        self.iterations = iterations
        self.inner_trace = [] if inner_trace is None else inner_trace

    @property
    def cond_precision(self):
        if self._cond is None and isinstance(self.factor, DeviceFactor):
            self._cond = self.factor.evaluator.cond_precision(self.factor.theta,
                                                              self.factor.warm_start)
        return self._cond


@dataclass
class ObjectiveValue:
    """One f(theta) with its additive pieces (reference objective.py:53-76)."""

    f: float
    log_prior_hyper: float
    log_prior_latent: float
    log_likelihood: float
    log_gaussian_approx: float
    timings: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        return {
            "f": self.f,
            "log_prior_hyper": self.log_prior_hyper,
            "log_prior_latent": self.log_prior_latent,
            "log_likelihood": self.log_likelihood,
            "log_gaussian_approx": self.log_gaussian_approx,
            "timings": dict(self.timings),
        }


_ORDERING_ALIASES = {"nested-dissection": "structured"}
# "structured": lattice ND (2-D fields) / time-major BTA (spatio-temporal),
# else the reference's nested dissection (native, separator-aligned tiles);
# "minimum-degree": the reference's minimum degree; "band": row-major band
# for 2-D fields; "rcm": reverse Cuthill-McKee


class ObjectiveEvaluator:
    """Evaluates f(theta) = -log p~(theta | y) on one B200.

    ``ordering``: the reference's names are accepted; "nested-dissection"
    (the reference default) maps to the engine's ``structured`` ordering
    (lattice ND / BTA tiles for lattice and ST models, otherwise the
    reference's own nested dissection with ``leaf_cutoff``, natively, on
    separator-aligned tiles).
    ``max_slots``: theta points resident concurrently on the device
    (default 2d+1, the central FD batch width).
    """

    def __init__(self, spec: ModelSpec, y, A=None, ordering: str = "nested-dissection",
                 leaf_cutoff: int = 64, inner_tol: float = 1e-8, max_inner: int = 50,
                 cache_size: int | None = None, max_slots: int | None = None,
                 device: int | None = None, analytic_prior_logdet: bool = True):
        self.spec = spec
        self.y = np.asarray(y, dtype=np.float64)
        if self.y.shape != (spec.m,):
            raise DimensionMismatch("y must have length m")
        self.inner_tol = float(inner_tol)
        self.max_inner = int(max_inner)
        d = max(spec.theta_dim, 1)
        slots = max_slots if max_slots is not None else 2 * d + 1
        t0 = time.perf_counter()
        self.engine = Engine(spec, self.y, A=A, ordering=_ORDERING_ALIASES.get(ordering, ordering),
                             max_slots=slots, inner_tol=inner_tol, max_inner=max_inner,
                             device=device, analytic_prior_logdet=analytic_prior_logdet,
                             leaf_cutoff=leaf_cutoff)
        self.analyze_s = time.perf_counter() - t0
        self.A = self.engine.A
        self._lock = threading.Lock()
        self.n_evaluations = 0
        self.analyze_calls = 1
        self._cache_size = cache_size if cache_size is not None else 2 * d + 1
        self._cache: OrderedDict = OrderedDict()
        self.engine_calls = 0      # device calls that may overwrite slot 0 / Sigma
        self._resident = None      # (engine_calls, theta, warm) whose factor is in slot 0
        self._sym_cond = None

    @property
    def sym_cond(self):
        """SymbolicFactor of the conditional pattern under the engine's
        ordering (the reference's ``sym_cond``, objective.py:160); its scalar
        pattern is computed on first use."""
        if self._sym_cond is None:
            from .cholesky import SymbolicFactor

            ip, ix = self.engine.cond_pattern()
            self._sym_cond = SymbolicFactor(self.n, self.engine.perm, self.engine, ip, ix,
                                            self.engine.ordering)
        return self._sym_cond

    def _mark(self, theta=None, warm=None):
        self.engine_calls += 1
        self._resident = None if theta is None else (
            self.engine_calls, np.asarray(theta, dtype=np.float64).tobytes(),
            None if warm is None else np.asarray(warm, dtype=np.float64).tobytes())

    def _is_resident(self, theta, warm) -> bool:
        r = self._resident
        return r is not None and r[0] == self.engine_calls and \
            r[1] == np.asarray(theta, dtype=np.float64).tobytes() and \
            r[2] == (None if warm is None else np.asarray(warm, dtype=np.float64).tobytes())

    def _make_resident(self, theta, warm):
        if not self._is_resident(theta, warm):
            x, its, st, bc, ld = self.engine.mode(self._hp(theta).theta, self._warm(warm))
            self._mark(theta, warm)
            self._raise_for(st, bc, self._hp(theta).theta)

    def cond_precision(self, theta, warm_start=None):
        """Q_c(theta) at the conditional mode (original order, lower CSC)."""
        from .sparse import SparseSymMatrix

        self._make_resident(theta, warm_start)
        ip, ix = self.engine.cond_pattern()
        return SparseSymMatrix(self.n, ip, ix, self.engine.cond_values(0), validate=False)

    @property
    def n(self) -> int:
        return self.spec.latent_dim

    def stats(self) -> dict:
        es = self.engine.stats()
        with self._lock:
            return {
                "n_evaluations": self.n_evaluations,
                "n_factorizations": es["n_factorizations"],
                "analyze_calls": self.analyze_calls,
                "nnz_factor_prior": es["n_tiles"] * 64 * 64,
                "nnz_factor_cond": es["n_tiles"] * 64 * 64,
                "engine": es,
            }

    # ------------------------------------------------------------------
    def _hp(self, theta) -> HyperParams:
        return self.spec.hyper_params(theta)

    def _warm(self, warm_start, k: int | None = None):
        """One warm start (n,) or, for batches, one per point (k, n)."""
        if warm_start is None:
            return None
        w = np.asarray(warm_start, dtype=np.float64)
        if w.shape != (self.n,) and not (k is not None and w.shape == (k, self.n)):
            raise DimensionMismatch("warm start must have the latent dimension")
        return w

    @staticmethod
    def _raise_for(status: int, badcol: int, theta):
        if status == STATUS_NOT_PD:
            raise NotPositiveDefinite(badcol)
        if status == STATUS_INNER:
            raise InnerDivergence(theta, "no ascent step found or not converged")

    def _values(self, points, warm_start, want_modes=False):
        th = np.stack([self._hp(p).theta for p in points]) if len(points) else np.zeros((0, self.spec.theta_dim))
        t0 = time.perf_counter()
        res = self.engine.eval_batch(th, self._warm(warm_start, len(points)), want_modes=want_modes)
        self._mark()
        wall = time.perf_counter() - t0
        with self._lock:
            # the reference counts an evaluation once its Newton loop and the
            # prior factorization succeeded (objective.py:309)
            self.n_evaluations += int(np.count_nonzero(res["status"] == STATUS_OK))
        res["theta"] = th
        res["wall_s"] = wall
        return res

    def eval_objective(self, theta, warm_start=None, budget: ThreadBudget = SERIAL):
        """f(theta) together with the Gaussian approximation it used
        (reference objective.py:298-331)."""
        res = self._values([theta], warm_start, want_modes=True)
        hp = self._hp(res["theta"][0])
        st, bc = int(res["status"][0]), int(res["badcol"][0])
        self._raise_for(st, bc, hp.theta)
        c = res["comps"][0]
        value = ObjectiveValue(
            f=float(c[0]), log_prior_hyper=float(c[1]), log_prior_latent=float(c[2]),
            log_likelihood=float(c[3]), log_gaussian_approx=float(c[4]),
            timings={"mode_s": res["wall_s"], "total_s": res["wall_s"],
                     "inner_iterations": int(res["iters"][0])},
        )
        fac = DeviceFactor(self, hp.theta.copy(), None if warm_start is None else np.array(warm_start),
                           float(res["logdets"][0, 0]))
        approx = GaussianApprox(hp, res["modes"][0], None, fac, int(res["iters"][0]))
        return value, approx

    def objective(self, theta, warm_start=None, budget: ThreadBudget = SERIAL) -> float:
        return self.eval_objective(theta, warm_start, budget)[0].f

    def eval_values(self, points, warm_start=None, want_modes: bool = False):
        """Per-point ObjectiveValue or the exception the reference would raise
        (with ``want_modes`` also the conditional modes, k x n)."""
        res = self._values(list(points), warm_start, want_modes=want_modes)
        out = []
        for s in range(len(points)):
            st, bc = int(res["status"][s]), int(res["badcol"][s])
            if st != STATUS_OK:
                try:
                    self._raise_for(st, bc, res["theta"][s])
                except (NotPositiveDefinite, InnerDivergence) as exc:
                    out.append(exc)
                continue
            c = res["comps"][s]
            out.append(ObjectiveValue(float(c[0]), float(c[1]), float(c[2]), float(c[3]),
                                      float(c[4]), {"inner_iterations": int(res["iters"][s])}))
        if want_modes:
            return out, res["modes"]
        return out

    def eval_batch(self, points, warm_start=None):
        """f at every point in one device batch; the lowest failing slot is
        raised as BatchError (the reference run_batch contract)."""
        vals = self.eval_values(points, warm_start)
        for slot, v in enumerate(vals):
            if isinstance(v, Exception):
                raise BatchError(slot, v) from v
        return [v.f for v in vals]

    def gaussian_approx(self, theta, warm_start=None, budget: ThreadBudget = SERIAL) -> GaussianApprox:
        """Conditional mode and factor at fixed theta (objective.py:218-233)."""
        hp = self._hp(theta)
        w = self._warm(warm_start)
        x, its, st, bc, ld = self.engine.mode(hp.theta, w)
        self._mark(hp.theta, w)
        self._raise_for(st, bc, hp.theta)
        fac = DeviceFactor(self, hp.theta.copy(), None if w is None else w.copy(), ld)
        return GaussianApprox(hp, x, None, fac, its)

    def marginal_variances(self, theta, warm_start=None):
        """diag(Q_c(theta)^-1) in original order plus the mode."""
        hp = self._hp(theta)
        w = self._warm(warm_start)
        var, x, st, bc = self.engine.selinv_diag(hp.theta, w)
        self._mark(hp.theta, w)
        self._raise_for(st, bc, hp.theta)
        return var, x

    # cache (objective.py:339-354)
    def cache_put(self, theta, approx: GaussianApprox):
        key = np.asarray(theta, dtype=np.float64).tobytes()
        with self._lock:
            self._cache[key] = approx
            self._cache.move_to_end(key)
            while len(self._cache) > self._cache_size:
                self._cache.popitem(last=False)

    def cache_get(self, theta):
        key = np.asarray(theta, dtype=np.float64).tobytes()
        with self._lock:
            return self._cache.get(key)

    def cache_clear(self):
        with self._lock:
            self._cache.clear()

    def close(self):
        self.engine.close()
