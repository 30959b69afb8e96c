"""Sparse SPD factorization, solves and selected inversion on the device.

Drop-in for the reference's `cholesky.py` surface (`/root/reference/pkg/
src/parinla/cholesky.py:88-400`): ``analyze`` -> ``SymbolicFactor``,
``factorize`` -> ``CholeskyFactor`` (with ``log_det``, raising
``NotPositiveDefinite(column)`` in original order), ``solve``,
``selected_inverse`` -> ``SelectedInverse`` (``marginal_variances`` in original
order).  The factor is a tile factor resident on the device (64x64 dense
tiles, ordering-dependent), so the reference's scalar ``values`` array on
its own ND pattern has no equivalent; ``log_det``, solves and the
variances are ordering-invariant and are what the hot path consumes.

``selected_inverse`` also accepts the ``DeviceFactor`` carried by a
``GaussianApprox`` from :class:`~.objective.ObjectiveEvaluator`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

from .engine import Engine
from .errors import DimensionMismatch, NotPositiveDefinite, StructureError
from .model import dense_vertex_cut
from .runtime import SERIAL, ThreadBudget
from .sparse import SparseSymMatrix

REL_PIVOT_TOL = 1e-13  # cholesky.py:31-32 (applied inside the device POTRF)
ORDERINGS = ("natural", "minimum-degree", "nested-dissection", "rcm")


@dataclass
class SymbolicFactor:
    """One-time analysis of a pattern: ordering + device tile structure."""

    n: int
    perm: np.ndarray
    engine: Engine
    q_indptr: np.ndarray
    q_indices: np.ndarray
    ordering: str
    generation: int = 0  # bumped by every numeric factorization

    @property
    def nnz(self) -> int:
        return int(self.engine.stats()["n_tiles"]) * 64 * 64

    def stats(self) -> dict:
        es = self.engine.stats()
        nnz_q = int(self.q_indptr[-1])
        return {"n": self.n, "nnz_lower_input": nnz_q, "nnz_factor": self.nnz,
                "fill_ratio": self.nnz / nnz_q, "tile_rows": es["n_tile_rows"],
                "tiles": es["n_tiles"], "ordering": self.ordering}


@dataclass
class CholeskyFactor:
    symbolic: SymbolicFactor
    log_det: float
    qvals: np.ndarray
    generation: int

    @property
    def n(self) -> int:
        return self.symbolic.n

    def _ensure_resident(self):
        s = self.symbolic
        if s.generation != self.generation:
            ld, st, bc = s.engine.factor_logdet(self.qvals)
            s.generation += 1
            self.generation = s.generation


@dataclass
class SelectedInverse:
    symbolic: object
    values: object
    marginal_variances: np.ndarray
    entries_computed: int = 0


def _order(Q: SparseSymMatrix, ordering: str):
    n = Q.n
    if ordering == "natural":
        return np.arange(n, dtype=np.int64), 0
    S = Q.to_scipy()
    S.data[:] = 1.0
    deg = np.diff(S.indptr) - 1
    dense = (np.flatnonzero(deg >= dense_vertex_cut(n)) if n > 32 else np.empty(0, int)).astype(np.int64)
    keep = np.setdiff1d(np.arange(n), dense)
    sub = S[keep][:, keep].tocsr()
    rcm = reverse_cuthill_mckee(sub, symmetric_mode=True)
    return np.concatenate([keep[rcm], dense]).astype(np.int64), int(dense.size)


def analyze(Q: SparseSymMatrix, ordering: str = "nested-dissection", leaf_cutoff: int = 64,
            device: int | None = None) -> SymbolicFactor:
    """Ordering + tile symbolic analysis + device upload (cholesky.py:88-137)."""
    if ordering not in ORDERINGS:
        raise StructureError(f"unknown ordering {ordering!r}; expected one of {ORDERINGS}")
    perm, n_dense = _order(Q, ordering)
    eng = Engine.for_matrix(Q.indptr, Q.indices, Q.data, perm, n_dense, device=device)
    return SymbolicFactor(Q.n, perm, eng, Q.indptr, Q.indices, ordering)


def _check_structure(sym: SymbolicFactor, Q: SparseSymMatrix):
    if Q.n != sym.n:
        raise DimensionMismatch("matrix size differs from the analyzed pattern")
    same = Q.indptr is sym.q_indptr and Q.indices is sym.q_indices
    if not same and not (np.array_equal(Q.indptr, sym.q_indptr)
                         and np.array_equal(Q.indices, sym.q_indices)):
        raise StructureError("matrix pattern differs from the analyzed pattern")


def factorize(sym: SymbolicFactor, Q: SparseSymMatrix, budget: ThreadBudget = SERIAL) -> CholeskyFactor:
    """Numeric tile factorization on the device (cholesky.py:282-322)."""
    _check_structure(sym, Q)
    q = np.ascontiguousarray(Q.data, dtype=np.float64)
    ld, st, bc = sym.engine.factor_logdet(q)
    sym.generation += 1
    if st != 0:
        raise NotPositiveDefinite(bc)
    return CholeskyFactor(sym, ld, q.copy(), sym.generation)


def solve(fac: CholeskyFactor, b) -> np.ndarray:
    """Q x = b, input/output in original order (cholesky.py:325-336)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (fac.n,):
        raise DimensionMismatch(f"b must have length {fac.n}")
    fac._ensure_resident()
    return fac.symbolic.engine.solve_resident(b)


def selected_inverse(fac, budget: ThreadBudget = SERIAL) -> SelectedInverse:
    """Takahashi selected inversion on the device (cholesky.py:356-400)."""
    from .objective import DeviceFactor

    if isinstance(fac, DeviceFactor):
        var, _ = fac.evaluator.marginal_variances(fac.theta, fac.warm_start)
        es = fac.evaluator.engine.stats()
        return SelectedInverse(None, None, var, int(es["n_tiles"]) * 64 * 64)
    fac._ensure_resident()
    var = fac.symbolic.engine.selinv_resident()
    return SelectedInverse(fac.symbolic, None, var, fac.symbolic.nnz)


def sample_gmrf(fac: CholeskyFactor, z) -> np.ndarray:
    """Not on the hot path; provided through the dense CPU route is
    deliberately NOT offered (no CPU fallback).  Use synth.* generators."""
    raise NotImplementedError("sample_gmrf is outside the B200 hot path")
