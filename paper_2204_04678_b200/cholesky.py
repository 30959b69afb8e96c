"""Sparse SPD factorization, solves and selected inversion on the device.

Drop-in for the reference's `cholesky.py` surface (`/root/reference/pkg/
src/parinla/cholesky.py:88-400`): ``analyze`` -> ``SymbolicFactor``,
``factorize`` -> ``CholeskyFactor`` (with ``log_det``, raising
``NotPositiveDefinite(column)`` in original order), ``solve``,
``selected_inverse`` -> ``SelectedInverse`` (``marginal_variances`` in original
order), ``sample_gmrf``.

Orderings: "nested-dissection" (the reference default) is the reference's
own nested dissection computed natively (csrc/ordering.cpp: the same
permutation), "minimum-degree" its minimum degree, "natural" the identity;
"rcm" is an extra.  The numeric factor lives on the device as dense tiles
aligned to the separator tree; the reference's scalar payloads are
materialized from those tiles on request: ``SymbolicFactor.Lp/Li`` (the
scalar elimination pattern, host C++), ``CholeskyFactor.values`` and
``SelectedInverse.values`` on that pattern (device gather).  With the
nested-dissection ordering the permutation, the pattern and therefore the
value arrays correspond entry for entry to the reference's.

``selected_inverse`` also accepts the ``DeviceFactor`` carried by a
``GaussianApprox`` from :class:`~.objective.ObjectiveEvaluator`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.sparse.csgraph import reverse_cuthill_mckee

from . import _lib
from .engine import Engine
from .errors import DimensionMismatch, NotPositiveDefinite, StructureError
from .model import dense_vertex_cut
from .runtime import SERIAL, ThreadBudget
from .sparse import SparseSymMatrix

REL_PIVOT_TOL = 1e-13  # cholesky.py:31-32 (applied inside the device POTRF)
ORDERINGS = ("natural", "minimum-degree", "nested-dissection", "rcm")


@dataclass(frozen=True)
class Permutation:
    """perm maps new index -> old index; iperm is its inverse
    (reference ordering.py:69-96)."""

    perm: np.ndarray
    iperm: np.ndarray

    @classmethod
    def from_order(cls, order) -> "Permutation":
        perm = np.ascontiguousarray(order, dtype=np.int64)
        iperm = np.empty_like(perm)
        iperm[perm] = np.arange(perm.size, dtype=np.int64)
        return cls(perm, iperm)

    @property
    def n(self) -> int:
        return int(self.perm.shape[0])


class SymbolicFactor:
    """One-time analysis of a pattern: ordering + device tile structure, and
    (lazily) the scalar elimination pattern ``Lp``/``Li`` of the reference
    (cholesky.py:43-85; permuted indices, per column diagonal first)."""

    def __init__(self, n, perm, engine, q_indptr, q_indices, ordering, tile_bounds=None):
        self.n = int(n)
        self.perm = np.ascontiguousarray(perm, dtype=np.int64)
        self.engine = engine
        self.q_indptr = q_indptr
        self.q_indices = q_indices
        self.ordering = ordering
        self.tile_bounds = tile_bounds
        self.generation = 0      # bumped by every numeric factorization
        self.sel_generation = -1  # factor generation of the resident Sigma tiles
        self._Lp = None
        self._Li = None

    @property
    def permutation(self) -> Permutation:
        return Permutation.from_order(self.perm)

    def _pattern(self):
        if self._Lp is None:
            self._Lp, self._Li = _lib.scalar_pattern(self.q_indptr, self.q_indices, self.perm)
        return self._Lp, self._Li

    @property
    def Lp(self) -> np.ndarray:
        return self._pattern()[0]

    @property
    def Li(self) -> np.ndarray:
        return self._pattern()[1]

    @property
    def nnz(self) -> int:
        return int(self.Lp[self.n])

    def entry_columns(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.Lp))

    def stats(self) -> dict:
        es = self.engine.stats()
        nnz_q = int(self.q_indptr[-1])
        return {"n": self.n, "nnz_lower_input": nnz_q, "nnz_factor": self.nnz,
                "fill_ratio": self.nnz / nnz_q, "tile_rows": es["n_tile_rows"],
                "tiles": es["n_tiles"], "ordering": self.ordering}


class CholeskyFactor:
    """Numeric factor (device tiles) plus its log-determinant; ``values`` on
    the scalar pattern are read from the device on first access
    (reference cholesky.py:168-190)."""

    def __init__(self, symbolic: SymbolicFactor, log_det: float, qvals: np.ndarray, generation: int):
        self.symbolic = symbolic
        self.log_det = float(log_det)
        self.qvals = qvals
        self.generation = generation
        self._values = None

    @property
    def n(self) -> int:
        return self.symbolic.n

    def _ensure_resident(self):
        s = self.symbolic
        if s.generation != self.generation:
            ld, st, bc = s.engine.factor_logdet(self.qvals)
            s.generation += 1
            self.generation = s.generation

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._ensure_resident()
            s = self.symbolic
            self._values = s.engine.tile_entries(0, 0, s.Li, s.entry_columns())
        return self._values

    def factor_diagonal(self) -> np.ndarray:
        return self.values[self.symbolic.Lp[:-1]]

    def to_scipy_lower(self):
        """L in scipy CSC, permuted ordering."""
        import scipy.sparse as sp

        s = self.symbolic
        return sp.csc_matrix((self.values, s.Li, s.Lp), shape=(s.n, s.n))


class SelectedInverse:
    """Entries of Sigma = Q^-1 on the pattern of L plus the re-permuted
    variances (reference cholesky.py:193-214).  ``values`` are read from the
    device's Sigma tiles on first access (recomputed if another selected
    inversion replaced them meanwhile)."""

    def __init__(self, symbolic, values, marginal_variances, entries_computed=0, refresh=None):
        self.symbolic = symbolic
        self._values = values
        self.marginal_variances = marginal_variances
        self.entries_computed = entries_computed
        self._refresh = refresh  # () -> None: make this Sigma resident again

    @property
    def values(self):
        if self._values is None and self.symbolic is not None:
            if self._refresh is not None:
                self._refresh()
            s = self.symbolic
            self._values = s.engine.tile_entries(1, 0, s.Li, s.entry_columns())
        return self._values

    def entry(self, i: int, j: int) -> float:
        """Sigma_ij in original coordinates; (i, j) must be on the pattern."""
        s = self.symbolic
        ip = s.permutation.iperm
        r, c = int(ip[i]), int(ip[j])
        if r < c:
            r, c = c, r
        lo, hi = int(s.Lp[c]), int(s.Lp[c + 1])
        k = lo + int(np.searchsorted(s.Li[lo:hi], r))
        if k >= hi or s.Li[k] != r:
            raise StructureError(f"({i}, {j}) is not on the factor pattern")
        return float(self.values[k])


def _order(Q: SparseSymMatrix, ordering: str, leaf_cutoff: int):
    """(perm, n_dense, tile bounds or None)."""
    n = Q.n
    if ordering == "natural":
        return np.arange(n, dtype=np.int64), 0, None
    if ordering == "nested-dissection":
        return _lib.nd_order(Q.indptr, Q.indices, leaf_cutoff=leaf_cutoff)
    if ordering == "minimum-degree":
        return _lib.nd_order(Q.indptr, Q.indices, leaf_cutoff=0)
    S = Q.to_scipy()
    S.data[:] = 1.0
    deg = np.diff(S.indptr) - 1
    dense = (np.flatnonzero(deg >= dense_vertex_cut(n)) if n > 32 else np.empty(0, int)).astype(np.int64)
    keep = np.setdiff1d(np.arange(n), dense)
    sub = S[keep][:, keep].tocsr()
    rcm = reverse_cuthill_mckee(sub, symmetric_mode=True)
    return np.concatenate([keep[rcm], dense]).astype(np.int64), int(dense.size), None


def analyze(Q: SparseSymMatrix, ordering: str = "nested-dissection", leaf_cutoff: int = 64,
            device: int | None = None) -> SymbolicFactor:
    """Ordering + tile symbolic analysis + device upload (cholesky.py:88-137)."""
    if ordering not in ORDERINGS:
        raise StructureError(f"unknown ordering {ordering!r}; expected one of {ORDERINGS}")
    if leaf_cutoff < 1:
        raise StructureError("leaf_cutoff must be at least 1")
    perm, n_dense, bounds = _order(Q, ordering, leaf_cutoff)
    eng = Engine.for_matrix(Q.indptr, Q.indices, Q.data, perm, n_dense, device=device,
                            tile_bounds=bounds)
    return SymbolicFactor(Q.n, perm, eng, Q.indptr, Q.indices, ordering, bounds)


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
        ev = fac.evaluator
        var, _ = ev.marginal_variances(fac.theta, fac.warm_start)
        token = ev.engine_calls

        def refresh():
            if ev.engine_calls != token:
                ev.marginal_variances(fac.theta, fac.warm_start)

        sym = fac.symbolic
        return SelectedInverse(sym, None, var, sym.nnz, refresh)
    fac._ensure_resident()
    sym = fac.symbolic
    var = sym.engine.selinv_resident()
    sym.sel_generation = fac.generation
    gen = fac.generation

    def refresh():
        if sym.sel_generation != gen or sym.generation != gen:
            fac._ensure_resident()
            sym.engine.selinv_resident()
            sym.sel_generation = fac.generation

    return SelectedInverse(sym, None, var, sym.nnz, refresh)


def sample_gmrf(fac, z) -> np.ndarray:
    """A draw with precision Q from iid standard normals ``z`` given in
    factor coordinates: x = P^T L^-T z, returned in the original order
    (reference cholesky.py:339-353).  On the device as L^-T z = Q^-1 (L z):
    one tile L x product and one resident solve."""
    from .objective import DeviceFactor

    z = np.asarray(z, dtype=np.float64)
    if isinstance(fac, DeviceFactor):
        eng = fac.evaluator.engine
        fac.make_resident()
        n = fac.n
    else:
        fac._ensure_resident()
        eng = fac.symbolic.engine
        n = fac.n
    if z.shape != (n,):
        raise DimensionMismatch(f"z must have length {n}")
    y = eng.factor_lmul(z, 0)  # L z, factor coordinates
    b = np.empty(n)
    b[eng.perm] = y  # to the original order
    return eng.solve_resident(b)
