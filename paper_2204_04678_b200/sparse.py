"""Lower-triangular CSC storage of symmetric sparse matrices (boundary layout).

Same contract as the reference `SparseSymMatrix` (`/root/reference/pkg/src/
parinla/sparse.py:15-127`): lower triangle only, column compressed, the
diagonal structurally present and FIRST in every column, rows strictly
ascending, int64 indices and float64 values.  Q(theta) crosses the
boundary in this layout; inside the engine it is re-laid into dense tiles.
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionMismatch, StructureError


class SparseSymMatrix:
    __slots__ = ("n", "indptr", "indices", "data")

    def __init__(self, n, indptr, indices, data, validate: bool = True):
        self.n = int(n)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        if validate:
            self._check()

    def _check(self):
        n = self.n
        if n < 1:
            raise StructureError("matrix dimension must be positive")
        if self.indptr.shape != (n + 1,) or self.indptr[0] != 0:
            raise StructureError("bad column pointer array")
        nnz = int(self.indptr[n])
        if self.indices.shape != (nnz,) or self.data.shape != (nnz,):
            raise StructureError("index/value arrays disagree with column pointers")
        if np.any(np.diff(self.indptr) < 1):
            raise StructureError("every column needs its diagonal entry")
        if np.any(self.indices[self.indptr[:-1]] != np.arange(n)):
            raise StructureError("missing diagonal entry or row above the diagonal")
        if np.any(self.indices < 0) or np.any(self.indices >= n):
            raise StructureError("row index out of range")
        step = np.diff(self.indices)
        interior = np.ones(step.shape[0], dtype=bool)
        interior[self.indptr[1:-1] - 1] = False
        if np.any(step[interior] <= 0):
            raise StructureError("row indices must ascend within each column")

    @property
    def nnz(self) -> int:
        return int(self.indptr[self.n])

    def col_of_entry(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.indptr))

    def diagonal(self) -> np.ndarray:
        return self.data[self.indptr[:-1]].copy()

    def with_values(self, data) -> "SparseSymMatrix":
        data = np.ascontiguousarray(data, dtype=np.float64)
        if data.shape != (self.nnz,):
            raise DimensionMismatch("value array does not match pattern")
        out = SparseSymMatrix.__new__(SparseSymMatrix)
        out.n, out.indptr, out.indices, out.data = self.n, self.indptr, self.indices, data
        return out

    def same_pattern(self, other: "SparseSymMatrix") -> bool:
        if self.indptr is other.indptr and self.indices is other.indices:
            return True
        return (
            self.n == other.n
            and np.array_equal(self.indptr, other.indptr)
            and np.array_equal(self.indices, other.indices)
        )

    def to_scipy(self):
        """Full symmetric scipy CSC (both triangles)."""
        import scipy.sparse as sp

        L = sp.csc_matrix((self.data, self.indices, self.indptr), shape=(self.n, self.n))
        return (L + sp.tril(L, -1).T).tocsc()

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    @classmethod
    def from_coo(cls, n, rows, cols, vals) -> "SparseSymMatrix":
        """Lower-triangle coordinates (i >= j); duplicates are summed,
        a zero diagonal is inserted where missing."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if np.any(rows < cols):
            raise StructureError("from_coo expects lower-triangle entries (i >= j)")
        diag = np.arange(n, dtype=np.int64)
        rows = np.concatenate([rows, diag])
        cols = np.concatenate([cols, diag])
        vals = np.concatenate([vals, np.zeros(n)])
        key = cols * n + rows
        uniq, inv = np.unique(key, return_inverse=True)
        summed = np.zeros(uniq.shape[0])
        np.add.at(summed, inv, vals)
        c = uniq // n
        r = uniq % n
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(indptr, c + 1, 1)
        np.cumsum(indptr, out=indptr)
        return cls(n, indptr, r, summed)

    @classmethod
    def from_dense(cls, M, tol: float = 0.0) -> "SparseSymMatrix":
        M = np.asarray(M, dtype=np.float64)
        r, c = np.nonzero(np.abs(np.tril(M)) > tol)
        return cls.from_coo(M.shape[0], r, c, M[r, c])

    @classmethod
    def from_scipy(cls, S) -> "SparseSymMatrix":
        import scipy.sparse as sp

        T = sp.tril(sp.coo_matrix(S))
        return cls.from_coo(S.shape[0], T.row, T.col, T.data)

    def __repr__(self):
        return f"SparseSymMatrix(n={self.n}, nnz={self.nnz})"
