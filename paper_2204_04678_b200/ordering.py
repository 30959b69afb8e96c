"""Fill-reducing orderings for the tile engine (one-time, host).

The reference orders every pattern by nested dissection in pure Python
(`/root/reference/pkg/src/parinla/ordering.py:206-274`) and factorizes with
a scalar up-looking kernel.  The B200 engine factorizes dense 64x64 tiles,
so the ordering goal is different: a *tile-banded* (block-tridiagonal-
arrow) structure whose tiles are dense and whose dependency chains are
regular.

* ``structured``  lattice / spatio-temporal models: time-major blocks
  (all field nodes of time t, then the temporal main-effect node of t),
  row-major lattice inside a block; this is the BTA layout of SURVEY.md
  Appendix A.  Pure 2-D fields are row-major (band of 2 lattice rows).
* ``rcm``         any other pattern (the reference's iid/rw1/rw2/besag
  models): reverse Cuthill-McKee on the conditional graph.
* ``natural``     identity (tests).

In all cases the dense vertices (degree >= max(16, (n-1)/2), the
reference's ND peel rule at `ordering.py:221-226`; in practice the fixed
effects) are moved to the end, where they form the arrow tiles.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

from .errors import StructureError
from .model import ModelSpec, dense_vertex_cut

ORDERINGS = ("structured", "rcm", "natural", "nested-dissection", "minimum-degree")


def conditional_graph(spec: ModelSpec, A, prior_indptr, prior_indices) -> sp.csr_matrix:
    """Symmetric boolean pattern of Q_prior + A^T A (original order)."""
    n = spec.latent_dim
    cols = np.repeat(np.arange(n), np.diff(prior_indptr))
    P = sp.coo_matrix((np.ones(cols.size), (prior_indices, cols)), shape=(n, n))
    B = sp.csr_matrix(A, copy=True)
    B.data[:] = 1.0
    G = (P + P.T + B.T @ B).tocsr()
    G.data[:] = 1.0
    return G


def dense_vertices(G: sp.csr_matrix) -> np.ndarray:
    n = G.shape[0]
    if n <= 32:
        return np.empty(0, dtype=np.int64)
    deg = np.diff(G.indptr) - 1  # minus the diagonal
    return np.flatnonzero(deg >= dense_vertex_cut(n)).astype(np.int64)


def structured_order(spec: ModelSpec):
    """perm (new -> old) and n_dense for lattice / ST models, or None."""
    comps = spec.components
    kinds = [c.kind for c in comps]
    fixed = np.arange(spec.n_fixed, dtype=np.int64)
    if kinds == ["spde2d"]:
        ofs = spec.component_offset(comps[0])
        body = ofs + np.arange(comps[0].size, dtype=np.int64)
        return np.concatenate([body, fixed]), fixed.size
    if kinds and kinds[0] == "ar1_spde2d" and all(k == "ar1" for k in kinds[1:]):
        st = comps[0]
        nt, ns = st.nt, st.graph.n
        ofs = spec.component_offset(st)
        extra = []
        for c in comps[1:]:
            if c.nt != nt:
                return None
            extra.append(spec.component_offset(c))
        blocks = []
        for t in range(nt):
            blocks.append(ofs + t * ns + np.arange(ns, dtype=np.int64))
            for e in extra:
                blocks.append(np.array([e + t], dtype=np.int64))
        return np.concatenate(blocks + [fixed]), fixed.size
    return None


def choose_order(spec: ModelSpec, A, prior_indptr, prior_indices, ordering: str = "structured"):
    """Return (perm, n_dense)."""
    n = spec.latent_dim
    if ordering not in ORDERINGS:
        raise StructureError(f"unknown ordering {ordering!r}; expected one of {ORDERINGS}")
    if ordering == "natural":
        return np.arange(n, dtype=np.int64), 0
    if ordering == "structured":
        got = structured_order(spec)
        if got is not None:
            return got
    # generic: RCM of the conditional graph with the dense vertices last
    G = conditional_graph(spec, A, prior_indptr, prior_indices)
    dense = dense_vertices(G)
    keep = np.setdiff1d(np.arange(n), dense)
    sub = G[keep][:, keep]
    rcm = reverse_cuthill_mckee(sub.tocsr(), symmetric_mode=True)
    perm = np.concatenate([keep[rcm], dense]).astype(np.int64)
    return perm, dense.size
