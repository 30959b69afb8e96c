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
  Appendix A, taken two-sided (both time ends toward a middle separator
  block: same fill, half the dependency depth).  Pure 2-D fields: lattice
  nested dissection.
* any other pattern (the reference's iid/rw1/rw2/besag models): the
  reference's own nested dissection of the conditional graph, computed
  natively (csrc/ordering.cpp; the permutation equals the reference's), with
  the tile partition aligned to its separator tree: small subtrees become one
  dense tile each, larger separators balanced <= 64-row tiles.
* ``rcm``         reverse Cuthill-McKee on the conditional graph.
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

ORDERINGS = ("structured", "band", "rcm", "natural", "nested-dissection", "minimum-degree")
LEAF = 64


ND_LEAF = 256  # leaf regions of up to 4 tiles: fewer, fuller tiles (measured on c2)


def nd_lattice(nx: int, ny: int, reach: int = 2, leaf: int = ND_LEAF, sep_tile: int = LEAF,
               tile_max: int = LEAF):
    """Geometric nested dissection of an nx-by-ny lattice whose couplings
    reach ``reach`` lattice steps (G^2 stencil + bilinear cells: 2).

    Regions are split across their longer side by a separator ``reach``
    lines wide, children first, separator last (reference ND convention,
    ordering.py:206-274, here with geometric separators).  Returns the
    vertex order (row-major ids) and the tile sizes: leaf regions (<= ``leaf``
    vertices) and separators are each cut into the fewest balanced tiles of
    <= 64 vertices, laid out along the region, so that no tile couples two
    subtrees.
    """
    order: list = []
    tiles: list = []

    def emit_tiles(ids, size=None):
        # balanced cut into the fewest <= tile_max pieces (no thin remainder)
        size = min(size or leaf, tile_max)
        if not ids:
            return
        k = -(-len(ids) // size)
        base, rem = divmod(len(ids), k)
        order.extend(ids)
        tiles.extend(base + (1 if i < rem else 0) for i in range(k))

    def rec(r0, r1, c0, c1):
        h, w = r1 - r0, c1 - c0
        if h <= 0 or w <= 0:
            return
        if h * w <= leaf:
            emit_tiles([r * nx + c for r in range(r0, r1) for c in range(c0, c1)])
            return
        if h >= w:
            if h <= reach:
                emit_tiles([r * nx + c for c in range(c0, c1) for r in range(r0, r1)])
                return
            mid = r0 + (h - reach) // 2
            rec(r0, mid, c0, c1)
            rec(mid + reach, r1, c0, c1)
            emit_tiles([r * nx + c for c in range(c0, c1) for r in range(mid, mid + reach)], sep_tile)
        else:
            if w <= reach:
                emit_tiles([r * nx + c for r in range(r0, r1) for c in range(c0, c1)])
                return
            mid = c0 + (w - reach) // 2
            rec(r0, r1, c0, mid)
            rec(r0, r1, mid + reach, c1)
            emit_tiles([r * nx + c for r in range(r0, r1) for c in range(mid, mid + reach)], sep_tile)

    rec(0, ny, 0, nx)
    return np.asarray(order, dtype=np.int64), np.asarray(tiles, dtype=np.int64)


def _bounds(sizes_main, n_main, n_dense):
    sizes = list(sizes_main) + [min(LEAF, n_dense - s) for s in range(0, n_dense, LEAF)]
    b = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    assert b[-1] == n_main + n_dense
    return b


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


def structured_order(spec: ModelSpec, band: bool = False, two_sided: bool = True):
    """(perm (new -> old), n_dense, tile bounds or None) for lattice / ST
    models, or None.  2-D fields: lattice nested dissection (``band``:
    row-major band instead).  Spatio-temporal: time-major blocks, two-sided
    (``two_sided=False``: one-sided time-major BTA)."""
    comps = spec.components
    kinds = [c.kind for c in comps]
    fixed = np.arange(spec.n_fixed, dtype=np.int64)
    if kinds == ["spde2d"]:
        ofs = spec.component_offset(comps[0])
        if band:
            body = ofs + np.arange(comps[0].size, dtype=np.int64)
            return np.concatenate([body, fixed]), fixed.size, None
        order, sizes = nd_lattice(comps[0].graph.nx, comps[0].graph.ny)
        perm = np.concatenate([ofs + order, fixed])
        return perm, fixed.size, _bounds(sizes, order.size, fixed.size)
    if kinds and kinds[0] == "ar1_spde2d" and all(k == "ar1" for k in kinds[1:]):
        st = comps[0]
        nt, ns = st.nt, st.graph.n
        ofs = spec.component_offset(st)
        extra = []
        for c in comps[1:]:
            if c.nt != nt:
                return None
            extra.append(spec.component_offset(c))
        def block(t):
            return np.concatenate([ofs + t * ns + np.arange(ns, dtype=np.int64)]
                                  + [np.array([e + t], dtype=np.int64) for e in extra])

        if nt < 3 or not two_sided:
            return np.concatenate([block(t) for t in range(nt)] + [fixed]), fixed.size, None
        # two-sided time order: blocks 0..h-1 forward, blocks nt-1..h+1
        # backward, separator block h last.  Each segment is eliminated from
        # its outer end toward h, so no fill is created beyond the BTA
        # pattern (h couples to h-1 and h+1 only) while the two segments'
        # block chains are independent: half the DAG depth of the one-sided
        # time-major order for the factorization and both solve sweeps.
        # Tiles are cut per segment so that none couples the two chains.
        h = nt // 2
        seg_a = [block(t) for t in range(h)]
        seg_b = [block(t) for t in range(nt - 1, h, -1)]
        sep = block(h)
        sizes = []
        for seg in (seg_a, seg_b, [sep]):
            length = sum(b.size for b in seg)
            sizes += [LEAF] * (length // LEAF) + ([length % LEAF] if length % LEAF else [])
        perm = np.concatenate(seg_a + seg_b + [sep, fixed])
        return perm, fixed.size, _bounds(sizes, perm.size - fixed.size, fixed.size)
    return None


def nd_pattern_order(indptr, indices, leaf_cutoff: int = 64):
    """Native nested dissection of a lower-CSC pattern (libpinla, host only):
    the reference's nested_dissection_order permutation (ordering.py:206-274)
    plus separator-aligned tile bounds.  Returns (perm, n_dense, bounds)."""
    import os

    from . import _lib

    tile_max = int(os.environ.get("PINLA_ND_TILE_MAX", LEAF))  # tuning switch
    return _lib.nd_order(indptr, indices, leaf_cutoff=leaf_cutoff, tile_max=tile_max)


def md_pattern_order(indptr, indices):
    """The reference's minimum_degree_order (ordering.py:168-175): greedy
    minimum degree over the whole graph (no dense peel), natively."""
    from . import _lib

    return _lib.nd_order(indptr, indices, leaf_cutoff=0, tile_max=LEAF)


def lower_pattern(G: sp.csr_matrix):
    """Lower-CSC (indptr, indices) of a symmetric pattern."""
    T = sp.tril(G, format="csc")
    T.sort_indices()
    return T.indptr.astype(np.int64), T.indices.astype(np.int64)


def choose_order(spec: ModelSpec, A, prior_indptr, prior_indices, ordering: str = "structured",
                 leaf_cutoff: int = 64):
    """Return (perm, n_dense, tile_bounds or None).

    ``structured``: lattice ND / time-major BTA where the model is a lattice
    or spatio-temporal field, else the reference's nested dissection of the
    conditional pattern (native, separator-aligned tiles) — the ordering the
    reference's ObjectiveEvaluator analyzes its conditional matrix with
    (objective.py:160)."""
    n = spec.latent_dim
    if ordering not in ORDERINGS:
        raise StructureError(f"unknown ordering {ordering!r}; expected one of {ORDERINGS}")
    if ordering == "natural":
        return np.arange(n, dtype=np.int64), 0, None
    if ordering in ("structured", "band"):
        got = structured_order(spec, band=ordering == "band")
        if got is not None:
            return got
    G = conditional_graph(spec, A, prior_indptr, prior_indices)
    if ordering in ("structured", "band", "nested-dissection"):
        return nd_pattern_order(*lower_pattern(G), leaf_cutoff=leaf_cutoff)
    if ordering == "minimum-degree":
        return md_pattern_order(*lower_pattern(G))
    # rcm: reverse Cuthill-McKee of the conditional graph, dense vertices last
    dense = dense_vertices(G)
    keep = np.setdiff1d(np.arange(n), dense)
    sub = G[keep][:, keep]
    rcm = reverse_cuthill_mckee(sub.tocsr(), symmetric_mode=True)
    perm = np.concatenate([keep[rcm], dense]).astype(np.int64)
    return perm, dense.size, None
