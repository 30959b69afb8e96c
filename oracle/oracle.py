"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's f(theta) path (`/root/reference/pkg/src/
parinla/`), used exclusively as the CHECKER by tests/, by
``__graft_entry__.smoke()`` and by bench.py's ``cpu_baseline`` leg and
``--impl reference`` arm (the reference itself is Python and cannot travel to
the GPU box).  Nothing in the product package imports this module.

Pinning: every function here is checked against (a) the reference's own
known-answer tests and (b) golden vectors produced by running the unmodified
reference here through the three-patch adapter of SURVEY.md Appendix B
(``tests/golden/make_golden.py``); see ``tests/test_oracle_pins.py``.

What is restated (reference file:line):
  * ordering: nested dissection with BFS level-set separators, dense peel,
    minimum-degree leaves           ordering.py:168-423
  * analyze / permuted row form     cholesky.py:88-165
  * factorize / solve / selinv      cholesky.py:282-400, numerics in
                                    oracle/ckernels.c (kernels.py); factorize
                                    also on the level-2 schedule (separator
                                    tree ordering.py:206-274, _pruned_tasks
                                    cholesky.py:217-258, run_tree_tasks
                                    runtime.py:180-268), bitwise = serial
  * conditional mode + f(theta)     objective.py:79-331
  * likelihood / hyper prior        model.py:285-331
Prior assembly for the BASELINE field kinds (absent from the reference,
SURVEY s0.4) is written independently of the product's term plan: scipy
Kronecker / matrix products of the structure matrices.
"""

from __future__ import annotations

import ctypes
import heapq
import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
REL_PIVOT_TOL = 1e-13  # cholesky.py:31-32
LOG_2PI = math.log(2.0 * math.pi)

_lib = None
_P = ctypes.c_void_p
_I = ctypes.c_int64


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "build", "liboracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.check_call(["make", "-s", "-C", HERE])
        L = ctypes.CDLL(path)
        L.orc_factor_range.restype = ctypes.c_int64
        L.orc_selinv_range.restype = ctypes.c_int64
        L.orc_logdiag_sum.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class NotPD(Exception):
    def __init__(self, column):
        self.column = int(column)
        super().__init__(f"non-positive pivot at column {column}")


class InnerDiv(Exception):
    pass


# ----------------------------------------------------------------------
# ordering (ordering.py)


class Graph:
    def __init__(self, n, indptr, indices):
        self.n, self.indptr, self.indices = n, indptr, indices

    def nb(self, v):
        return self.indices[self.indptr[v] : self.indptr[v + 1]]

    @classmethod
    def of_lower(cls, n, indptr, indices):
        cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
        off = indices != cols
        u, v = indices[off], cols[off]
        S = sp.coo_matrix((np.ones(2 * u.size), (np.concatenate([u, v]), np.concatenate([v, u]))),
                          shape=(n, n)).tocsr()
        S.sum_duplicates()
        S.sort_indices()
        return cls(n, S.indptr.astype(np.int64), S.indices.astype(np.int64))


def _min_degree(g: Graph, verts):
    """ordering.py:178-203 — greedy minimum degree on the induced subgraph."""
    vs = [int(v) for v in verts]
    vset = set(vs)
    adj = {v: {int(u) for u in g.nb(v) if int(u) in vset} for v in vs}
    heap = [(len(adj[v]), v) for v in vs]
    heapq.heapify(heap)
    out, alive = [], set(vs)
    while heap:
        deg, v = heapq.heappop(heap)
        if v not in alive or deg != len(adj[v]):
            continue
        out.append(v)
        alive.discard(v)
        nbr = adj.pop(v)
        for u in nbr:
            adj[u].discard(v)
        nbr = sorted(nbr)
        for i, a in enumerate(nbr):
            for b in nbr[i + 1 :]:
                if b not in adj[a]:
                    adj[a].add(b)
                    adj[b].add(a)
        for u in nbr:
            heapq.heappush(heap, (len(adj[u]), u))
    return out


def _components(g, verts):
    member = np.zeros(g.n, dtype=bool)
    member[verts] = True
    seen = np.zeros(g.n, dtype=bool)
    comps = []
    for v in np.sort(verts):
        v = int(v)
        if seen[v]:
            continue
        comp = [v]
        seen[v] = True
        h = 0
        while h < len(comp):
            u = comp[h]
            h += 1
            for w in g.nb(u):
                w = int(w)
                if member[w] and not seen[w]:
                    seen[w] = True
                    comp.append(w)
        comps.append(np.sort(np.asarray(comp, dtype=np.int64)))
    return comps


def _levels(g, member, root):
    lev = {root: 0}
    levels = [[root]]
    front = [root]
    while front:
        nxt = []
        for u in front:
            for w in g.nb(u):
                w = int(w)
                if member[w] and w not in lev:
                    lev[w] = lev[u] + 1
                    nxt.append(w)
        if nxt:
            levels.append(sorted(nxt))
        front = nxt
    return levels


def _peripheral(g, comp, member):
    degs = np.diff(g.indptr)[comp]
    root = int(comp[int(np.argmin(degs))])
    ecc = -1
    for _ in range(8):
        lv = _levels(g, member, root)
        if len(lv) - 1 <= ecc:
            break
        ecc = len(lv) - 1
        root = min(lv[-1], key=lambda v: (int(g.indptr[v + 1] - g.indptr[v]), v))
    return root


def _boundary(g, levels, level_of, m):
    prev = {v for v in levels[m] if any(level_of[int(w)] == m - 1 for w in g.nb(v))}
    nxt = ({v for v in levels[m] if any(level_of[int(w)] == m + 1 for w in g.nb(v))}
           if m < len(levels) - 1 else set())
    opts = []
    if prev:
        opts.append((len(prev), 0, prev, "prev"))
    if nxt:
        opts.append((len(nxt), 1, nxt, "next"))
    if not opts:
        return None
    opts.sort(key=lambda o: (o[0], o[1]))
    return set(opts[0][2]), opts[0][3]


def _shrink(g, sep, a, b):
    changed = True
    while changed:
        changed = False
        for v in sorted(sep):
            ta = any(int(w) in a for w in g.nb(v))
            tb = any(int(w) in b for w in g.nb(v))
            if ta and tb:
                continue
            sep.discard(v)
            if ta:
                a.add(v)
            elif tb:
                b.add(v)
            else:
                (a if len(a) <= len(b) else b).add(v)
            changed = True
    return sep, a, b


def _separator(g, comp):
    """ordering.py:334-382."""
    member = np.zeros(g.n, dtype=bool)
    member[comp] = True
    root = _peripheral(g, comp, member)
    levels = _levels(g, member, root)
    h = len(levels) - 1
    if h < 1:
        return None
    cum = np.cumsum([len(lv) for lv in levels])
    m_star = min(max(int(np.searchsorted(cum, cum[-1] / 2.0)), 1), h)
    level_of = np.full(g.n, -1, dtype=np.int64)
    for d, lv in enumerate(levels):
        level_of[lv] = d
    for m in sorted(range(1, h + 1), key=lambda q: (abs(q - m_star), q)):
        picked = _boundary(g, levels, level_of, m)
        if picked is None:
            continue
        sep, side = picked
        below = [v for d in range(m) for v in levels[d]]
        at = [v for v in levels[m] if v not in sep]
        above = [v for d in range(m + 1, h + 1) for v in levels[d]]
        a, b = (below, at + above) if side == "prev" else (below + at, above)
        if not a or not b:
            continue
        sep, a, b = _shrink(g, sep, set(a), set(b))
        if sep and a and b:
            return (np.sort(np.fromiter(sep, np.int64)), np.sort(np.fromiter(a, np.int64)),
                    np.sort(np.fromiter(b, np.int64)))
    return None


def nested_dissection(g: Graph, leaf_cutoff=64, with_tree=False):
    """ordering.py:206-274 — returns perm (new -> old); with ``with_tree``
    also the separator tree (nodes, root) the level-2 schedule runs on.
    Nodes are dicts {start, end, span_start, children}, built in the
    reference's node order (leaves and separators as emitted, then a root over
    the dense vertices when there are several tops or dense vertices)."""
    order = []
    nodes = []
    deg = np.diff(g.indptr)
    cut = max(16, (g.n - 1) // 2)
    dense = np.flatnonzero(deg >= cut).astype(np.int64) if g.n > 32 else np.empty(0, np.int64)

    def new_node(start, end, children):
        span = min([start] + [nodes[c]["span_start"] for c in children])
        nodes.append(dict(start=start, end=end, span_start=span, children=list(children)))
        return len(nodes) - 1

    def leaf(verts):
        start = len(order)
        order.extend(_min_degree(g, verts))
        return new_node(start, len(order), [])

    def dissect(verts):
        if 0 < verts.shape[0] <= leaf_cutoff:
            return [leaf(np.sort(verts))]
        tops = []
        for comp in _components(g, verts):
            if comp.shape[0] <= leaf_cutoff:
                tops.append(leaf(comp))
                continue
            split = _separator(g, comp)
            if split is None:
                tops.append(leaf(comp))
                continue
            sep, a, b = split
            kids = dissect(a) + dissect(b)
            start = len(order)
            order.extend(int(v) for v in sep)
            tops.append(new_node(start, len(order), kids))
        return tops

    import sys

    sys.setrecursionlimit(max(10000, sys.getrecursionlimit()))
    keep = np.setdiff1d(np.arange(g.n, dtype=np.int64), dense, assume_unique=True)
    tops = dissect(keep)
    if len(tops) == 1 and dense.size == 0:
        root = tops[0]
    else:
        start = len(order)
        order.extend(int(v) for v in dense)
        root = new_node(start, len(order), tops)
    perm = np.asarray(order, dtype=np.int64)
    return (perm, (nodes, root)) if with_tree else perm


# ----------------------------------------------------------------------
# symbolic + numeric factorization (cholesky.py)


class Symbolic:
    pass


def analyze(n, indptr, indices, ordering="nested-dissection", leaf_cutoff=64, perm=None):
    """cholesky.py:88-165 (serial schedule only)."""
    L = lib()
    tree = None
    if perm is None:
        if ordering == "natural":
            perm = np.arange(n, dtype=np.int64)
        else:
            perm, tree = nested_dissection(Graph.of_lower(n, indptr, indices), leaf_cutoff,
                                           with_tree=True)
    perm = np.ascontiguousarray(perm, dtype=np.int64)
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    rp, cp = iperm[indices], iperm[cols]
    r, c = np.maximum(rp, cp), np.minimum(rp, cp)
    pos = np.arange(indices.shape[0], dtype=np.int64)
    diag = r == c
    adiag = np.empty(n, dtype=np.int64)
    adiag[r[diag]] = pos[diag]
    ro, co, po = r[~diag], c[~diag], pos[~diag]
    o = np.lexsort((co, ro))
    ro, co, po = ro[o], co[o], po[o]
    arowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(arowptr, ro + 1, 1)
    np.cumsum(arowptr, out=arowptr)
    s = Symbolic()
    s.n, s.perm, s.iperm = n, perm, iperm
    s.arowptr, s.arowcol, s.asrc, s.adiag = arowptr, np.ascontiguousarray(co), np.ascontiguousarray(po), adiag
    parent = np.empty(n, np.int64)
    work = np.empty(n, np.int64)
    L.orc_etree(_I(n), _p(arowptr), _p(s.arowcol), _p(parent), _p(work))
    cc = np.empty(n, np.int64)
    L.orc_colcount(_I(n), _p(arowptr), _p(s.arowcol), _p(parent), _p(work), _p(cc))
    Lp = np.zeros(n + 1, np.int64)
    np.cumsum(cc, out=Lp[1:])
    Li = np.empty(int(Lp[-1]), np.int64)
    nxt = np.empty(n, np.int64)
    L.orc_pattern(_I(n), _p(arowptr), _p(s.arowcol), _p(parent), _p(Lp), _p(Li), _p(work), _p(nxt))
    rowptr = np.empty(n + 1, np.int64)
    rowcol = np.empty(int(Lp[-1]) - n, np.int64)
    rowpos = np.empty(int(Lp[-1]) - n, np.int64)
    L.orc_row_form(_I(n), _p(Lp), _p(Li), _p(rowptr), _p(rowcol), _p(rowpos), _p(work))
    s.parent, s.Lp, s.Li, s.rowptr, s.rowcol, s.rowpos = parent, Lp, Li, rowptr, rowcol, rowpos
    s.nnz = int(Lp[-1])
    s.tree = tree
    return s


def pruned_tasks(s, n_workers):
    """cholesky.py:217-258 — coarsen the separator tree into a task forest:
    subtrees whose factor work (sum of squared column counts) is at most
    max(total / (24 n_workers), 2e5) become one task over their contiguous
    span.  Returns (parents, children, ranges)."""
    nodes, root = s.tree
    colsz = np.diff(s.Lp).astype(np.float64)
    prefix = np.concatenate([[0.0], np.cumsum(colsz * colsz)])
    sub = [prefix[nd["end"]] - prefix[nd["start"]] for nd in nodes]
    post, stack = [], [root]
    while stack:  # cholesky.py:261-269 postorder
        i = stack.pop()
        post.append(i)
        stack.extend(nodes[i]["children"])
    for i in reversed(post):
        for c in nodes[i]["children"]:
            sub[i] += sub[c]
    threshold = max(sub[root] / (n_workers * 24.0), 2.0e5)
    parents, children, ranges = [], [], []

    def emit(node, parent_task):
        nd = nodes[node]
        tid = len(parents)
        parents.append(parent_task)
        children.append([])
        if parent_task >= 0:
            children[parent_task].append(tid)
        if sub[node] <= threshold or not nd["children"]:
            ranges.append((nd["span_start"], nd["end"]))
        else:
            ranges.append((nd["start"], nd["end"]))
            for c in nd["children"]:
                emit(c, tid)
        return tid

    emit(root, -1)
    return parents, children, ranges


def run_tree_tasks(parents, children, run, n_workers):
    """runtime.py:180-268 (children before parents): a shared ready queue,
    ``run(node, slot)`` on worker slot 0..n_workers-1, the caller is slot 0,
    first error re-raised after all workers stop."""
    n = len(parents)
    pending = [len(children[i]) for i in range(n)]
    ready = [i for i in range(n) if pending[i] == 0]
    cond = threading.Condition()
    state = {"remaining": n, "error": None}

    def worker(slot):
        while True:
            with cond:
                while not ready and state["remaining"] > 0 and state["error"] is None:
                    cond.wait()
                if state["error"] is not None or state["remaining"] == 0:
                    return
                node = ready.pop(0)
            try:
                run(node, slot)
            except BaseException as exc:  # noqa: BLE001 - re-raised below
                with cond:
                    if state["error"] is None:
                        state["error"] = exc
                    cond.notify_all()
                return
            with cond:
                state["remaining"] -= 1
                p = parents[node]
                if p >= 0:
                    pending[p] -= 1
                    if pending[p] == 0:
                        ready.append(p)
                cond.notify_all()
                if state["remaining"] == 0:
                    return

    helpers = [threading.Thread(target=worker, args=(k,)) for k in range(1, n_workers)]
    for t in helpers:
        t.start()
    worker(0)
    for t in helpers:
        t.join()
    if state["error"] is not None:
        raise state["error"]


def factorize(s, qvals, workers=1):
    """cholesky.py:282-322 -> (Lx, log_det).  ``workers`` > 1 runs the
    level-2 schedule (sibling subtrees as parallel tasks, cholesky.py:300-319;
    the C kernel releases the GIL under ctypes); bit-identical to serial."""
    L = lib()
    qvals = np.ascontiguousarray(qvals, dtype=np.float64)
    Lx = np.zeros(s.nnz)
    tree = getattr(s, "tree", None)
    workers = max(1, min(int(workers), os.cpu_count() or 1, len(tree[0]) if tree else 1))

    def rng(start, end, x):
        fail = L.orc_factor_range(_I(start), _I(end), _p(s.Lp), _p(s.Li), _p(Lx), _p(s.rowptr),
                                  _p(s.rowcol), _p(s.rowpos), _p(s.arowptr), _p(s.arowcol),
                                  _p(s.asrc), _p(s.adiag), _p(qvals), _p(x),
                                  ctypes.c_double(REL_PIVOT_TOL))
        if fail >= 0:
            raise NotPD(s.perm[fail])

    if workers == 1:
        rng(0, s.n, np.zeros(s.n))
    else:
        parents, children, ranges = pruned_tasks(s, workers)
        ws = [np.zeros(s.n) for _ in range(workers)]
        run_tree_tasks(parents, children, lambda node, slot: rng(*ranges[node], ws[slot]), workers)
    # cholesky.py:321 — 2 * np.sum(np.log(diag))
    log_det = 2.0 * float(np.sum(np.log(Lx[s.Lp[:-1]])))
    return Lx, log_det


def solve(s, Lx, b):
    """cholesky.py:325-336."""
    L = lib()
    w = np.ascontiguousarray(np.asarray(b, dtype=np.float64)[s.perm])
    L.orc_solve_lower(_I(s.n), _p(s.Lp), _p(s.Li), _p(Lx), _p(w))
    L.orc_solve_lower_t(_I(s.n), _p(s.Lp), _p(s.Li), _p(Lx), _p(w))
    out = np.empty(s.n)
    out[s.perm] = w
    return out


def selected_inverse(s, Lx):
    """cholesky.py:356-400 serial branch; returns (Sx, variances in original order)."""
    L = lib()
    Sx = np.zeros(s.nnz)
    z = np.zeros(s.n)
    stamp = np.full(s.n, -1, dtype=np.int64)
    L.orc_selinv_range(_I(0), _I(s.n), _p(s.Lp), _p(s.Li), _p(np.ascontiguousarray(Lx)), _p(Sx),
                       _p(s.rowptr), _p(s.rowcol), _p(s.rowpos), _p(z), _p(stamp))
    var = np.empty(s.n)
    var[s.perm] = Sx[s.Lp[:-1]]
    return Sx, var


def sym_matvec(n, indptr, indices, data, x):
    L = lib()
    out = np.zeros(n)
    L.orc_sym_matvec(_I(n), _p(indptr), _p(indices), _p(np.ascontiguousarray(data)),
                     _p(np.ascontiguousarray(x, dtype=np.float64)), _p(out))
    return out


# ----------------------------------------------------------------------
# model pieces (independent of the product's term plan)


def _lattice_G(nx, ny):
    n = nx * ny
    idx = np.arange(n).reshape(ny, nx)
    u = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
    v = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
    W = sp.coo_matrix((np.ones(u.size), (u, v)), shape=(n, n))
    W = (W + W.T).tocsr()
    return (sp.diags(np.asarray(W.sum(1)).ravel()) - W).tocsr()


def _q_ar1(nt, rho):
    main = np.full(nt, 1.0 + rho * rho)
    main[0] = main[-1] = 1.0
    off = np.full(nt - 1, -rho)
    return sp.diags([off, main, off], [-1, 0, 1], format="csr") / (1.0 - rho * rho)


def _structure(kind, size, graph):
    if kind == "iid":
        return sp.identity(size, format="csr")
    if kind == "rw1":
        D = sp.diags([-np.ones(size - 1), np.ones(size - 1)], [0, 1], shape=(size - 1, size))
        return (D.T @ D).tocsr()
    if kind == "rw2":
        D = sp.diags([np.ones(size - 2), -2 * np.ones(size - 2), np.ones(size - 2)], [0, 1, 2],
                     shape=(size - 2, size))
        return (D.T @ D).tocsr()
    if kind == "besag":
        indptr, indices = (graph.indptr, graph.indices) if hasattr(graph, "indptr") else graph
        W = sp.csr_matrix((np.ones(len(indices)), indices, indptr), shape=(size, size))
        return (sp.diags(np.diff(indptr).astype(float)) - W).tocsr()
    raise ValueError(kind)


class OracleModel:
    """Q_prior(theta), design and likelihood of a product ``ModelSpec``,
    recomputed independently (no use of the spec's prior plan)."""

    def __init__(self, spec, y):
        self.spec = spec
        self.y = np.asarray(y, dtype=np.float64)
        self.n = spec.latent_dim
        self.m = spec.m
        blocks = []
        if spec.intercept:
            blocks.append(sp.csr_matrix(np.ones((spec.m, 1))))
        if spec.Z.shape[1]:
            blocks.append(sp.csr_matrix(spec.Z))
        for c in spec.components:
            if c.design is not None:
                blocks.append(sp.csr_matrix(c.design))
            else:
                blocks.append(sp.csr_matrix((np.ones(spec.m), (np.arange(spec.m), c.obs_index)),
                                            shape=(spec.m, c.size)))
        self.A = sp.hstack(blocks, format="csr")
        self.AT = self.A.T.tocsr()
        # fixed pattern: union of every basis at unit gains
        pat = self._prior_matrix(np.zeros(spec.theta_dim), pattern=True)
        T = sp.tril(pat).tocsc()
        T.sort_indices()
        self.p_indptr = T.indptr.astype(np.int64)
        self.p_indices = T.indices.astype(np.int64)
        self._pat = T

    def _prior_matrix(self, theta, pattern=False):
        spec = self.spec
        th = np.asarray(theta, dtype=np.float64)
        blocks = []
        if spec.n_fixed:
            blocks.append(sp.identity(spec.n_fixed, format="csr") * spec.fixed_prior_prec)
        for c in spec.components:
            k = c.theta_index
            if c.kind in ("iid", "rw1", "rw2", "besag"):
                R = _structure(c.kind, c.size, c.graph)
                g = 1.0 if pattern else math.exp(th[k])
                blocks.append((R * g + sp.identity(c.size) * spec.jitter).tocsr())
                continue
            if c.kind == "ar1":
                rho = 0.5 if pattern else 1.0 / (1.0 + math.exp(-th[k + 1]))
                tau = 1.0 if pattern else math.exp(th[k])
                blocks.append((tau * _q_ar1(c.nt, rho)).tocsr())
                continue
            G = _lattice_G(c.graph.nx, c.graph.ny)
            tau = 1.0 if pattern else math.exp(th[k])
            kap2 = 1.0 if pattern else math.exp(2.0 * th[k + 1])
            Qs = tau * (kap2 * kap2 * sp.identity(G.shape[0]) + 2.0 * kap2 * G + G @ G)
            if c.kind == "spde2d":
                blocks.append(Qs.tocsr())
            else:
                rho = 0.5 if pattern else 1.0 / (1.0 + math.exp(-th[k + 2]))
                blocks.append(sp.kron(_q_ar1(c.nt, rho), Qs, format="csr"))
        return sp.block_diag(blocks, format="csr")

    def prior_values(self, theta):
        """Values of Q_prior(theta) on the fixed lower-CSC pattern."""
        with np.errstate(over="ignore", invalid="ignore"):
            M = sp.tril(self._prior_matrix(theta)).tocsc()
        M.sort_indices()
        # map onto the fixed pattern (entries may be missing if a gain is 0)
        out = np.zeros(self.p_indices.shape[0])
        cols = np.repeat(np.arange(self.n), np.diff(M.indptr))
        key = cols * self.n + M.indices
        pcols = np.repeat(np.arange(self.n), np.diff(self.p_indptr))
        pkey = pcols * self.n + self.p_indices
        out[np.searchsorted(pkey, key)] = M.data
        return out

    def tau_noise(self, theta):
        sp_ = self.spec
        return math.exp(theta[sp_.noise_theta]) if sp_.noise_theta is not None else float(sp_.noise_precision)

    def lik(self, eta, theta):
        """model.py:302-331."""
        spec = self.spec
        full = eta + spec.offsets
        if spec.family == "gaussian":
            tau = self.tau_noise(theta)
            r = self.y - full
            ll = 0.5 * self.m * (math.log(tau) - LOG_2PI) - 0.5 * tau * float(r @ r)
            return ll, tau * r, np.full(self.m, -tau)
        from scipy.special import gammaln

        mu = spec.exposures * np.exp(full)
        y = self.y
        ll = float(np.sum(y * full + y * np.log(spec.exposures)) - np.sum(mu) - np.sum(gammaln(y + 1.0)))
        return ll, y - mu, -mu

    def log_prior_hyper(self, theta):
        """model.py:285-299 applied to every theta_j."""
        a, b = self.spec.hyper_shapes_rates()
        th = np.asarray(theta, dtype=np.float64)
        terms = a * np.log(b) + a * th - b * np.exp(th)
        terms -= np.array([math.lgamma(v) for v in a])
        return float(np.sum(terms))


# ----------------------------------------------------------------------
# objective (objective.py)


class OracleEvaluator:
    """objective.py:104-331 restated on the oracle kernels."""

    def __init__(self, spec, y, inner_tol=1e-8, max_inner=50, ordering="nested-dissection",
                 leaf_cutoff=64, ascent="reference"):
        # ascent: "reference" = g(x_try) >= g(x) on rounded totals
        # (objective.py:283-287); "termwise" = the same test evaluated as a sum
        # of per-term differences (the B200 engine's rule, engine.cu
        # mode_batch / vec.cu gdiff_kernel), which decides the near-floor
        # steps where the totals' rounding would otherwise flip a coin
        self.ascent = ascent
        self.model = OracleModel(spec, y)
        mdl = self.model
        n = mdl.n
        self.n = n
        self.inner_tol, self.max_inner = float(inner_tol), int(max_inner)
        self.spec = spec
        self.l2 = 1  # level-2 workers per factorization (ThreadBudget.l2)
        self.sym_prior = analyze(n, mdl.p_indptr, mdl.p_indices, ordering, leaf_cutoff)
        # Gram pairs (objective.py:79-101, 137-146)
        A = mdl.A
        rows, cols, obs, coef = [], [], [], []
        cnt = np.diff(A.indptr)
        # vectorised pair enumeration per row-length class
        for r in np.unique(cnt):
            ri = np.flatnonzero(cnt == r)
            base = A.indptr[ri]
            for a in range(r):
                for b in range(a, r):
                    ja = A.indices[base + a]
                    jb = A.indices[base + b]
                    rows.append(np.maximum(ja, jb))
                    cols.append(np.minimum(ja, jb))
                    obs.append(ri)
                    coef.append(A.data[base + a] * A.data[base + b])
        pr = np.concatenate(rows).astype(np.int64)
        pc = np.concatenate(cols).astype(np.int64)
        pobs = np.concatenate(obs).astype(np.int64)
        pcoef = np.concatenate(coef)
        o = np.lexsort((pobs, pr, pc))  # by col, row, then observation (reference order)
        pr, pc, pobs, pcoef = pr[o], pc[o], pobs[o], pcoef[o]
        gkey = pc * n + pr
        gram_keys, self.gram_dst = np.unique(gkey, return_inverse=True)
        self.gram_obs, self.gram_coef, self.gram_nnz = pobs, pcoef, gram_keys.shape[0]
        pcols = np.repeat(np.arange(n, dtype=np.int64), np.diff(mdl.p_indptr))
        prior_keys = pcols * n + mdl.p_indices
        ckeys = np.union1d(prior_keys, gram_keys)
        cr, cc = ckeys % n, ckeys // n
        self.c_indptr = np.zeros(n + 1, np.int64)
        np.add.at(self.c_indptr, cc + 1, 1)
        np.cumsum(self.c_indptr, out=self.c_indptr)
        self.c_indices = cr.astype(np.int64)
        self.prior_to_cond = np.searchsorted(ckeys, prior_keys)
        self.gram_to_cond = np.searchsorted(ckeys, gram_keys)
        self.c_nnz = ckeys.shape[0]
        self.sym_cond = analyze(n, self.c_indptr, self.c_indices, ordering, leaf_cutoff)
        self.gram_unit = np.bincount(self.gram_dst, weights=self.gram_coef, minlength=self.gram_nnz)

    def cond_values(self, pvals, weights=None, tau=None):
        vals = np.zeros(self.c_nnz)
        vals[self.prior_to_cond] += pvals
        if weights is None:
            vals[self.gram_to_cond] += tau * self.gram_unit
        else:
            g = np.bincount(self.gram_dst, weights=weights[self.gram_obs] * self.gram_coef,
                            minlength=self.gram_nnz)
            vals[self.gram_to_cond] += g
        return vals

    def mode(self, theta, warm=None):
        """objective.py:235-296 -> (x, Lx_cond, logdet_cond, pvals, iterations)."""
        mdl = self.model
        theta = np.asarray(theta, dtype=np.float64)
        pv = mdl.prior_values(theta)
        n = self.n
        if self.spec.family == "gaussian":
            tau = mdl.tau_noise(theta)
            cv = self.cond_values(pv, tau=tau)
            Lx, ld = factorize(self.sym_cond, cv, self.l2)
            rhs = mdl.AT @ (tau * (mdl.y - self.spec.offsets))
            return solve(self.sym_cond, Lx, rhs), Lx, ld, pv, 1
        x = np.zeros(n) if warm is None else np.array(warm, dtype=np.float64)
        for it in range(1, self.max_inner + 1):
            ll, d1, d2 = mdl.lik(mdl.A @ x, theta)
            qx = sym_matvec(n, mdl.p_indptr, mdl.p_indices, pv, x)
            g0 = -0.5 * float(x @ qx) + ll
            w = np.clip(-d2, 1e-12, None)
            cv = self.cond_values(pv, weights=w)
            Lx, ld = factorize(self.sym_cond, cv, self.l2)
            grad = (mdl.AT @ d1) - qx
            delta = solve(self.sym_cond, Lx, grad)
            if np.max(np.abs(delta)) <= self.inner_tol * (1.0 + np.max(np.abs(x))):
                return x, Lx, ld, pv, it
            ok, alpha, best = False, 1.0, -np.inf
            eta = mdl.A @ x
            for _ in range(11):
                xt = x + alpha * delta
                lt, _, _ = mdl.lik(mdl.A @ xt, theta)
                qt = sym_matvec(n, mdl.p_indptr, mdl.p_indices, pv, xt)
                gt = -0.5 * float(xt @ qt) + lt
                if self.ascent == "termwise":
                    de = mdl.A @ xt - eta
                    diff = float(np.sum(mdl.y * de + d2 * np.expm1(de))) - 0.5 * float((xt - x) @ (qt + qx))
                else:
                    diff = gt - g0
                if np.isfinite(gt):
                    best = max(best, diff)
                if np.isfinite(gt) and diff >= 0.0:
                    x, ok = xt, True
                    break
                alpha *= 0.5
            if not ok:
                if best >= -1e-9 * (1.0 + abs(g0)):
                    return x, Lx, ld, pv, it
                raise InnerDiv("no ascent step found")
        raise InnerDiv("not converged")

    def eval(self, theta, warm=None):
        """objective.py:298-331 -> dict of f and its components."""
        mdl = self.model
        theta = np.asarray(theta, dtype=np.float64)
        x, Lc, ldc, pv, its = self.mode(theta, warm)
        _, ldp = factorize(self.sym_prior, pv, self.l2)
        quad = float(x @ sym_matvec(self.n, mdl.p_indptr, mdl.p_indices, pv, x))
        ll, _, _ = mdl.lik(mdl.A @ x, theta)
        lph = mdl.log_prior_hyper(theta)
        lpl = 0.5 * ldp - 0.5 * self.n * LOG_2PI - 0.5 * quad
        lga = 0.5 * ldc - 0.5 * self.n * LOG_2PI
        return dict(f=-(lph + lpl + ll - lga), log_prior_hyper=lph, log_prior_latent=lpl,
                    log_likelihood=ll, log_gaussian_approx=lga, logdet_cond=ldc, logdet_prior=ldp,
                    iterations=its, mode=x, Lcond=Lc)

    def objective(self, theta, warm=None):
        try:
            return self.eval(theta, warm)["f"]
        except (NotPD, InnerDiv):
            return float("inf")

    def variances(self, theta, warm=None):
        x, Lc, _, _, _ = self.mode(theta, warm)
        return selected_inverse(self.sym_cond, Lc)[1]

    def eval_batch(self, points, warm=None, threads=None, l2=None):
        """Level-1 parallel batch (runtime.py:134-177): one thread per point,
        each factorization on ``l2`` level-2 workers (cholesky.py:295-319);
        the C kernels release the GIL (ctypes)."""
        threads = threads or min(len(points), os.cpu_count() or 1)
        if l2 is not None:
            self.l2 = max(1, int(l2))
        with ThreadPoolExecutor(max_workers=threads) as pool:
            return list(pool.map(lambda p: self.objective(p, warm), points))
