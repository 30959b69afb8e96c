// Native nested-dissection ordering for general GMRF patterns (host, C++).
//
// The reference orders every pattern with a pure-Python recursive
// vertex-separator nested dissection (/root/reference/pkg/src/parinla/
// ordering.py:206-423): dense vertices peeled into the root separator
// (:221-226), connected components in ascending-seed order (:277-301),
// BFS level-set separators from a pseudo-peripheral root (:304-382),
// boundary side selection (:385-404) and separator shrinking (:407-423),
// minimum-degree leaves with smallest-index tie break (:168-203).  This file
// restates that algorithm decision for decision, so the permutation is the
// reference's (bitwise; tests/test_nd_native.py pins it against golden
// permutations the reference produced), in O(n log n)-ish native code: the
// Python version takes minutes at n = 1e5 and more at 1e6
// (SURVEY s2, s6.2).
//
// The separator tree then drives the TILE partition of the B200 engine:
// every subtree that spans at most `tile_max` vertices becomes ONE dense
// tile (supernode amalgamation of small subtrees), consecutive small
// sibling subtrees are packed into one tile, and larger separators are cut
// into the fewest balanced tiles.  No tile crosses from one subtree into a
// sibling's separator, so the tile pattern keeps the ND fill structure.
#include <algorithm>
#include <cstdint>
#include <functional>
#include <queue>
#include <set>
#include <stdexcept>
#include <utility>
#include <vector>

#include "ordering.hpp"

namespace pinla {

namespace {

struct Graph {
  int64_t n;
  std::vector<int64_t> ptr, idx;  // sorted neighbour lists, no self loops
  int64_t deg(int64_t v) const { return ptr[v + 1] - ptr[v]; }
};

// build_adjacency (ordering.py:62-66 + :36-50): one edge per strictly-lower
// entry of the lower-CSC pattern, symmetrised, deduplicated, sorted.
Graph graph_of_lower(int64_t n, const int64_t* indptr, const int64_t* indices) {
  Graph g;
  g.n = n;
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t k = indptr[c]; k < indptr[c + 1]; ++k) {
      const int64_t r = indices[k];
      if (r < 0 || r >= n) throw std::runtime_error("pattern index out of range");
      if (r == c) continue;
      cnt[r + 1]++;
      cnt[c + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int64_t> tmp(cnt[n]);
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t k = indptr[c]; k < indptr[c + 1]; ++k) {
      const int64_t r = indices[k];
      if (r == c) continue;
      tmp[pos[r]++] = c;
      tmp[pos[c]++] = r;
    }
  g.ptr.assign(n + 1, 0);
  g.idx.reserve(tmp.size());
  for (int64_t v = 0; v < n; ++v) {
    auto b = tmp.begin() + cnt[v], e = tmp.begin() + cnt[v + 1];
    std::sort(b, e);
    e = std::unique(b, e);
    g.idx.insert(g.idx.end(), b, e);
    g.ptr[v + 1] = (int64_t)g.idx.size();
  }
  return g;
}

struct ND {
  const Graph& g;
  int64_t leaf_cutoff;
  std::vector<int64_t> order;
  std::vector<NDNode> nodes;
  // scratch, all reset to their neutral value after use
  std::vector<char> member, seen;
  std::vector<int64_t> level_of;
  std::vector<char> side;  // 1 = part A, 2 = part B, 3 = separator

  ND(const Graph& gr, int64_t lc)
      : g(gr), leaf_cutoff(lc), member(gr.n, 0), seen(gr.n, 0), level_of(gr.n, -1), side(gr.n, 0) {}

  int new_node(int64_t start, int64_t end, bool leaf, const std::vector<int>& children) {
    NDNode nd;
    nd.start = start;
    nd.end = end;
    nd.leaf = leaf;
    nd.children = children;
    nd.span_start = start;
    for (int c : children) nd.span_start = std::min(nd.span_start, nodes[c].span_start);
    const int id = (int)nodes.size();
    for (int c : children) nodes[c].parent = id;
    nodes.push_back(std::move(nd));
    return id;
  }

  // _minimum_degree_sequence (ordering.py:178-203): greedy elimination on
  // the induced subgraph with explicit fill; the heap pops the smallest
  // (degree, vertex) pair, stale entries are skipped.  The pop sequence is a
  // function of the heap CONTENTS only, so it is the reference's.
  void min_degree(const std::vector<int64_t>& verts) {
    const int64_t k = (int64_t)verts.size();
    std::vector<std::set<int64_t>> adj(k);
    // local ids follow the (sorted) vertex order, so comparisons on local
    // ids equal comparisons on vertex ids
    auto local = [&](int64_t v) {
      auto it = std::lower_bound(verts.begin(), verts.end(), v);
      return (it != verts.end() && *it == v) ? (int64_t)(it - verts.begin()) : (int64_t)-1;
    };
    for (int64_t i = 0; i < k; ++i) {
      const int64_t v = verts[i];
      for (int64_t e = g.ptr[v]; e < g.ptr[v + 1]; ++e) {
        const int64_t u = local(g.idx[e]);
        if (u >= 0) adj[i].insert(u);
      }
    }
    using P = std::pair<int64_t, int64_t>;
    std::priority_queue<P, std::vector<P>, std::greater<P>> heap;
    for (int64_t i = 0; i < k; ++i) heap.push({(int64_t)adj[i].size(), i});
    std::vector<char> alive(k, 1);
    while (!heap.empty()) {
      auto [d, v] = heap.top();
      heap.pop();
      if (!alive[v] || d != (int64_t)adj[v].size()) continue;
      order.push_back(verts[v]);
      alive[v] = 0;
      std::vector<int64_t> nb(adj[v].begin(), adj[v].end());  // sorted
      adj[v].clear();
      for (int64_t u : nb) adj[u].erase(v);
      for (size_t a = 0; a < nb.size(); ++a)
        for (size_t b = a + 1; b < nb.size(); ++b)
          if (!adj[nb[a]].count(nb[b])) {
            adj[nb[a]].insert(nb[b]);
            adj[nb[b]].insert(nb[a]);
          }
      for (int64_t u : nb) heap.push({(int64_t)adj[u].size(), u});
    }
  }

  int emit_leaf(const std::vector<int64_t>& comp) {  // comp sorted
    const int64_t start = (int64_t)order.size();
    min_degree(comp);
    return new_node(start, (int64_t)order.size(), true, {});
  }

  // _connected_components (ordering.py:277-301): ascending seeds, each sorted
  std::vector<std::vector<int64_t>> components(const std::vector<int64_t>& verts) {
    for (int64_t v : verts) member[v] = 1;
    std::vector<std::vector<int64_t>> comps;
    for (int64_t v : verts) {  // verts sorted
      if (seen[v]) continue;
      std::vector<int64_t> comp{v};
      seen[v] = 1;
      for (size_t h = 0; h < comp.size(); ++h) {
        const int64_t u = comp[h];
        for (int64_t e = g.ptr[u]; e < g.ptr[u + 1]; ++e) {
          const int64_t w = g.idx[e];
          if (member[w] && !seen[w]) {
            seen[w] = 1;
            comp.push_back(w);
          }
        }
      }
      std::sort(comp.begin(), comp.end());
      comps.push_back(std::move(comp));
    }
    for (int64_t v : verts) member[v] = seen[v] = 0;
    return comps;
  }

  // _bfs_levels (ordering.py:304-318): member set is `member`; levels sorted.
  // Leaves level_of set for the returned vertices (caller resets).
  std::vector<std::vector<int64_t>> bfs_levels(int64_t root) {
    std::vector<std::vector<int64_t>> levels{{root}};
    level_of[root] = 0;
    std::vector<int64_t> frontier{root};
    while (!frontier.empty()) {
      std::vector<int64_t> nxt;
      for (int64_t u : frontier)
        for (int64_t e = g.ptr[u]; e < g.ptr[u + 1]; ++e) {
          const int64_t w = g.idx[e];
          if (member[w] && level_of[w] < 0) {
            level_of[w] = level_of[u] + 1;
            nxt.push_back(w);
          }
        }
      if (!nxt.empty()) {
        std::sort(nxt.begin(), nxt.end());
        levels.push_back(nxt);
      }
      frontier = std::move(nxt);
    }
    return levels;
  }
  void clear_levels(const std::vector<std::vector<int64_t>>& levels) {
    for (auto& lv : levels)
      for (int64_t v : lv) level_of[v] = -1;
  }

  // _pseudo_peripheral (ordering.py:321-331): start at the first vertex of
  // minimum (full-graph) degree, then up to 8 sweeps to the min-(degree,
  // id) vertex of the last level while the eccentricity grows
  int64_t pseudo_peripheral(const std::vector<int64_t>& comp) {
    int64_t root = comp[0];
    for (int64_t v : comp)
      if (g.deg(v) < g.deg(root)) root = v;
    int64_t ecc = -1;
    for (int it = 0; it < 8; ++it) {
      auto levels = bfs_levels(root);
      clear_levels(levels);
      const int64_t h = (int64_t)levels.size() - 1;
      if (h <= ecc) break;
      ecc = h;
      const auto& last = levels.back();
      int64_t best = last[0];
      for (int64_t v : last)
        if (g.deg(v) < g.deg(best) || (g.deg(v) == g.deg(best) && v < best)) best = v;
      root = best;
    }
    return root;
  }

  bool touches(int64_t v, char s) const {
    for (int64_t e = g.ptr[v]; e < g.ptr[v + 1]; ++e)
      if (side[g.idx[e]] == s) return true;
    return false;
  }

  // _level_set_separator (ordering.py:334-382) + _boundary_separator
  // (:385-404) + _shrink_separator (:407-423).  Returns false when the
  // component has no usable level structure.
  bool separator(const std::vector<int64_t>& comp, std::vector<int64_t>& sep,
                 std::vector<int64_t>& pa, std::vector<int64_t>& pb) {
    for (int64_t v : comp) member[v] = 1;
    const int64_t root = pseudo_peripheral(comp);
    auto levels = bfs_levels(root);
    const int64_t h = (int64_t)levels.size() - 1;
    bool found = false;
    if (h >= 1) {
      std::vector<int64_t> cum(levels.size());
      int64_t acc = 0;
      for (size_t d = 0; d < levels.size(); ++d) cum[d] = acc += (int64_t)levels[d].size();
      const double half = (double)cum.back() / 2.0;
      int64_t m_star = (int64_t)(std::lower_bound(cum.begin(), cum.end(), half,
                                                  [](int64_t a, double b) { return (double)a < b; }) -
                                 cum.begin());
      m_star = std::min(std::max<int64_t>(m_star, 1), h);
      std::vector<int64_t> cand;
      for (int64_t m = 1; m <= h; ++m) cand.push_back(m);
      std::stable_sort(cand.begin(), cand.end(), [&](int64_t a, int64_t b) {
        const int64_t da = std::llabs(a - m_star), db = std::llabs(b - m_star);
        return da != db ? da < db : a < b;
      });
      for (int64_t m : cand) {
        // boundary sides of level m
        std::vector<int64_t> prev, next;
        for (int64_t v : levels[m]) {
          bool p = false, q = false;
          for (int64_t e = g.ptr[v]; e < g.ptr[v + 1]; ++e) {
            const int64_t l = level_of[g.idx[e]];
            if (l == m - 1) p = true;
            if (m < h && l == m + 1) q = true;
          }
          if (p) prev.push_back(v);
          if (q) next.push_back(v);
        }
        if (prev.empty() && next.empty()) continue;
        bool use_prev;
        if (prev.empty()) use_prev = false;
        else if (next.empty()) use_prev = true;
        else use_prev = prev.size() <= next.size();
        const std::vector<int64_t>& s0 = use_prev ? prev : next;
        // parts: below / at / above (ordering.py:365-372)
        for (int64_t v : s0) side[v] = 3;
        int64_t na = 0, nb = 0;
        for (int64_t d = 0; d <= h; ++d)
          for (int64_t v : levels[d]) {
            if (side[v] == 3) continue;
            char s;
            if (d < m) s = 1;
            else if (d == m) s = use_prev ? 2 : 1;
            else s = 2;
            side[v] = s;
            (s == 1 ? na : nb)++;
          }
        if (na == 0 || nb == 0) {
          for (int64_t v : comp) side[v] = 0;
          continue;
        }
        // shrink: repeated passes over the (sorted) separator
        std::vector<int64_t> cur(s0.begin(), s0.end());  // sorted (levels sorted)
        bool changed = true;
        while (changed) {
          changed = false;
          std::vector<int64_t> keep;
          for (int64_t v : cur) {
            const bool ta = touches(v, 1), tb = touches(v, 2);
            if (ta && tb) {
              keep.push_back(v);
              continue;
            }
            char s;
            if (ta) s = 1;
            else if (tb) s = 2;
            else s = na <= nb ? 1 : 2;
            side[v] = s;
            (s == 1 ? na : nb)++;
            changed = true;
          }
          cur.swap(keep);
        }
        if (!cur.empty() && na > 0 && nb > 0) {
          sep.clear();
          pa.clear();
          pb.clear();
          for (int64_t v : comp) {  // comp sorted -> outputs sorted
            if (side[v] == 3) sep.push_back(v);
            else if (side[v] == 1) pa.push_back(v);
            else pb.push_back(v);
          }
          found = true;
        }
        for (int64_t v : comp) side[v] = 0;
        if (found) break;
      }
    }
    clear_levels(levels);
    for (int64_t v : comp) member[v] = 0;
    return found;
  }

  // dissect (ordering.py:239-262)
  std::vector<int> dissect(const std::vector<int64_t>& verts) {
    if (!verts.empty() && (int64_t)verts.size() <= leaf_cutoff) return {emit_leaf(verts)};
    std::vector<int> tops;
    for (auto& comp : components(verts)) {
      if ((int64_t)comp.size() <= leaf_cutoff) {
        tops.push_back(emit_leaf(comp));
        continue;
      }
      std::vector<int64_t> sep, pa, pb;
      if (!separator(comp, sep, pa, pb)) {
        tops.push_back(emit_leaf(comp));
        continue;
      }
      std::vector<int> kids = dissect(pa);
      std::vector<int> kb = dissect(pb);
      kids.insert(kids.end(), kb.begin(), kb.end());
      const int64_t start = (int64_t)order.size();
      order.insert(order.end(), sep.begin(), sep.end());
      tops.push_back(new_node(start, (int64_t)order.size(), false, kids));
    }
    return tops;
  }
};

}  // namespace

NDResult nested_dissection(int64_t n, const int64_t* indptr, const int64_t* indices,
                           int64_t leaf_cutoff) {
  if (leaf_cutoff < 0) throw std::runtime_error("leaf_cutoff must be at least 1");
  Graph g = graph_of_lower(n, indptr, indices);
  if (leaf_cutoff == 0) {
    // minimum_degree_order (ordering.py:168-175): the whole graph as one
    // minimum-degree block, no dense peel
    ND md(g, n);
    std::vector<int64_t> all(n);
    for (int64_t v = 0; v < n; ++v) all[v] = v;
    NDResult r;
    r.root = n > 0 ? md.emit_leaf(all) : md.new_node(0, 0, true, {});
    r.perm = std::move(md.order);
    r.nodes = std::move(md.nodes);
    return r;
  }
  ND nd(g, leaf_cutoff);
  // dense peel (ordering.py:221-226)
  std::vector<int64_t> dense, keep;
  const int64_t cut = std::max<int64_t>(16, (n - 1) / 2);
  for (int64_t v = 0; v < n; ++v) {
    if (n > 32 && g.deg(v) >= cut) dense.push_back(v);
    else keep.push_back(v);
  }
  std::vector<int> tops = nd.dissect(keep);
  NDResult r;
  if (tops.size() == 1 && dense.empty()) {
    r.root = tops[0];
  } else {
    const int64_t start = (int64_t)nd.order.size();
    nd.order.insert(nd.order.end(), dense.begin(), dense.end());
    r.root = nd.new_node(start, (int64_t)nd.order.size(), false, tops);
  }
  r.n_dense = (int64_t)dense.size();
  r.perm = std::move(nd.order);
  r.nodes = std::move(nd.nodes);
  if ((int64_t)r.perm.size() != n) throw std::runtime_error("nested dissection lost vertices");
  return r;
}

// Tile partition from the separator tree (see the file comment).  Returns
// the tile start offsets (tile_max-bounded, covering [0, n - n_dense) and
// then the dense tail in tile_max pieces), as bounds t_0 = 0 < ... < t_NT = n.
std::vector<int64_t> nd_tile_bounds(const NDResult& r, int64_t tile_max) {
  std::vector<int64_t> sizes;
  const int64_t n = (int64_t)r.perm.size();
  auto span = [&](int id) { return r.nodes[id].end - r.nodes[id].span_start; };
  auto cut = [&](int64_t len) {  // fewest balanced pieces <= tile_max
    if (len <= 0) return;
    const int64_t k = (len + tile_max - 1) / tile_max;
    for (int64_t i = 0; i < k; ++i) sizes.push_back(len / k + (i < len % k ? 1 : 0));
  };
  // iterative post-order over the tree: (node, phase)
  std::function<void(int)> part = [&](int id) {
    const NDNode& nd = r.nodes[id];
    if (span(id) <= tile_max) {
      cut(span(id));
      return;
    }
    int64_t pack = 0;  // open tile of consecutive small sibling subtrees
    for (int c : nd.children) {
      if (span(c) <= tile_max) {
        if (pack + span(c) > tile_max) {
          cut(pack);
          pack = 0;
        }
        pack += span(c);
      } else {
        cut(pack);
        pack = 0;
        part(c);
      }
    }
    cut(pack);
    cut(nd.end - nd.start);
  };
  const NDNode& root = r.nodes[r.root];
  if (r.n_dense > 0) {
    // the dense root separator: its children first, then the arrow tiles
    int64_t pack = 0;
    for (int c : root.children) {
      if (span(c) <= tile_max) {
        if (pack + span(c) > tile_max) {
          cut(pack);
          pack = 0;
        }
        pack += span(c);
      } else {
        cut(pack);
        pack = 0;
        part(c);
      }
    }
    cut(pack);
    cut(root.end - root.start);
  } else {
    part(r.root);
  }
  std::vector<int64_t> b{0};
  for (int64_t s : sizes) b.push_back(b.back() + s);
  if (b.back() != n) throw std::runtime_error("tile partition does not cover the ordering");
  return b;
}

// Scalar symbolic factorization of the permuted pattern (the reference's
// analyze: etree + column patterns, cholesky.py:88-165 / kernels.py:16-96):
// Lp (n+1) and Li (nnz, per column the diagonal first, rows ascending).
// Liu's elimination tree with path compression, then each row's pattern by
// walking the tree up from the row's entries (row subtrees).
void scalar_pattern(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* perm,
                    std::vector<int64_t>& Lp, std::vector<int64_t>& Li) {
  std::vector<int64_t> iperm(n);
  for (int64_t k = 0; k < n; ++k) iperm[perm[k]] = k;
  std::vector<int64_t> rp(n + 1, 0);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t k = indptr[c]; k < indptr[c + 1]; ++k) {
      const int64_t a = iperm[indices[k]], b = iperm[c];
      if (a != b) rp[std::max(a, b) + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
  std::vector<int64_t> rc(rp[n]);
  {
    std::vector<int64_t> w(rp.begin(), rp.end() - 1);
    for (int64_t c = 0; c < n; ++c)
      for (int64_t k = indptr[c]; k < indptr[c + 1]; ++k) {
        const int64_t a = iperm[indices[k]], b = iperm[c];
        if (a != b) rc[w[std::max(a, b)]++] = std::min(a, b);
      }
  }
  std::vector<int64_t> parent(n, -1), anc(n, -1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
      int64_t j = rc[q];
      while (anc[j] != -1 && anc[j] != i) {
        const int64_t nx = anc[j];
        anc[j] = i;
        j = nx;
      }
      if (anc[j] == -1) {
        anc[j] = i;
        parent[j] = i;
      }
    }
  std::vector<int64_t> mark(n, -1), cnt(n, 1);
  auto walk = [&](auto&& visit) {
    std::fill(mark.begin(), mark.end(), -1);
    for (int64_t i = 0; i < n; ++i) {
      mark[i] = i;
      for (int64_t q = rp[i]; q < rp[i + 1]; ++q)
        for (int64_t j = rc[q]; mark[j] != i; j = parent[j]) {
          mark[j] = i;
          visit(i, j);
        }
    }
  };
  walk([&](int64_t, int64_t j) { cnt[j]++; });
  Lp.assign(n + 1, 0);
  for (int64_t j = 0; j < n; ++j) Lp[j + 1] = Lp[j] + cnt[j];
  Li.assign(Lp[n], 0);
  std::vector<int64_t> nxt(n);
  for (int64_t j = 0; j < n; ++j) {
    Li[Lp[j]] = j;
    nxt[j] = Lp[j] + 1;
  }
  walk([&](int64_t i, int64_t j) { Li[nxt[j]++] = i; });
}

}  // namespace pinla
