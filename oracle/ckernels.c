/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product.
 *
 * Plain-C restatement of the reference's numba kernels
 * (/root/reference/pkg/src/parinla/kernels.py).  Used by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * --impl reference arm as the CPU implementation of the reference path.
 * All indices are int64 like the reference; all values float64.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef int64_t i64;

/* kernels.py:16-30 — elimination tree from the strictly-lower row pattern */
void orc_etree(i64 n, const i64* rowptr, const i64* rowcol, i64* parent, i64* ancestor) {
  for (i64 j = 0; j < n; ++j) { parent[j] = -1; ancestor[j] = -1; }
  for (i64 j = 0; j < n; ++j) {
    for (i64 t = rowptr[j]; t < rowptr[j + 1]; ++t) {
      i64 k = rowcol[t];
      while (k != -1 && k < j) {
        i64 next = ancestor[k];
        ancestor[k] = j;
        if (next == -1) parent[k] = j;
        k = next;
      }
    }
  }
}

/* kernels.py:33-69, first pass — column counts of L (diagonal included) */
void orc_colcount(i64 n, const i64* rowptr, const i64* rowcol, const i64* parent, i64* mark,
                  i64* colcount) {
  for (i64 j = 0; j < n; ++j) { mark[j] = -1; colcount[j] = 1; }
  for (i64 j = 0; j < n; ++j) {
    mark[j] = j;
    for (i64 t = rowptr[j]; t < rowptr[j + 1]; ++t) {
      i64 k = rowcol[t];
      while (mark[k] != j) { mark[k] = j; colcount[k] += 1; k = parent[k]; }
    }
  }
}

/* kernels.py:33-69, second pass — row indices of L, diagonal first, ascending */
void orc_pattern(i64 n, const i64* rowptr, const i64* rowcol, const i64* parent, const i64* Lp,
                 i64* Li, i64* mark, i64* next) {
  for (i64 j = 0; j < n; ++j) { Li[Lp[j]] = j; next[j] = Lp[j] + 1; mark[j] = -1; }
  for (i64 j = 0; j < n; ++j) {
    mark[j] = j;
    for (i64 t = rowptr[j]; t < rowptr[j + 1]; ++t) {
      i64 k = rowcol[t];
      while (mark[k] != j) { mark[k] = j; Li[next[k]++] = j; k = parent[k]; }
    }
  }
}

/* kernels.py:72-96 — strictly-lower row form of L with storage positions */
void orc_row_form(i64 n, const i64* Lp, const i64* Li, i64* rowptr, i64* rowcol, i64* rowpos,
                  i64* w) {
  for (i64 j = 0; j <= n; ++j) rowptr[j] = 0;
  for (i64 j = 0; j < n; ++j)
    for (i64 p = Lp[j] + 1; p < Lp[j + 1]; ++p) rowptr[Li[p] + 1] += 1;
  for (i64 j = 0; j < n; ++j) rowptr[j + 1] += rowptr[j];
  for (i64 j = 0; j < n; ++j) w[j] = rowptr[j];
  for (i64 k = 0; k < n; ++k)
    for (i64 p = Lp[k] + 1; p < Lp[k + 1]; ++p) {
      i64 j = Li[p];
      i64 t = w[j]++;
      rowcol[t] = k;
      rowpos[t] = p;
    }
}

/* kernels.py:99-143 — up-looking Cholesky of permuted rows [start, end).
 * x is a zeroed scatter workspace of length n (restored on exit).
 * Returns the failing permuted row, or -1. */
i64 orc_factor_range(i64 start, i64 end, const i64* Lp, const i64* Li, double* Lx,
                     const i64* rowptr, const i64* rowcol, const i64* rowpos, const i64* arowptr,
                     const i64* arowcol, const i64* asrc, const i64* adiag, const double* qvals,
                     double* x, double rel_tol) {
  for (i64 j = start; j < end; ++j) {
    for (i64 t = arowptr[j]; t < arowptr[j + 1]; ++t) x[arowcol[t]] = qvals[asrc[t]];
    double qjj = qvals[adiag[j]];
    double d = qjj;
    for (i64 t = rowptr[j]; t < rowptr[j + 1]; ++t) {
      i64 k = rowcol[t];
      double xk = x[k];
      x[k] = 0.0;
      double ljk = xk / Lx[Lp[k]];
      i64 pend = rowpos[t];
      for (i64 p = Lp[k] + 1; p < pend; ++p) x[Li[p]] -= Lx[p] * ljk;
      Lx[pend] = ljk;
      d -= ljk * ljk;
    }
    if (qjj <= 0.0 || !(d > rel_tol * qjj)) {
      for (i64 t = rowptr[j]; t < rowptr[j + 1]; ++t) x[rowcol[t]] = 0.0;
      return j;
    }
    Lx[Lp[j]] = sqrt(d);
  }
  return -1;
}

/* kernels.py:146-154 — forward solve L y = b in place */
void orc_solve_lower(i64 n, const i64* Lp, const i64* Li, const double* Lx, double* b) {
  for (i64 j = 0; j < n; ++j) {
    double yj = b[j] / Lx[Lp[j]];
    b[j] = yj;
    for (i64 p = Lp[j] + 1; p < Lp[j + 1]; ++p) b[Li[p]] -= Lx[p] * yj;
  }
}

/* kernels.py:157-165 — backward solve L^T x = b in place */
void orc_solve_lower_t(i64 n, const i64* Lp, const i64* Li, const double* Lx, double* b) {
  for (i64 j = n - 1; j >= 0; --j) {
    double s = b[j];
    for (i64 p = Lp[j] + 1; p < Lp[j + 1]; ++p) s -= Lx[p] * b[Li[p]];
    b[j] = s / Lx[Lp[j]];
  }
}

/* kernels.py:185-246 — Takahashi recursion over columns [start, end), descending,
 * on V = L D^{-1/2}; zwork (n) / stamp (n, init -1) are scatter workspaces. */
i64 orc_selinv_range(i64 start, i64 end, const i64* Lp, const i64* Li, const double* Lx, double* Sx,
                     const i64* rowptr, const i64* rowcol, const i64* rowpos, double* zwork,
                     i64* stamp) {
  i64 count = 0;
  for (i64 i = end - 1; i >= start; --i) {
    i64 p0 = Lp[i], p1 = Lp[i + 1];
    double lii = Lx[p0];
    for (i64 t = p0 + 1; t < p1; ++t) {
      i64 k = Li[t];
      double v = Lx[t] / lii;
      for (i64 p = Lp[k]; p < Lp[k + 1]; ++p) {
        i64 r = Li[p];
        double c = v * Sx[p];
        if (stamp[r] == i) zwork[r] += c; else { stamp[r] = i; zwork[r] = c; }
      }
      i64 lo = rowptr[k], hi = rowptr[k + 1];
      while (lo < hi) {
        i64 mid = (lo + hi) >> 1;
        if (rowcol[mid] <= i) lo = mid + 1; else hi = mid;
      }
      for (i64 q = lo; q < rowptr[k + 1]; ++q) {
        i64 j = rowcol[q];
        double c = v * Sx[rowpos[q]];
        if (stamp[j] == i) zwork[j] += c; else { stamp[j] = i; zwork[j] = c; }
      }
    }
    for (i64 idx = p1 - 1; idx > p0; --idx) {
      i64 j = Li[idx];
      Sx[idx] = (stamp[j] == i) ? -zwork[j] : 0.0;
      count++;
    }
    double s = 0.0;
    for (i64 t = p0 + 1; t < p1; ++t) s += (Lx[t] / lii) * Sx[t];
    Sx[p0] = 1.0 / (lii * lii) - s;
    count++;
  }
  return count;
}

/* kernels.py:283-298 — out += Q x for lower-stored symmetric Q */
void orc_sym_matvec(i64 n, const i64* indptr, const i64* indices, const double* data,
                    const double* x, double* out) {
  for (i64 j = 0; j < n; ++j) {
    double xj = x[j], acc = 0.0;
    for (i64 p = indptr[j]; p < indptr[j + 1]; ++p) {
      i64 i = indices[p];
      double v = data[p];
      if (i == j) acc += v * xj;
      else { acc += v * x[i]; out[i] += v * xj; }
    }
    out[j] += acc;
  }
}

/* log det = 2 * sum(log diag L) (cholesky.py:321, numpy np.sum there).
 * Summed with Kahan compensation rather than numpy's pairwise order: both
 * are accurate to ~1e-16 relative, so they agree far inside the 1e-14 pins. */
double orc_logdiag_sum(i64 n, const i64* Lp, const double* Lx) {
  double s = 0.0, c = 0.0;  /* Kahan-compensated: order-independent to ~1e-16 */
  for (i64 j = 0; j < n; ++j) {
    double y = log(Lx[Lp[j]]) - c;
    double t = s + y;
    c = (t - s) - y;
    s = t;
  }
  return s;
}
