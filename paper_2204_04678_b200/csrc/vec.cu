// Batched vector kernels of the f(theta) pipeline: prior / conditional
// precision assembly, design SpMVs, likelihood terms, prior quadratic form and
// deterministic (fixed-order) reductions.  All are HBM-bound streaming
// kernels; every one processes all active theta slots of the batch in a
// single launch (gridDim.y = slot).
//
// Reference counterparts (/root/reference/pkg/src/parinla):
//   prior_values_kernel   assemble_prior_precision       model.py:263-282
//   cond_values_kernel    _cond_matrix / _cond_matrix_gaussian
//                                                         objective.py:195-210
//   spmv_A_kernel         A @ x (scipy CSR)              objective.py:262, 280, 313
//   at_chunk/at_combine   AT @ d1 - qx                   objective.py:271
//   symv_kernel + dot     _prior_matvec / x @ qx         objective.py:212-215, 264-265
//   lik_kernel            likelihood_terms               model.py:302-331
#include <algorithm>
#include <cmath>

#include "vec.cuh"

namespace pinla {

constexpr int kVT = 256;

// max that propagates NaN (np.max semantics): a NaN step or iterate must not
// pass the convergence test as a small |delta|
__device__ __forceinline__ double nan_max(double a, double b) {
  return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(a, b);
}

__global__ void prior_values_kernel(int64_t nnz, const int64_t* term_ptr, const int* term_gain,
                                    const double* term_coef, const double* pconst,
                                    const double* gains, int n_gains, double* pv,
                                    const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  const double* g = gains + (int64_t)s * n_gains;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t t = term_ptr[e]; t < term_ptr[e + 1]; ++t) v += term_coef[t] * g[term_gain[t]];
    pv[(int64_t)s * nnz + e] = v + pconst[e];
  }
}

// Gram chunk sums: chunk c = <= kGramChunk pairs of ONE entry, summed by one
// thread in pair order.  Chunks are laid out by length, 32 per group, pair k
// of the chunk at position 32 g + l at gbase[g] + 32 k + l (engine.cu): the
// lanes of a warp load consecutive words, and all of a thread's pair loads
// and weight gathers are in flight at once (two unrolled half-chunks).
__global__ void __launch_bounds__(256, 4) gram_chunk_kernel(
    int64_t npos, const int64_t* gbase, const uint8_t* clen, const int32_t* cperm, const int* gobs,
    const double* gcoef, const double* w, int64_t m, double* ch_out, int64_t nch,
    const int* active) {
  constexpr int kH = kGramChunk / 2;
  const int s = blockIdx.y;
  if (!active[s]) return;
  const double* ws = w + (int64_t)s * m;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < npos;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int n = clen[c];
    if (n == 0) continue;
    const int64_t b = gbase[c >> 5] + (c & 31);
    double g = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int ob[kH];
      double cf[kH], wv[kH];
#pragma unroll
      for (int k = 0; k < kH; ++k)
        if (h * kH + k < n) {
          ob[k] = gobs[b + 32 * (h * kH + k)];
          cf[k] = gcoef[b + 32 * (h * kH + k)];
        }
#pragma unroll
      for (int k = 0; k < kH; ++k)
        if (h * kH + k < n) wv[k] = ws[ob[k]];
#pragma unroll
      for (int k = 0; k < kH; ++k)
        if (h * kH + k < n) g += wv[k] * cf[k];
    }
    ch_out[(int64_t)s * nch + cperm[c]] = g;
  }
}

// mode: 0 gaussian (tau * gram_unit), 1 weights (sum of Gram chunk sums), 2 prior only
__global__ void cond_values_kernel(int64_t nq, const int64_t* psrc, int64_t nnz_p, const double* pv,
                                   const int64_t* gptr, const int64_t* e_ch, const double* ch_out,
                                   int64_t nch, const double* gunit, const double* tau, int mode,
                                   double* qv, const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  const double* pvs = pv + (int64_t)s * nnz_p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nq;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ps = psrc[e];
    double v = ps >= 0 ? pvs[ps] : 0.0;
    if (mode == 0) {
      if (gptr[e + 1] > gptr[e]) v += tau[s] * gunit[e];
    } else if (mode == 1) {
      const int64_t b = e_ch[e], en = e_ch[e + 1];
      if (en - b > kHeavyChunks) continue;  // written by heavy_entries_kernel
      if (en > b) {
        double g = 0.0;
        for (int64_t c = b; c < en; ++c) g += ch_out[(int64_t)s * nch + c];
        v += g;
      }
    }
    qv[(int64_t)s * nq + e] = v;
  }
}

// entries with many Gram chunks (fixed effect x fixed effect): one block per
// entry, fixed strided assignment + tree reduction (deterministic)
// Entries with many Gram chunks (fixed-effect pairs: up to m/16 chunks) in
// two fixed-order stages: part k of a heavy entry sums chunks [hp_c0[k],
// hp_c1[k]) with one block (strided per thread, then a tree), then each
// entry adds its parts in order to the prior value.
__global__ void heavy_parts_kernel(int64_t nhp, const int64_t* hp_c0, const int64_t* hp_c1,
                                   const double* ch_out, int64_t nch, double* hbuf,
                                   const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  __shared__ double red[kVT];
  for (int64_t k = blockIdx.x; k < nhp; k += gridDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const double* cs = ch_out + (int64_t)s * nch;
    int64_t c = hp_c0[k] + threadIdx.x;
    const int64_t ce = hp_c1[k];
    for (; c + 3 * kVT < ce; c += 4 * kVT) {
      a0 += cs[c];
      a1 += cs[c + kVT];
      a2 += cs[c + 2 * kVT];
      a3 += cs[c + 3 * kVT];
    }
    for (; c < ce; c += kVT) a0 += cs[c];
    red[threadIdx.x] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    for (int o = kVT / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) hbuf[(int64_t)s * nhp + k] = red[0];
    __syncthreads();
  }
}
__global__ void heavy_entries_kernel(int64_t nheavy, const int64_t* heavy, const int64_t* hpart_ptr,
                                     int64_t nhp, const double* hbuf, const int64_t* psrc,
                                     int64_t nnz_p, const double* pv, int64_t nq, double* qv,
                                     const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nheavy;
       h += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t k = hpart_ptr[h]; k < hpart_ptr[h + 1]; ++k) acc += hbuf[(int64_t)s * nhp + k];
    const int64_t e = heavy[h];
    const int64_t ps = psrc[e];
    qv[(int64_t)s * nq + e] = (ps >= 0 ? pv[(int64_t)s * nnz_p + ps] : 0.0) + acc;
  }
}
__global__ void spmv_A_kernel(int64_t m, const int64_t* ap, const int* aj, const double* ax,
                              const double* x, int64_t npad, double* eta, const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  const double* xs = x + (int64_t)s * npad;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t p = ap[i]; p < ap[i + 1]; ++p) v += ax[p] * xs[aj[p]];
    eta[(int64_t)s * m + i] = v;
  }
}

// likelihood at eta; writes d1 and the Newton weights w = max(-d2, 1e-12)
// (objective.py:267) when d1/w are non-null; per-block partial sums:
//   gaussian: part0 = sum r^2
//   poisson : part0 = sum (y*full + y*log E), part1 = sum mu
__global__ void lik_kernel(int64_t m, int family, const double* eta, const double* y,
                           const double* off, const double* logE, const double* E,
                           const double* tau, double* d1, double* w, double* parts, int nblk,
                           const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  __shared__ double red0[kVT], red1[kVT];
  double a0 = 0.0, a1 = 0.0;
  const double* es = eta + (int64_t)s * m;
  const double ts = tau[s];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double full = es[i] + off[i];
    if (family == 0) {
      const double r = y[i] - full;
      a0 += r * r;
      if (d1) d1[(int64_t)s * m + i] = ts * r;
    } else {
      const double mu = E[i] * exp(full);
      a0 += y[i] * full + y[i] * logE[i];
      a1 += mu;
      if (d1) {
        d1[(int64_t)s * m + i] = y[i] - mu;
        w[(int64_t)s * m + i] = mu != mu ? mu : fmax(mu, 1e-12);  // np.clip keeps NaN
      }
    }
  }
  red0[threadIdx.x] = a0;
  red1[threadIdx.x] = a1;
  __syncthreads();
  for (int o = kVT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red0[threadIdx.x] += red0[threadIdx.x + o];
      red1[threadIdx.x] += red1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    parts[((int64_t)s * nblk + blockIdx.x) * 2 + 0] = red0[0];
    parts[((int64_t)s * nblk + blockIdx.x) * 2 + 1] = red1[0];
  }
}

// g(x_t) - g(x) as sums of per-term differences (the halving search's ascent
// test, objective.py:283-286, evaluated without the cancellation of two
// rounded totals): parts[.., 0] = sum_i l_i(eta_t) - l_i(eta),
// parts[.., 1] = (x_t - x)^T Qp (x_t + x) = sum_j (x_t - x)_j (qx_t + qx)_j.
//   Poisson:  l_i(eta_t) - l_i(eta) = y (eta_t - eta) - mu expm1(eta_t - eta)
//   Gaussian: -tau/2 (r_t^2 - r^2) = tau/2 (eta_t - eta)(r_t + r)
__global__ void gdiff_kernel(int64_t m, int64_t npad, int family, const double* eta,
                             const double* eta_t, const double* y, const double* off,
                             const double* E, const double* tau, const double* x,
                             const double* x_t, const double* qx, const double* qx_t,
                             double* parts, int nblk, const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  __shared__ double red0[kVT], red1[kVT];
  double a0 = 0.0, a1 = 0.0;
  const double* es = eta + (int64_t)s * m;
  const double* et = eta_t + (int64_t)s * m;
  const double ts = tau[s];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double de = et[i] - es[i];
    if (family == 0) {
      const double r = y[i] - es[i] - off[i], rt = y[i] - et[i] - off[i];
      a0 += 0.5 * ts * de * (rt + r);
    } else {
      const double mu = E[i] * exp(es[i] + off[i]);
      a0 += y[i] * de - mu * expm1(de);
    }
  }
  const double* xs = x + (int64_t)s * npad;
  const double* xt = x_t + (int64_t)s * npad;
  const double* qs = qx + (int64_t)s * npad;
  const double* qt = qx_t + (int64_t)s * npad;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < npad;
       j += (int64_t)gridDim.x * blockDim.x)
    a1 += (xt[j] - xs[j]) * (qt[j] + qs[j]);
  red0[threadIdx.x] = a0;
  red1[threadIdx.x] = a1;
  __syncthreads();
  for (int o = kVT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red0[threadIdx.x] += red0[threadIdx.x + o];
      red1[threadIdx.x] += red1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    parts[((int64_t)s * nblk + blockIdx.x) * 2 + 0] = red0[0];
    parts[((int64_t)s * nblk + blockIdx.x) * 2 + 1] = red1[0];
  }
}

// chunked A^T d: chunk c covers entries [cb, ce) of padded row cr
__global__ void at_chunk_kernel(int64_t nch, const int* ch_row, const int64_t* ch_beg,
                                const int* at_obs, const double* at_val, const double* d1,
                                int64_t m, double* ch_out, const int* active) {
  // half a warp per chunk (rows of A^T are short: a lattice node sees the
  // observations of its few cells; the dense design columns have 256-entry
  // chunks and simply loop); fixed per-lane order + xor tree: deterministic
  const int s = blockIdx.y;
  if (!active[s]) return;
  const int hw = threadIdx.x >> 4, lane = threadIdx.x & 15;
  const double* ds = d1 + (int64_t)s * m;
  const int64_t nhw = (int64_t)gridDim.x * (blockDim.x / 16);
  for (int64_t c0 = (int64_t)blockIdx.x * (blockDim.x / 16) + hw - (hw & 1); c0 < nch; c0 += nhw) {
    // both halves of a warp iterate together (shuffles need the full warp)
    const int64_t c = c0 + (hw & 1);
    double v = 0.0;
    if (c < nch)
      for (int64_t p = ch_beg[c] + lane; p < ch_beg[c + 1]; p += 16) v += at_val[p] * ds[at_obs[p]];
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && c < nch) ch_out[(int64_t)s * nch + c] = v;
  }
}
// out[row] = sum of its chunks - sub[row]   (sub may be null)
__global__ void at_combine_kernel(int64_t npad, const int64_t* row_ch, int64_t nch,
                                  const double* ch_out, const double* sub, double* out,
                                  const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < npad;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (row_ch[r + 1] - row_ch[r] > kHeavyChunks) continue;  // at_heavy_rows_kernel
    double v = 0.0;
    for (int64_t c = row_ch[r]; c < row_ch[r + 1]; ++c) v += ch_out[(int64_t)s * nch + c];
    if (sub) v -= sub[(int64_t)s * npad + r];
    out[(int64_t)s * npad + r] = v;
  }
}
// rows of A^T with many chunks (the dense fixed-effect columns of A: m/256
// chunks): one block per row, fixed strided order + tree
__global__ void at_heavy_rows_kernel(int64_t nrows, const int64_t* rows, const int64_t* row_ch,
                                     int64_t nch, const double* ch_out, const double* sub,
                                     int64_t npad, double* out, const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  __shared__ double red[kVT];
  for (int64_t h = blockIdx.x; h < nrows; h += gridDim.x) {
    const int64_t r = rows[h];
    const double* cs = ch_out + (int64_t)s * nch;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t c = row_ch[r] + threadIdx.x;
    const int64_t ce = row_ch[r + 1];
    for (; c + 3 * kVT < ce; c += 4 * kVT) {
      a0 += cs[c];
      a1 += cs[c + kVT];
      a2 += cs[c + 2 * kVT];
      a3 += cs[c + 3 * kVT];
    }
    for (; c < ce; c += kVT) a0 += cs[c];
    red[threadIdx.x] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    for (int o = kVT / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[(int64_t)s * npad + r] = red[0] - (sub ? sub[(int64_t)s * npad + r] : 0.0);
    __syncthreads();
  }
}

// qx = Q_prior x (full symmetric CSR over padded rows, values from pv)
__global__ void symv_kernel(int64_t npad, const int64_t* qp, const int* qj, const int64_t* qvi,
                            const double* pv, int64_t nnz_p, const double* x, double* qx,
                            const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  const double* xs = x + (int64_t)s * npad;
  const double* ps = pv + (int64_t)s * nnz_p;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < npad;
       r += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t p = qp[r]; p < qp[r + 1]; ++p) v += ps[qvi[p]] * xs[qj[p]];
    qx[(int64_t)s * npad + r] = v;
  }
}

// per-block partials of (sum a*b, max|a|, max|b|)
__global__ void dot_max_kernel(int64_t npad, const double* a, const double* b, double* parts,
                               int nblk, const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  __shared__ double r0[kVT], r1[kVT], r2[kVT];
  double d = 0.0, ma = 0.0, mb = 0.0;
  const double* as = a + (int64_t)s * npad;
  const double* bs = b + (int64_t)s * npad;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npad;
       i += (int64_t)gridDim.x * blockDim.x) {
    d += as[i] * bs[i];
    ma = nan_max(ma, fabs(as[i]));
    mb = nan_max(mb, fabs(bs[i]));
  }
  r0[threadIdx.x] = d;
  r1[threadIdx.x] = ma;
  r2[threadIdx.x] = mb;
  __syncthreads();
  for (int o = kVT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      r0[threadIdx.x] += r0[threadIdx.x + o];
      r1[threadIdx.x] = nan_max(r1[threadIdx.x], r1[threadIdx.x + o]);
      r2[threadIdx.x] = nan_max(r2[threadIdx.x], r2[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* p = parts + ((int64_t)s * nblk + blockIdx.x) * 3;
    p[0] = r0[0];
    p[1] = r1[0];
    p[2] = r2[0];
  }
}

// fixed-order reduction of nblk partial records of width wdt per slot;
// op mask bit k: 1 = max, 0 = sum
__global__ void reduce_parts_kernel(const double* parts, int nblk, int wdt, int maxmask, double* out,
                                    const int* active) {
  const int s = blockIdx.x;
  if (!active[s]) return;
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k >= wdt) return;
  const bool mx = (maxmask >> k) & 1;
  double v = 0.0;
  for (int b = lane; b < nblk; b += 32) {
    const double p = parts[((int64_t)s * nblk + b) * wdt + k];
    v = mx ? nan_max(v, p) : v + p;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = mx ? nan_max(v, u) : v + u;
  }
  if (lane == 0) out[(int64_t)s * wdt + k] = v;
}

// accepted halving try -> iterate: for slots with sel[s] = t >= 0 copy try t's
// x, Qp x (npad) and eta, d1, w (m) into the iterate buffers
__global__ void take_try_kernel(int64_t npad, int64_t m, int S, const int* sel, const double* tx,
                                const double* tqx, const double* teta, const double* td1,
                                const double* tw, double* x, double* qx, double* eta, double* d1,
                                double* w) {
  const int s = blockIdx.y;
  const int t = sel[s];
  if (t < 0) return;
  const int64_t sn = (int64_t)s * npad, tn = ((int64_t)t * S + s) * npad;
  const int64_t sm = (int64_t)s * m, tm = ((int64_t)t * S + s) * m;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += stride) {
    x[sn + i] = tx[tn + i];
    qx[sn + i] = tqx[tn + i];
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    eta[sm + i] = teta[tm + i];
    d1[sm + i] = td1[tm + i];
    w[sm + i] = tw[tm + i];
  }
}

// y = x + alpha[s] * d   (per slot)
__global__ void axpy_kernel(int64_t npad, const double* x, const double* d, const double* alpha,
                            double* y, const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  const double al = alpha[s];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npad;
       i += (int64_t)gridDim.x * blockDim.x)
    y[(int64_t)s * npad + i] = x[(int64_t)s * npad + i] + al * d[(int64_t)s * npad + i];
}

// y = alpha[s] * x
__global__ void scale_kernel(int64_t npad, const double* x, const double* alpha, double* y,
                             const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npad;
       i += (int64_t)gridDim.x * blockDim.x)
    y[(int64_t)s * npad + i] = alpha[s] * x[i];
}


// ---------------------------------------------------------------------------

static dim3 grid_for(int64_t n, int S, int cap = 148 * 8) {
  int64_t b = (n + kVT - 1) / kVT;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return dim3((unsigned)b, (unsigned)S);
}

void vk_prior_values(const VecModel& M, const double* gains, double* pv, const int* active, int S,
                     cudaStream_t st) {
  prior_values_kernel<<<grid_for(M.nnz_p, S), kVT, 0, st>>>(M.nnz_p, M.term_ptr, M.term_gain,
                                                             M.term_coef, M.pconst, gains,
                                                             M.n_gains, pv, active);
}
void vk_cond_values(const VecModel& M, const double* pv, const double* tau, const double* w,
                    int mode, double* qv, double* gch_out, const int* active, int S,
                    cudaStream_t st) {
  if (mode == 1)
    gram_chunk_kernel<<<grid_for(M.gpos, S, 148 * 16), kVT, 0, st>>>(
        M.gpos, M.gbase, M.clen, M.cperm, M.gobs, M.gcoef, w, M.m, gch_out, M.ngch, active);
  cond_values_kernel<<<grid_for(M.nq, S), kVT, 0, st>>>(M.nq, M.psrc, M.nnz_p, pv, M.gptr, M.e_ch,
                                                         gch_out, M.ngch, M.gunit, tau, mode, qv,
                                                         active);
  if (mode == 1 && M.nheavy > 0) {
    heavy_parts_kernel<<<dim3((unsigned)std::min<int64_t>(M.nhp, 148 * 8), S), kVT, 0, st>>>(
        M.nhp, M.hp_c0, M.hp_c1, gch_out, M.ngch, M.hbuf, active);
    heavy_entries_kernel<<<grid_for(M.nheavy, S), kVT, 0, st>>>(M.nheavy, M.heavy, M.hpart_ptr,
                                                                M.nhp, M.hbuf, M.psrc, M.nnz_p, pv,
                                                                M.nq, qv, active);
  }
}
void vk_spmv_A(const VecModel& M, const double* x, double* eta, const int* active, int S,
               cudaStream_t st) {
  spmv_A_kernel<<<grid_for(M.m, S), kVT, 0, st>>>(M.m, M.ap, M.aj, M.ax, x, M.npad, eta, active);
}
void vk_lik(const VecModel& M, const double* eta, const double* tau, double* d1, double* w,
            double* parts, const int* active, int S, cudaStream_t st) {
  lik_kernel<<<dim3(M.nred, S), kVT, 0, st>>>(M.m, M.family, eta, M.y, M.off, M.logE, M.E,
                                               tau, d1, w, parts, M.nred, active);
}
void vk_take_try(int64_t npad, int64_t m, int S, const int* sel, const double* tx, const double* tqx,
                 const double* teta, const double* td1, const double* tw, double* x, double* qx,
                 double* eta, double* d1, double* w, cudaStream_t st) {
  take_try_kernel<<<grid_for(std::max(npad, m), S), kVT, 0, st>>>(npad, m, S, sel, tx, tqx, teta, td1,
                                                                  tw, x, qx, eta, d1, w);
}
void vk_gdiff(const VecModel& M, const double* eta, const double* eta_t, const double* tau,
              const double* x, const double* x_t, const double* qx, const double* qx_t,
              double* parts, const int* active, int S, cudaStream_t st) {
  gdiff_kernel<<<dim3(M.nred, S), kVT, 0, st>>>(M.m, M.npad, M.family, eta, eta_t, M.y, M.off,
                                                 M.E, tau, x, x_t, qx, qx_t, parts, M.nred,
                                                     active);
}
void vk_AT(const VecModel& M, const double* d1, const double* sub, double* out, double* ch_out,
           const int* active, int S, cudaStream_t st) {
  at_chunk_kernel<<<grid_for(M.nch * 16, S), kVT, 0, st>>>(M.nch, M.ch_row, M.ch_beg, M.at_obs,
                                                            M.at_val, d1, M.m, ch_out, active);
  at_combine_kernel<<<grid_for(M.npad, S), kVT, 0, st>>>(M.npad, M.row_ch, M.nch, ch_out, sub, out,
                                                          active);
  if (M.nheavy_rows > 0)
    at_heavy_rows_kernel<<<dim3((unsigned)std::min<int64_t>(M.nheavy_rows, 148 * 8), S), kVT, 0, st>>>(
        M.nheavy_rows, M.heavy_rows, M.row_ch, M.nch, ch_out, sub, M.npad, out, active);
}
void vk_symv(const VecModel& M, const double* pv, const double* x, double* qx, const int* active,
             int S, cudaStream_t st) {
  symv_kernel<<<grid_for(M.npad, S), kVT, 0, st>>>(M.npad, M.qp, M.qj, M.qvi, pv, M.nnz_p, x, qx,
                                                    active);
}
void vk_dot_max(const VecModel& M, const double* a, const double* b, double* parts,
                const int* active, int S, cudaStream_t st) {
  dot_max_kernel<<<dim3(M.nred, S), kVT, 0, st>>>(M.npad, a, b, parts, M.nred, active);
}
void vk_reduce(const double* parts, int nblk, int wdt, int maxmask, double* out, const int* active,
               int S, cudaStream_t st) {
  reduce_parts_kernel<<<S, 32 * wdt, 0, st>>>(parts, nblk, wdt, maxmask, out, active);
}
void vk_axpy(int64_t npad, const double* x, const double* d, const double* alpha, double* y,
             const int* active, int S, cudaStream_t st) {
  axpy_kernel<<<grid_for(npad, S), kVT, 0, st>>>(npad, x, d, alpha, y, active);
}
void vk_scale(int64_t npad, const double* x, const double* alpha, double* y, const int* active,
              int S, cudaStream_t st) {
  scale_kernel<<<grid_for(npad, S), kVT, 0, st>>>(npad, x, alpha, y, active);
}


// out[i] = src[idx[i]] (idx < 0 -> 0): entries of resident tiles / values
// (drop-in payloads: factor values, Sigma values, Q_c values)
__global__ void gather_kernel(const double* src, const int64_t* idx, int64_t k, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx[i];
    out[i] = j >= 0 ? src[j] : 0.0;
  }
}
void vk_gather(const double* src, const int64_t* idx, int64_t k, double* out, cudaStream_t st) {
  if (k <= 0) return;
  gather_kernel<<<(unsigned)std::min<int64_t>((k + kVT - 1) / kVT, 148 * 8), kVT, 0, st>>>(src, idx, k,
                                                                                           out);
}

// y = L x on the padded permuted layout: one block per tile row I, thread r
// owns row r and sums its row's tiles in row-form order (fixed => deterministic);
// the diagonal tile contributes its lower triangle only
__global__ void tile_lmv_kernel(const double* L, const int* rowptr, const int* row_col,
                                const int* row_tid, const double* x, double* y) {
  const int I = blockIdx.x, r = threadIdx.x;
  double acc = 0.0;
  for (int q = rowptr[I]; q < rowptr[I + 1]; ++q) {
    const int J = row_col[q];
    const double* t = L + (int64_t)row_tid[q] * 4096 + r * 64;
    const double* xj = x + (int64_t)J * 64;
    const int cmax = J == I ? r + 1 : 64;
    for (int c = 0; c < cmax; ++c) acc += t[c] * xj[c];
  }
  y[(int64_t)I * 64 + r] = acc;
}
void vk_tile_lmv(const double* L, int NT, const int* rowptr, const int* row_col, const int* row_tid,
                 const double* x, double* y, cudaStream_t st) {
  if (NT > 0) tile_lmv_kernel<<<NT, 64, 0, st>>>(L, rowptr, row_col, row_tid, x, y);
}

}  // namespace pinla
