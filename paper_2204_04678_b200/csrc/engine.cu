// libpinla engine: one-time analysis + upload, batched f(theta) with the
// inner Newton loop, selected inversion, and the C-ABI of include/pinla.h.
//
// Host orchestration mirrors ObjectiveEvaluator (/root/reference/pkg/src/
// parinla/objective.py:112-331) slot-parallel: every kernel launch covers all
// active theta slots of the batch (the reference runs one theta per thread,
// runtime.py:134-177).  Per-slot decisions of the Newton loop (convergence,
// step halving, flat-floor acceptance) are taken on the host from a handful
// of reduced scalars, with exactly the reference's rules
// (objective.py:259-296).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pinla.h"
#include "analysis.hpp"
#include "ordering.hpp"
#include "dag.cuh"
#include "vec.cuh"

namespace pinla {

static thread_local std::string g_err;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " + \
                               __FILE__ + ":" + std::to_string(__LINE__));             \
  } while (0)

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count, int64_t* acct) {
    free();
    n = count;
    if (count) {
      CK(cudaMalloc(&p, count * sizeof(T)));
      if (acct) *acct += (int64_t)(count * sizeof(T));
    }
  }
  void upload(const std::vector<T>& v, int64_t* acct) {
    alloc(v.size(), acct);
    if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  void zero(cudaStream_t st) {
    if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), st));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { free(); }
};

template <typename T>
static void d2h(T* h, const T* d, size_t n, cudaStream_t st) {
  CK(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, st));
}
template <typename T>
static void h2d(T* d, const T* h, size_t n, cudaStream_t st) {
  CK(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

static const double LOG_2PI = std::log(2.0 * M_PI);

struct Handle {
  // model (host copies)
  int64_t n = 0, m = 0;
  int d = 0, family = 0, noise_theta = -1;
  double noise_precision = 1.0;
  std::vector<double> hyper_shape, hyper_rate;
  std::vector<int> gain_kind, gain_theta, gain_sub;
  std::vector<int> ld_kind, ld_theta;
  std::vector<int64_t> ld_dims;
  std::vector<double> ld_value;
  bool analytic_logdet = false;
  double lgamma_const = 0.0;  // poisson: sum lgamma(y+1)
  int S = 1, Ssel = 1, max_inner = 50;
  double inner_tol = 1e-8;
  int device = 0;
  Analysis an;
  std::vector<int64_t> c_indptr, c_indices;  // conditional pattern, original order (CSC lower)
  std::vector<int64_t> q_newpos;            // CSC entry -> position in tile order
  int64_t nnz_p = 0, nq = 0;
  cudaStream_t st = nullptr;
  int epoch = 0;
  int64_t device_bytes = 0;
  double analyze_s = 0.0;
  // stats
  int64_t n_evals = 0, n_factor = 0, n_solve = 0, n_selinv = 0, launches = 0;
  int64_t factor_slot_runs = 0, solve_slot_runs = 0;
  double last_call_ms = 0;
  std::vector<int> active_h;  // host copy of the active mask
  double t_assemble = 0, t_factor = 0, t_solve = 0, t_selinv = 0, t_other = 0;
  double t_solvek = 0;
  int64_t assemble_slot_runs = 0;  // sum over assembly calls of active slots             // solve_kernel launches only (inside t_solve / t_other)
  int64_t asm_bytes[4] = {0, 0, 0, 0};  // per slot: prior_values, cond_values modes 0/1/2
  int64_t asm_bytes_done = 0;          // sum over assembly launches of active slots x bytes

  // ---- device structure ----
  DBuf<int4> d_ftasks, d_stasks, d_seltasks;
  DBuf<int> d_tile_row, d_tile_col, d_colptr, d_upd_a, d_upd_b, d_qloc, d_rowptr, d_row_tid,
      d_tbsz, d_chunk_tile, d_chunk_flags, d_grp_tile, d_chunk_grp_ptr, d_row_col;
  DBuf<int64_t> d_tstart, d_qptr, d_diagq, d_chunk_rng, d_grp_rng;
  DBuf<double> Gbuf;
  DBuf<FTask> d_frec;
  // solve chain-link tiles (SolveArgs::M); off for shallow (nested-dissection) DAGs
  DBuf<int4> d_sgrp;
  DBuf<int> d_sf_ptr, d_sb_ptr;
  bool links_on = false;
  DBuf<int4> d_links;
  int nlinks = 0;
  DBuf<double> Mlink;
  DBuf<int> d_upd_k;
  // vector model
  DBuf<int64_t> d_term_ptr, d_psrc, d_gptr, d_ap, d_ch_beg, d_row_ch, d_qp, d_qvi, d_gch_beg, d_e_ch,
      d_heavy, d_hpart_ptr, d_hp_c0, d_hp_c1, d_heavy_rows;
  DBuf<double> hbuf;
  DBuf<int64_t> d_gbase;
  DBuf<uint8_t> d_clen;
  DBuf<int32_t> d_cperm;
  DBuf<double> gchbuf;
  DBuf<int> d_term_gain, d_gobs, d_aj, d_ch_row, d_at_obs, d_qj;
  DBuf<double> d_term_coef, d_pconst, d_gcoef, d_gunit, d_ax, d_at_val, d_y, d_off, d_logE, d_E;
  VecModel vm;
  // ---- per-slot workspaces ----
  DBuf<double> L, Linv, Ps, Sg, qv, pv, gains, tau, logparts;
  DBuf<double> x, delta, b, qx, eta, d1, w, parts, red, chbuf, ldsum;
  DBuf<int> status, active, sel, counter, lslot;
  DBuf<unsigned long long> llY, llX, llP;
  DBuf<int> d_f_ndep, d_f_succ_ptr, d_f_succ, d_f_ready0, d_f_prio, d_f_order, qcnt, qctr, act_slots;
  DBuf<int> d_s_pa, d_s_pb, d_s_mode, d_s_chunk_tile, d_s_chunk_flags, d_s_ndep, d_s_succ_ptr,
      d_s_succ, d_s_order, sel_act;
  DBuf<int64_t> d_s_chunk_rng, d_s_grp_rng;
  DBuf<int> d_s_grp_tile, d_s_tile_grp_ptr, d_s_grp_buf, d_s_hot;
  DBuf<double> Gsel;
  DBuf<unsigned long long> qqueue;
  DBuf<int> fq, fclaim, d_s_ready0, d_f_ready0b;
  unsigned qepoch = 0;
  int qcap = 0;
  std::vector<int> pad_of_orig32;
  // phase timers are resolved lazily (no host sync per phase) and the
  // per-slot scalars of the Newton decisions come back through pinned
  // staging, so one host round trip serves a whole Newton iteration
  struct PendingTimer {
    cudaEvent_t a, b;
    double* acc;
  };
  std::vector<cudaEvent_t> ev_pool;
  std::vector<PendingTimer> pending;
  double* hpin = nullptr;  // [kPinPerSlot * S] pinned
  int* hpin_i = nullptr;   // [S] pinned
  double* hpin_x = nullptr;  // [npad] pinned warm-start staging
  // halving tries t = 0..kTries-1 (Poisson): x_try, eta, d1, w, Qp x_try
  // per (try, slot); pinned scalars pp[2S] | xq[3S] | dg[2S] per try
  DBuf<double> tx, teta, td1, tw, tqx, talpha;
  double* hpin_t = nullptr;
  double* hpin_xs = nullptr;  // [S][npad] pinned per-slot warm starts (lazy)
  ~Handle() {
    for (auto& p : pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    if (hpin) cudaFreeHost(hpin);
    if (hpin_i) cudaFreeHost(hpin_i);
    if (hpin_x) cudaFreeHost(hpin_x);
    if (hpin_t) cudaFreeHost(hpin_t);
    if (hpin_xs) cudaFreeHost(hpin_xs);
  }
};
constexpr int kPinPerSlot = 9;  // R[3] | ld[1] | pp[2] | xq[3]
constexpr int kTries = 11;      // halving tries alpha = 2^-t, t = 0..10 (objective.py:276)

// ---------------------------------------------------------------------------
// small device helpers local to the engine

__global__ void rowsum_kernel(const double* v, int64_t cnt, double* out, const int* active) {
  const int s = blockIdx.x;
  if (!active[s]) return;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < cnt; i += 32) acc += v[(int64_t)s * cnt + i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (threadIdx.x == 0) out[s] = acc;
}
// sum_j log L_jj over the diagonal tiles of each active slot (padding rows
// are identity: log 1 = 0), off the DAG chain: kLogParts partial sums per
// slot (fixed-order block reductions), then rowsum_kernel
constexpr int kLogParts = 64;
__global__ void logdiag_part_kernel(const double* L, int64_t nT, int NT, const int* colptr,
                                    double* parts, const int* active) {
  const int s = blockIdx.y;
  if (!active[s]) return;
  __shared__ double red[8];
  double acc = 0.0;
  const double* Ls = L + (int64_t)s * nT * 4096;
  const int64_t total = (int64_t)NT * 64, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int J = (int)(e >> 6), j = (int)(e & 63);
    acc += log(Ls[(int64_t)colptr[J] * 4096 + j * 65]);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    parts[(int64_t)s * kLogParts + blockIdx.x] = t;
  }
}
__global__ void set_int_kernel(int* p, int n, int v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// ---------------------------------------------------------------------------
// gains (host): mirrors model.prior_gains (python) — same formulas

static void compute_gains(const Handle& H, const double* th, double* out) {
  for (size_t g = 0; g < H.gain_kind.size(); ++g) {
    const int k = H.gain_theta[g], sub = H.gain_sub[g];
    auto spde = [&](int b) {
      double tau = std::exp(th[k]);
      double k2 = std::exp(2.0 * th[k + 1]);
      return b == 0 ? tau * k2 * k2 : (b == 1 ? 2.0 * tau * k2 : tau);
    };
    auto ar1 = [&](double lr, int a) {
      double rho = 1.0 / (1.0 + std::exp(-lr));
      double s = 1.0 / (1.0 - rho * rho);
      return a == 0 ? s : (a == 1 ? rho * rho * s : -rho * s);
    };
    switch (H.gain_kind[g]) {
      case PINLA_GAIN_EXP: out[g] = std::exp(th[k]); break;
      case PINLA_GAIN_SPDE: out[g] = spde(sub); break;
      case PINLA_GAIN_AR1: out[g] = std::exp(th[k]) * ar1(th[k + 1], sub); break;
      default: out[g] = ar1(th[k + 2], sub / 3) * spde(sub % 3); break;
    }
  }
}

static double log_prior_hyper(const Handle& H, const double* th) {
  // model.py:285-299: sum a log b + a th - b exp(th) - lgamma(a)
  std::vector<double> t(H.d);
  for (int j = 0; j < H.d; ++j)
    t[j] = H.hyper_shape[j] * std::log(H.hyper_rate[j]) + H.hyper_shape[j] * th[j] -
           H.hyper_rate[j] * std::exp(th[j]);
  for (int j = 0; j < H.d; ++j) t[j] -= std::lgamma(H.hyper_shape[j]);
  // numpy pairwise sum of <8 elements is sequential
  double s = 0.0;
  for (int j = 0; j < H.d; ++j) s += t[j];
  return s;
}

// ---------------------------------------------------------------------------
// create

static void build(Handle& H, const pinla_model* M, const pinla_options* O) {
  auto t0 = std::chrono::steady_clock::now();
  PhaseClock clk;
  H.n = M->n;
  H.m = M->m;
  H.d = M->d;
  H.family = M->family;
  H.noise_theta = M->noise_theta;
  H.noise_precision = M->noise_precision;
  H.hyper_shape.assign(M->hyper_shape, M->hyper_shape + M->d);
  H.hyper_rate.assign(M->hyper_rate, M->hyper_rate + M->d);
  H.gain_kind.assign(M->gain_kind, M->gain_kind + M->n_gains);
  H.gain_theta.assign(M->gain_theta, M->gain_theta + M->n_gains);
  H.gain_sub.assign(M->gain_sub, M->gain_sub + M->n_gains);
  if (M->n_logdet_terms > 0 && O->analytic_prior_logdet) {
    H.analytic_logdet = true;
    H.ld_kind.assign(M->ld_kind, M->ld_kind + M->n_logdet_terms);
    H.ld_theta.assign(M->ld_theta, M->ld_theta + M->n_logdet_terms);
    H.ld_dims.assign(M->ld_dims, M->ld_dims + 3 * M->n_logdet_terms);
    H.ld_value.assign(M->ld_value, M->ld_value + M->n_logdet_terms);
  }
  H.S = std::max(1, O->max_slots);
  H.Ssel = std::min(std::max(1, O->selinv_slots), H.S);
  H.max_inner = O->max_inner > 0 ? O->max_inner : 50;
  H.inner_tol = O->inner_tol > 0 ? O->inner_tol : 1e-8;
  H.device = O->device;
  CK(cudaSetDevice(H.device));
  CK(cudaStreamCreateWithFlags(&H.st, cudaStreamNonBlocking));
  const int64_t n = H.n, m = H.m;
  H.nnz_p = M->p_indptr[n];

  // ---- observation order (internal; nothing obs-indexed leaves the
  // library): rows of A sorted by their lowest permuted latent column outside
  // the dense tail, so the observations that feed one Gram entry (a bilinear
  // cell at one time) and one A^T row are adjacent in memory and the weight /
  // vector gathers of the assembly and SpMV kernels stay within few sectors.
  // PINLA_OBS_SORT=0 keeps the caller's order.
  pinla_model Ms = *M;
  std::vector<int64_t> s_ap, s_aj, s_perm;
  std::vector<double> s_ax, s_y, s_off, s_E;
  if (!(getenv("PINLA_OBS_SORT") && getenv("PINLA_OBS_SORT")[0] == '0') && m > 1) {
    std::vector<int64_t> iperm(n);
    for (int64_t k = 0; k < n; ++k) iperm[M->perm[k]] = k;
    const int64_t nmain = n - M->n_dense;
    std::vector<int64_t> key(m);
    for (int64_t i = 0; i < m; ++i) {
      int64_t kmin = INT64_MAX;
      for (int64_t p = M->a_indptr[i]; p < M->a_indptr[i + 1]; ++p) {
        const int64_t k = iperm[M->a_indices[p]];
        if (k < nmain) kmin = std::min(kmin, k);
      }
      key[i] = kmin;
    }
    s_perm.resize(m);
    std::iota(s_perm.begin(), s_perm.end(), 0);
    std::stable_sort(s_perm.begin(), s_perm.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
    s_ap.assign(m + 1, 0);
    for (int64_t i = 0; i < m; ++i) {
      const int64_t o = s_perm[i];
      s_ap[i + 1] = s_ap[i] + (M->a_indptr[o + 1] - M->a_indptr[o]);
    }
    s_aj.resize(s_ap[m]);
    s_ax.resize(s_ap[m]);
    s_y.resize(m);
    s_off.resize(m);
    s_E.resize(m);
    for (int64_t i = 0; i < m; ++i) {
      const int64_t o = s_perm[i];
      std::copy(M->a_indices + M->a_indptr[o], M->a_indices + M->a_indptr[o + 1], s_aj.begin() + s_ap[i]);
      std::copy(M->a_data + M->a_indptr[o], M->a_data + M->a_indptr[o + 1], s_ax.begin() + s_ap[i]);
      s_y[i] = M->y[o];
      s_off[i] = M->offsets[o];
      s_E[i] = M->exposures[o];
    }
    Ms.a_indptr = s_ap.data();
    Ms.a_indices = s_aj.data();
    Ms.a_data = s_ax.data();
    Ms.y = s_y.data();
    Ms.offsets = s_off.data();
    Ms.exposures = s_E.data();
    M = &Ms;
    clk.mark("build: observation order");
  }

  // ---- the prior pattern must be lower CSC with strictly ascending rows
  for (int64_t c = 0; c < n; ++c)
    for (int64_t p = M->p_indptr[c]; p < M->p_indptr[c + 1]; ++p)
      if (M->p_indices[p] < c || (p > M->p_indptr[c] && M->p_indices[p] <= M->p_indices[p - 1]))
        throw std::runtime_error("prior pattern must be lower CSC with ascending rows");

  // ---- Gram pairs (objective.py:79-101): every unordered pair (a <= b) of a
  // design row contributes coef = A_ia A_ib to entry (max, min).  Pairs are
  // enumerated on the fly (observation ascending), never stored as keys.
  int64_t npairs = 0;
  for (int64_t i = 0; i < m; ++i) {
    int64_t r = M->a_indptr[i + 1] - M->a_indptr[i];
    if (r < 1) throw std::runtime_error("every observation needs at least one design entry");
    npairs += r * (r + 1) / 2;
  }
  // the pairs grouped by column (stable counting sort: observation order is
  // kept inside a column), with their row, coefficient and observation
  // (observation ranges on host threads: per-range column counts, then
  // each range scatters at its own offsets inside every column, so a column
  // keeps observation order exactly as in one serial pass)
  std::vector<int64_t> pcnt(n + 1, 0);
  // (pair scratch left uninitialised: every slot is written by the scatter
  // below, and the first touch happens on the scatter's threads)
  std::unique_ptr<int32_t[]> prow(new int32_t[std::max<int64_t>(npairs, 1)]);
  std::unique_ptr<int32_t[]> pobs(new int32_t[H.family == PINLA_FAMILY_POISSON ? std::max<int64_t>(npairs, 1) : 1]);
  std::unique_ptr<double[]> pcf(new double[std::max<int64_t>(npairs, 1)]);
  {
    const int64_t hw = getenv("PINLA_BUILD_THREADS")
                           ? std::max(1, atoi(getenv("PINLA_BUILD_THREADS")))
                           : (int64_t)std::max(1u, std::thread::hardware_concurrency());
    const int nr = (int)std::max<int64_t>(1, std::min<int64_t>({hw, 16, m / 65536 + 1}));
    std::vector<std::vector<int64_t>> w(nr);
    auto pairs_of = [&](int64_t i0, int64_t i1, auto&& fn) {
      for (int64_t i = i0; i < i1; ++i)
        for (int64_t a = M->a_indptr[i]; a < M->a_indptr[i + 1]; ++a)
          for (int64_t b = a; b < M->a_indptr[i + 1]; ++b) {
            const int64_t ja = M->a_indices[a], jb = M->a_indices[b];
            fn(i, std::max(ja, jb), std::min(ja, jb), M->a_data[a] * M->a_data[b]);
          }
    };
    par_for(nr, [&](int64_t t0, int64_t t1) {
      for (int64_t t = t0; t < t1; ++t) {
        w[t].assign(n, 0);
        pairs_of(m * t / nr, m * (t + 1) / nr, [&](int64_t, int64_t, int64_t c, double) { w[t][c]++; });
      }
    }, 1);
    for (int64_t c = 0; c < n; ++c) {
      int64_t base = pcnt[c];
      for (int t = 0; t < nr; ++t) {
        const int64_t k = w[t][c];
        w[t][c] = base;
        base += k;
      }
      pcnt[c + 1] = base;
    }
    const bool with_obs = H.family == PINLA_FAMILY_POISSON;
    par_for(nr, [&](int64_t t0, int64_t t1) {
      for (int64_t t = t0; t < t1; ++t)
        pairs_of(m * t / nr, m * (t + 1) / nr, [&](int64_t i, int64_t r, int64_t c, double cf) {
          const int64_t q = w[t][c]++;
          prow[q] = (int32_t)r;
          pcf[q] = cf;
          if (with_obs) pobs[q] = (int32_t)i;
        });
    }, 1);
  }
  // conditional pattern = prior pattern U Gram pattern, built column-wise
  // (stamp dedup, small sorts)
  // (columns in parallel: one pass counts each column's union, the second
  // writes and sorts it in place)
  {
    H.c_indptr.assign(n + 1, 0);
    auto column = [&](int64_t c, std::vector<int64_t>& stamp, int64_t* out) -> int64_t {
      int64_t k = 0;
      for (int64_t p = M->p_indptr[c]; p < M->p_indptr[c + 1]; ++p) {
        const int64_t r = M->p_indices[p];
        if (stamp[r] != c) { stamp[r] = c; if (out) out[k] = r; ++k; }
      }
      for (int64_t q = pcnt[c]; q < pcnt[c + 1]; ++q) {
        const int64_t r = prow[q];
        if (stamp[r] != c) { stamp[r] = c; if (out) out[k] = r; ++k; }
      }
      if (stamp[c] != c) { if (out) out[k] = c; ++k; }  // structural diagonal
      if (out) std::sort(out, out + k);
      return k;
    };
    par_for(n, [&](int64_t c0, int64_t c1) {
      std::vector<int64_t> stamp(n, -1);
      for (int64_t c = c0; c < c1; ++c) H.c_indptr[c + 1] = column(c, stamp, nullptr);
    }, 1 << 14);
    for (int64_t c = 0; c < n; ++c) H.c_indptr[c + 1] += H.c_indptr[c];
    H.c_indices.resize(H.c_indptr[n]);
    par_for(n, [&](int64_t c0, int64_t c1) {
      std::vector<int64_t> stamp(n, -1);
      for (int64_t c = c0; c < c1; ++c) column(c, stamp, H.c_indices.data() + H.c_indptr[c]);
    }, 1 << 14);
  }
  H.nq = (int64_t)H.c_indices.size();
  for (int64_t c = 0; c < n; ++c)
    if (H.c_indptr[c + 1] == H.c_indptr[c] || H.c_indices[H.c_indptr[c]] != c)
      throw std::runtime_error("conditional pattern lacks a diagonal entry");

  clk.mark("build: conditional pattern");
  // ---- tile analysis
  int gcap = 0;  // solve product group cap: 0 = by DAG shape (PINLA_SOLVE_GROUP=1: one task per tile)
  if (const char* e = getenv("PINLA_SOLVE_GROUP")) gcap = std::max(0, atoi(e));
  int nlk = -1;  // fused chain links: -1 = by DAG shape (PINLA_SOLVE_LINKS=0/1/2)
  if (const char* e = getenv("PINLA_SOLVE_LINKS")) nlk = std::max(0, std::min(2, atoi(e)));
  int lane = -1;  // factor critical lane: -1 = when chain-bound (PINLA_FACTOR_LANE=0/1)
  if (const char* e = getenv("PINLA_FACTOR_LANE")) lane = atoi(e) != 0 ? 1 : 0;
  analyze_tiles(H.an, n, H.c_indptr.data(), H.c_indices.data(), M->perm, M->n_dense,
                M->tile_bounds, M->n_tile_bounds, std::max(1, 296 / std::max(1, O->max_slots)), gcap,
                nlk, lane);
  Analysis& A = H.an;
  const int64_t npad = A.npad();

  clk.mark("build: analyze_tiles");
  // The side tables that only need the padded row map (prior terms, design
  // transpose, prior symmetric CSR, likelihood data) are built on three host
  // threads while this one orders the conditional entries and the Gram
  // segments (joined before the uploads).
  std::vector<int64_t> term_ptr;
  std::vector<int> term_gain;
  std::vector<double> term_coef, pconst;
  std::vector<int64_t> ap;
  int64_t nnzA = 0;
  std::vector<int> aj;
  std::vector<double> ax;
  std::vector<int64_t> rcnt;
  std::vector<int> at_obs;
  std::vector<double> at_val;
  const int64_t kCh = 256;
  std::vector<int> ch_row;
  std::vector<int64_t> ch_beg, row_ch;
  std::vector<int64_t> qp;
  std::vector<int> qj;
  std::vector<int64_t> qvi_s;
  std::vector<double> y, off, E, logE;
  auto side_prior_terms_and_lik = [&]() {
  // ---- prior terms CSR by entry
  term_ptr.assign(H.nnz_p + 1, 0);
  for (int64_t t = 0; t < M->n_terms; ++t) term_ptr[M->term_entry[t] + 1]++;
  for (int64_t e = 0; e < H.nnz_p; ++e) term_ptr[e + 1] += term_ptr[e];
  term_gain.assign(M->term_gain, M->term_gain + M->n_terms);
  term_coef.assign(M->term_coef, M->term_coef + M->n_terms);
  pconst.assign(M->p_const, M->p_const + H.nnz_p);

  // ---- likelihood data
  y.assign(M->y, M->y + m);
  off.assign(M->offsets, M->offsets + m);
  E.assign(M->exposures, M->exposures + m);
  logE.resize(m);
  for (int64_t i = 0; i < m; ++i) logE[i] = std::log(E[i]);
  if (H.family == PINLA_FAMILY_POISSON) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += std::lgamma(y[i] + 1.0);
    H.lgamma_const = s;
  }

  };
  auto side_design_transpose = [&]() {
  // ---- design (padded columns) and chunked transpose
  ap.assign(M->a_indptr, M->a_indptr + m + 1);
  nnzA = ap[m];
  aj.resize(nnzA);
  ax.assign(M->a_data, M->a_data + nnzA);
  for (int64_t p = 0; p < nnzA; ++p) aj[p] = (int)A.pad_of_orig[M->a_indices[p]];
  rcnt.assign(npad + 1, 0);
  for (int64_t p = 0; p < nnzA; ++p) rcnt[aj[p] + 1]++;
  for (int64_t r = 0; r < npad; ++r) rcnt[r + 1] += rcnt[r];
  at_obs.resize(nnzA);
  at_val.resize(nnzA);
  {
    std::vector<int64_t> wpos(rcnt.begin(), rcnt.end() - 1);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t p = ap[i]; p < ap[i + 1]; ++p) {
        int64_t q = wpos[aj[p]]++;
        at_obs[q] = (int)i;
        at_val[q] = ax[p];
      }
  }
  row_ch.assign(npad + 1, 0);
  for (int64_t r = 0; r < npad; ++r) {
    for (int64_t s = rcnt[r]; s < rcnt[r + 1]; s += kCh) {
      ch_row.push_back((int)r);
      ch_beg.push_back(s);
    }
    row_ch[r + 1] = (int64_t)ch_row.size();
  }
  ch_beg.push_back(nnzA);

  };
  auto side_prior_csr = [&]() {
  // ---- prior symmetric CSR on padded rows: counting sort by row, then a
  // small sort by column inside each row
  qp.assign(npad + 1, 0);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t p = M->p_indptr[c]; p < M->p_indptr[c + 1]; ++p) {
      const int64_t r = M->p_indices[p];
      qp[A.pad_of_orig[r] + 1]++;
      if (r != c) qp[A.pad_of_orig[c] + 1]++;
    }
  for (int64_t r = 0; r < npad; ++r) qp[r + 1] += qp[r];
  qj.resize(qp[npad]);
  qvi_s.resize(qp[npad]);
  {
    std::vector<int64_t> w(qp.begin(), qp.end() - 1);
    for (int64_t c = 0; c < n; ++c)
      for (int64_t p = M->p_indptr[c]; p < M->p_indptr[c + 1]; ++p) {
        const int64_t r = M->p_indices[p];
        const int64_t pr = A.pad_of_orig[r], pc = A.pad_of_orig[c];
        int64_t q = w[pr]++;
        qj[q] = (int)pc;
        qvi_s[q] = p;
        if (r != c) {
          q = w[pc]++;
          qj[q] = (int)pr;
          qvi_s[q] = p;
        }
      }
    std::vector<std::pair<int, int64_t>> tmp;
    for (int64_t r = 0; r < npad; ++r) {
      const int64_t b0 = qp[r], b1 = qp[r + 1];
      if (b1 - b0 < 2) continue;
      tmp.clear();
      for (int64_t q = b0; q < b1; ++q) tmp.push_back({qj[q], qvi_s[q]});
      std::sort(tmp.begin(), tmp.end());
      for (int64_t q = b0; q < b1; ++q) {
        qj[q] = tmp[q - b0].first;
        qvi_s[q] = tmp[q - b0].second;
      }
    }
  }
  };
  std::exception_ptr side_err[3];
  std::thread side[3];
  side[0] = std::thread([&] {
    try {
      side_prior_terms_and_lik();
    } catch (...) {
      side_err[0] = std::current_exception();
    }
  });
  side[1] = std::thread([&] {
    try {
      side_design_transpose();
    } catch (...) {
      side_err[1] = std::current_exception();
    }
  });
  side[2] = std::thread([&] {
    try {
      side_prior_csr();
    } catch (...) {
      side_err[2] = std::current_exception();
    }
  });
  struct JoinAll {  // an exception below still joins the side threads
    std::thread* t;
    ~JoinAll() {
      for (int i = 0; i < 3; ++i)
        if (t[i].joinable()) t[i].join();
    }
  } join_side{side};
  // ---- conditional entries in tile order
  std::vector<int64_t> etid(H.nq), eloc(H.nq);
  par_for(n, [&](int64_t c0, int64_t c1) {
  for (int64_t c = c0; c < c1; ++c)
    for (int64_t p = H.c_indptr[c]; p < H.c_indptr[c + 1]; ++p) {
      int64_t r = H.c_indices[p];
      int64_t pr = A.iperm[r], pc = A.iperm[c];
      int64_t R = std::max(pr, pc), Cc = std::min(pr, pc);
      int64_t PR = A.pad_of_perm(R), PC = A.pad_of_perm(Cc);
      int32_t TI = (int32_t)(PR / TB), TJ = (int32_t)(PC / TB);
      int64_t tid = A.tid_of(TI, TJ);
      if (tid < 0) throw std::runtime_error("entry outside the tile pattern");
      etid[p] = tid;
      eloc[p] = (PR % TB) * TB + (PC % TB);
    }
  });
  // tile order = (tile id, position in tile): counting sort by tile, then a
  // small sort by position inside each tile (entries of a tile are few)
  std::vector<int64_t> qptr(A.nT + 1, 0);
  for (int64_t p = 0; p < H.nq; ++p) qptr[etid[p] + 1]++;
  for (int64_t t = 0; t < A.nT; ++t) qptr[t + 1] += qptr[t];
  std::vector<int64_t> order(H.nq);
  {
    std::vector<int64_t> w(qptr.begin(), qptr.end() - 1);
    for (int64_t p = 0; p < H.nq; ++p) order[w[etid[p]]++] = p;
    par_for(A.nT, [&](int64_t t0, int64_t t1) {
      for (int64_t t = t0; t < t1; ++t)
        std::sort(order.begin() + qptr[t], order.begin() + qptr[t + 1],
                  [&](int64_t x, int64_t y) { return eloc[x] < eloc[y]; });
    }, 1024);
  }
  std::vector<int64_t>& newpos = H.q_newpos;  // CSC position -> tile order (kept: payloads)
  newpos.resize(H.nq);
  for (int64_t i = 0; i < H.nq; ++i) newpos[order[i]] = i;
  // prior entry of every conditional entry: both patterns are sorted lower
  // CSC, so one merge walk per column
  std::vector<int64_t> psrc_orig(H.nq, -1);
  par_for(n, [&](int64_t c0, int64_t c1) {
  for (int64_t c = c0; c < c1; ++c) {
    int64_t pp = M->p_indptr[c];
    const int64_t pe = M->p_indptr[c + 1];
    for (int64_t q = H.c_indptr[c]; q < H.c_indptr[c + 1]; ++q) {
      const int64_t r = H.c_indices[q];
      while (pp < pe && M->p_indices[pp] < r) ++pp;
      if (pp < pe && M->p_indices[pp] == r) psrc_orig[q] = pp;
    }
  }
  });
  std::vector<int> qloc(H.nq);
  std::vector<int64_t> psrc(H.nq), diagq(npad, -1);
  par_for(H.nq, [&](int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      const int64_t e = order[i];
      qloc[i] = (int)eloc[e];
      psrc[i] = psrc_orig[e];
    }
  });
  for (int64_t c = 0; c < n; ++c) diagq[A.pad_of_orig[c]] = newpos[H.c_indptr[c]];  // diagonal first
  clk.mark("build: entries in tile order");
  // ---- Gram segments by (tile-order entry, obs): the destination of each
  // pair through a per-column row -> entry map, then a stable counting sort
  // by destination (pair order = observation order, the reference's bincount
  // order, objective.py:140-145).  Gaussian models only need the unit sums.
  std::vector<int64_t> gptr(H.nq + 1, 0);
  std::vector<double> gunit(H.nq, 0.0);
  std::unique_ptr<int[]> gobs_s;
  std::unique_ptr<double[]> gcoef_s;
  std::unique_ptr<int64_t[]> pdst(new int64_t[std::max<int64_t>(npairs, 1)]);
  // (a destination entry lies in one column: columns run in parallel, the
  // pairs of a column in observation order)
  par_for(n, [&](int64_t c0, int64_t c1) {
    std::vector<int64_t> slot(n, -1);
    for (int64_t c = c0; c < c1; ++c) {
      for (int64_t q = H.c_indptr[c]; q < H.c_indptr[c + 1]; ++q) slot[H.c_indices[q]] = q;
      for (int64_t k = pcnt[c]; k < pcnt[c + 1]; ++k) {
        const int64_t d = newpos[slot[prow[k]]];
        pdst[k] = d;
        gptr[d + 1]++;
        gunit[d] += pcf[k];
      }
    }
  }, 1 << 15);
  for (int64_t e = 0; e < H.nq; ++e) gptr[e + 1] += gptr[e];
  if (H.family == PINLA_FAMILY_POISSON) {
    gobs_s.reset(new int[std::max<int64_t>(npairs, 1)]);
    gcoef_s.reset(new double[std::max<int64_t>(npairs, 1)]);
    std::vector<int64_t> w(gptr.begin(), gptr.end() - 1);
    par_for(n, [&](int64_t c0, int64_t c1) {
      for (int64_t k = pcnt[c0]; k < pcnt[c1]; ++k) {
        const int64_t q = w[pdst[k]]++;
        gobs_s[q] = pobs[k];
        gcoef_s[q] = pcf[k];
      }
    }, 1 << 15);
  }
  pdst.reset();
  prow.reset();
  pobs.reset();
  pcf.reset();
  clk.mark("build: Gram segments");
  // chunks of <= kGramChunk pairs inside each entry (two-level segmented sum)
  std::vector<int64_t> gch_beg, e_ch(H.nq + 1, 0);
  for (int64_t e = 0; e < H.nq; ++e) {
    for (int64_t q = gptr[e]; q < gptr[e + 1]; q += kGramChunk) gch_beg.push_back(q);
    e_ch[e + 1] = (int64_t)gch_beg.size();
  }
  gch_beg.push_back(npairs);

  for (auto& t : side) t.join();
  for (auto& e : side_err)
    if (e) std::rethrow_exception(e);
  clk.mark("build: side tables (joined)");
  // ---- uploads
  int64_t* acct = &H.device_bytes;
  auto tasks_up = [&](DBuf<int4>& d, const std::vector<TileTask>& v) {
    std::vector<int4> t(v.size());
    for (size_t i = 0; i < v.size(); ++i) t[i] = make_int4(v[i].type, 0, v[i].id, v[i].level);
    d.upload(t, acct);
  };
  tasks_up(H.d_ftasks, A.factor_tasks);
  tasks_up(H.d_stasks, A.solve_tasks);
  tasks_up(H.d_seltasks, A.selinv_tasks);
  H.d_tile_row.upload(A.tile_row, acct);
  H.d_tile_col.upload(A.tile_col, acct);
  H.d_colptr.upload(A.colptr, acct);
  H.d_rowptr.upload(A.rowptr, acct);
  H.d_row_col.upload(A.row_col, acct);
  {
    std::vector<int4> g(std::max(A.n_sgrp, 1));
    for (int32_t i = 0; i < A.n_sgrp; ++i) g[i] = make_int4(A.sg_lo[i], A.sg_hi[i], A.sg_line[i], 0);
    H.d_sgrp.upload(g, acct);
    H.d_sf_ptr.upload(A.sf_ptr, acct);
    H.d_sb_ptr.upload(A.sb_ptr, acct);
  }
  {
    // chain-link tiles (Analysis::solve_links, SolveArgs::M): the newest one
    // or two products of each row / column for long tile-row chains
    H.links_on = A.solve_links > 0;
    std::vector<int4> lk;
    for (int32_t I = 0; I < A.NT && H.links_on; ++I) {
      const int32_t q1 = A.rowptr[I + 1] - 1, q0 = A.rowptr[I];
      for (int k = 0; k < A.solve_links && q1 - 1 - k >= q0; ++k)
        lk.push_back(make_int4(k, I, A.row_tid[q1 - 1 - k], A.row_col[q1 - 1 - k]));
    }
    for (int32_t J = 0; J < A.NT && H.links_on; ++J) {
      const int32_t q0 = A.colptr[J] + 1, q1 = A.colptr[J + 1];
      for (int k = 0; k < A.solve_links && q0 + k < q1; ++k)
        lk.push_back(make_int4(2 + k, J, q0 + k, A.tile_row[q0 + k]));
    }
    H.nlinks = (int)lk.size();
    H.d_links.upload(lk, acct);
  }
  H.d_f_ndep.upload(A.f_ndep, acct);
  H.d_f_succ_ptr.upload(A.f_succ_ptr, acct);
  H.d_f_succ.upload(A.f_succ.empty() ? std::vector<int>{0} : A.f_succ, acct);
  H.d_f_ready0.upload(A.f_ready0, acct);
  H.d_f_prio.upload(A.f_prio, acct);
  H.d_f_order.upload(A.f_order, acct);
  auto nz = [](const std::vector<int>& v) { return v.empty() ? std::vector<int>{0} : v; };
  H.d_s_pa.upload(nz(A.s_pa), acct);
  H.d_s_pb.upload(nz(A.s_pb), acct);
  H.d_s_mode.upload(nz(A.s_mode), acct);
  H.d_s_chunk_rng.upload(A.s_chunk_rng, acct);
  H.d_s_chunk_tile.upload(A.s_chunk_tile, acct);
  H.d_s_chunk_flags.upload(A.s_chunk_flags, acct);
  H.d_s_ndep.upload(A.s_ndep, acct);
  H.d_s_succ_ptr.upload(A.s_succ_ptr, acct);
  H.d_s_succ.upload(nz(A.s_succ), acct);
  H.d_s_order.upload(A.s_order, acct);
  H.d_s_ready0.upload(nz(A.s_ready0), acct);
  H.d_s_grp_rng.upload(A.s_grp_rng, acct);
  H.d_s_grp_tile.upload(nz(A.s_grp_tile), acct);
  H.d_s_grp_buf.upload(nz(A.s_grp_buf), acct);
  H.d_s_hot.upload(nz(A.s_hot), acct);
  H.d_s_tile_grp_ptr.upload(A.s_tile_grp_ptr, acct);
  {
    std::vector<int> tb(A.NT);
    for (int32_t t = 0; t < A.NT; ++t) tb[t] = (int)(A.tstart[t + 1] - A.tstart[t]);
    H.d_tbsz.upload(tb, acct);
  }
  H.d_row_tid.upload(A.row_tid, acct);
  H.d_tstart.upload(A.tstart, acct);
  H.d_upd_a.upload(A.upd_a.empty() ? std::vector<int>{0} : A.upd_a, acct);
  H.d_upd_b.upload(A.upd_b.empty() ? std::vector<int>{0} : A.upd_b, acct);
  H.d_chunk_rng.upload(A.chunk_rng, acct);
  H.d_chunk_tile.upload(A.chunk_tile, acct);
  H.d_chunk_flags.upload(A.chunk_flags, acct);
  H.d_grp_rng.upload(A.grp_rng, acct);
  H.d_grp_tile.upload(A.grp_tile.empty() ? std::vector<int>{0} : A.grp_tile, acct);
  H.d_chunk_grp_ptr.upload(A.chunk_grp_ptr, acct);
  H.d_qptr.upload(qptr, acct);
  {
    // factor task records (dag.cuh FTask) and per-pair K extents
    std::vector<int> tbh(A.NT);
    for (int32_t t = 0; t < A.NT; ++t) tbh[t] = (int)(A.tstart[t + 1] - A.tstart[t]);
    std::vector<FTask> rec(A.factor_tasks.size());
    par_for((int64_t)rec.size(), [&](int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      const TileTask& tt = A.factor_tasks[i];
      FTask& r = rec[i];
      std::memset(&r, 0, sizeof(r));
      r.type = tt.type;
      r.id = tt.id;
      if (tt.type == 1) {
        r.tid = A.grp_tile[tt.id];
        r.u0 = A.grp_rng[tt.id];
        r.u1 = A.grp_rng[tt.id + 1];
      } else {
        r.tid = A.chunk_tile[tt.id];
        r.flags = A.chunk_flags[tt.id];
        r.u0 = A.chunk_rng[tt.id];
        r.u1 = A.chunk_rng[tt.id + 1];
        r.g0 = A.chunk_grp_ptr[tt.id];
        r.g1 = A.chunk_grp_ptr[tt.id + 1];
      }
      r.I = A.tile_row[r.tid];
      r.J = A.tile_col[r.tid];
      r.mI = tbh[r.I];
      r.nJ = tbh[r.J];
      r.q0 = qptr[r.tid];
      r.q1 = qptr[r.tid + 1];
      r.succ0 = A.f_succ_ptr[i];
      r.succ1 = A.f_succ_ptr[i + 1];
      r.pa0 = r.u1 > r.u0 ? A.upd_a[r.u0] : -1;
      r.pb0 = r.u1 > r.u0 ? A.upd_b[r.u0] : -1;
      r.k0 = r.u1 > r.u0 ? tbh[A.tile_col[A.upd_a[r.u0]]] : 0;
      // continuation target (factor_ws.cu): an inner chunk's single successor is the next chunk
      // of its tile; lane tasks are claimed only by the lane CTAs
      r.next = -1;
      if (tt.type == 0 && !(r.flags & 2) && r.succ1 - r.succ0 == 1) {
        const int32_t t2 = A.f_succ[r.succ0];
        const TileTask& n2 = A.factor_tasks[t2];
        const bool lane2 = A.f_nlane > 0 && t2 >= (int64_t)A.factor_tasks.size() - A.f_nlane;
        if (n2.type == 0 && A.chunk_tile[n2.id] == r.tid && !(A.chunk_flags[n2.id] & 1) && !lane2) r.next = t2;
      }
    }
    });
    H.d_frec.upload(rec, acct);
    std::vector<int> uk(std::max<size_t>(A.upd_a.size(), 1), 0);
    par_for((int64_t)A.upd_a.size(), [&](int64_t u0, int64_t u1) {
      for (int64_t u = u0; u < u1; ++u) uk[u] = tbh[A.tile_col[A.upd_a[u]]];
    }, 1 << 16);
    H.d_upd_k.upload(uk, acct);
  }
  clk.mark("build: uploads (DAG tables)");
  H.d_qloc.upload(qloc, acct);
  H.d_diagq.upload(diagq, acct);
  H.d_term_ptr.upload(term_ptr, acct);
  H.d_term_gain.upload(term_gain, acct);
  H.d_term_coef.upload(term_coef, acct);
  H.d_pconst.upload(pconst, acct);
  H.d_psrc.upload(psrc, acct);
  H.d_gptr.upload(gptr, acct);
  if (H.family == PINLA_FAMILY_POISSON) {
    // Gram pairs for gram_chunk_kernel: chunks ordered by length (counting
    // sort, longest first), 32 per group; pair k of the chunk at position
    // 32 g + l lives at gbase[g] + 32 k + l, so a warp's pair loads are
    // coalesced and padding stays within groups of equal-length chunks.
    // The per-chunk sum order is unchanged (k ascending).
    {
      const int64_t ngc = (int64_t)gch_beg.size() - 1;
      // (one counting pass: lengths kGramChunk..1 in turn, chunk order
      // kept inside a length)
      int64_t lcnt[kGramChunk + 2] = {0};
      for (int64_t c = 0; c < ngc; ++c) lcnt[gch_beg[c + 1] - gch_beg[c]]++;
      int64_t lpos[kGramChunk + 2] = {0};
      int64_t at = 0;
      for (int64_t len = kGramChunk; len >= 1; --len) {
        lpos[len] = at;
        at += lcnt[len];
      }
      std::vector<int32_t> order(at);
      for (int64_t c = 0; c < ngc; ++c) {
        const int64_t len = gch_beg[c + 1] - gch_beg[c];
        if (len >= 1) order[lpos[len]++] = (int32_t)c;
      }
      const int64_t npos = (ngc + 31) / 32 * 32, ng = npos / 32;
      std::vector<int64_t> gbase(ng + 1, 0);
      std::vector<uint8_t> clen(npos, 0);
      std::vector<int32_t> cperm(npos, -1);
      for (int64_t p = 0; p < (int64_t)order.size(); ++p) {
        cperm[p] = order[p];
        clen[p] = (uint8_t)(gch_beg[order[p] + 1] - gch_beg[order[p]]);
      }
      for (int64_t g = 0; g < ng; ++g) gbase[g + 1] = gbase[g] + 32 * (int64_t)clen[32 * g];
      std::vector<int> gobs2(std::max<int64_t>(gbase[ng], 1), 0);
      std::vector<double> gcoef2(std::max<int64_t>(gbase[ng], 1), 0.0);
      par_for((int64_t)order.size(), [&](int64_t p0, int64_t p1) {
        for (int64_t p = p0; p < p1; ++p) {
          const int64_t q0 = gch_beg[order[p]], b = gbase[p >> 5] + (p & 31);
          for (int k = 0; k < clen[p]; ++k) {
            gobs2[b + 32 * k] = gobs_s[q0 + k];
            gcoef2[b + 32 * k] = gcoef_s[q0 + k];
          }
        }
      }, 1 << 16);
      H.d_gobs.upload(gobs2, acct);
      H.d_gcoef.upload(gcoef2, acct);
      H.d_gbase.upload(gbase, acct);
      H.d_clen.upload(clen, acct);
      H.d_cperm.upload(cperm, acct);
      H.vm.gpos = npos;
    }
    clk.mark("build: uploads (Gram layout)");
    H.d_gch_beg.upload(gch_beg, acct);
    H.d_e_ch.upload(e_ch, acct);
    std::vector<int64_t> heavy, hpp{0}, hc0, hc1;
    for (int64_t e = 0; e < H.nq; ++e)
      if (e_ch[e + 1] - e_ch[e] > kHeavyChunks) {
        heavy.push_back(e);
        for (int64_t c = e_ch[e]; c < e_ch[e + 1]; c += kHeavyPart) {
          hc0.push_back(c);
          hc1.push_back(std::min(c + kHeavyPart, e_ch[e + 1]));
        }
        hpp.push_back((int64_t)hc0.size());
      }
    H.d_heavy.upload(heavy.empty() ? std::vector<int64_t>{0} : heavy, acct);
    H.vm.nheavy = (int64_t)heavy.size();
    H.d_hpart_ptr.upload(hpp, acct);
    H.d_hp_c0.upload(hc0.empty() ? std::vector<int64_t>{0} : hc0, acct);
    H.d_hp_c1.upload(hc1.empty() ? std::vector<int64_t>{0} : hc1, acct);
    H.vm.nhp = (int64_t)hc0.size();
  }
  const int64_t ngch = (int64_t)gch_beg.size() - 1;
  H.d_gunit.upload(gunit, acct);
  H.d_ap.upload(ap, acct);
  H.d_aj.upload(aj, acct);
  H.d_ax.upload(ax, acct);
  H.d_ch_row.upload(ch_row, acct);
  H.d_ch_beg.upload(ch_beg, acct);
  H.d_at_obs.upload(at_obs, acct);
  H.d_at_val.upload(at_val, acct);
  H.d_row_ch.upload(row_ch, acct);
  {
    std::vector<int64_t> hr;
    for (int64_t r = 0; r < npad; ++r)
      if (row_ch[r + 1] - row_ch[r] > kHeavyChunks) hr.push_back(r);
    H.vm.nheavy_rows = (int64_t)hr.size();
    H.d_heavy_rows.upload(hr.empty() ? std::vector<int64_t>{0} : hr, acct);
  }
  H.d_y.upload(y, acct);
  H.d_off.upload(off, acct);
  H.d_E.upload(E, acct);
  H.d_logE.upload(logE, acct);
  H.d_qp.upload(qp, acct);
  H.d_qj.upload(qj, acct);
  H.d_qvi.upload(qvi_s, acct);

  VecModel& V = H.vm;
  V.nred = (int)std::min<int64_t>(kRedBlocks, std::max<int64_t>(296, (std::max(m, npad) + 4095) / 4096));
  V.m = m;
  V.npad = npad;
  V.nnz_p = H.nnz_p;
  V.nq = H.nq;
  V.nch = (int64_t)ch_row.size();
  V.family = H.family;
  V.n_gains = (int)H.gain_kind.size();
  V.term_ptr = H.d_term_ptr.p;
  V.term_gain = H.d_term_gain.p;
  V.term_coef = H.d_term_coef.p;
  V.pconst = H.d_pconst.p;
  V.psrc = H.d_psrc.p;
  V.gptr = H.d_gptr.p;
  V.gobs = H.d_gobs.p;
  V.gbase = H.d_gbase.p;
  V.clen = H.d_clen.p;
  V.cperm = H.d_cperm.p;
  V.gcoef = H.d_gcoef.p;
  V.gunit = H.d_gunit.p;
  V.ngch = H.family == PINLA_FAMILY_POISSON ? ngch : 0;
  V.gch_beg = H.d_gch_beg.p;
  V.e_ch = H.d_e_ch.p;
  V.heavy = H.d_heavy.p;
  V.hpart_ptr = H.d_hpart_ptr.p;
  V.hp_c0 = H.d_hp_c0.p;
  V.hp_c1 = H.d_hp_c1.p;
  V.heavy_rows = H.d_heavy_rows.p;
  // algorithmic bytes of the assembly kernels per slot, every index /
  // coefficient / value streamed once: prior_values; cond_values mode 0
  // (gaussian, tau * unit Gram), mode 1 (poisson: Gram chunk sums of
  // w[obs] * coef + their per-entry sums), mode 2 (prior only)
  {
    const int64_t nt = (int64_t)H.d_term_coef.n;
    H.asm_bytes[0] = H.nnz_p * (8 + 8 + 8) + nt * (8 + 4);
    H.asm_bytes[1] = H.nq * (8 + 8 + 8 + 8 + 8);
    H.asm_bytes[2] = (int64_t)H.d_gcoef.n * (4 + 8 + 8) + V.gpos + 2 * (int64_t)V.ngch * (4 + 8) +
                     H.nq * (8 + 8 + 8 + 8);
    H.asm_bytes[3] = H.nq * (8 + 8 + 8);
  }
  V.ap = H.d_ap.p;
  V.aj = H.d_aj.p;
  V.ax = H.d_ax.p;
  V.ch_row = H.d_ch_row.p;
  V.ch_beg = H.d_ch_beg.p;
  V.at_obs = H.d_at_obs.p;
  V.at_val = H.d_at_val.p;
  V.row_ch = H.d_row_ch.p;
  V.y = H.d_y.p;
  V.off = H.d_off.p;
  V.logE = H.d_logE.p;
  V.E = H.d_E.p;
  V.qp = H.d_qp.p;
  V.qj = H.d_qj.p;
  V.qvi = H.d_qvi.p;

  clk.mark("build: uploads (rest)");
  // ---- per-slot workspaces: as many of the requested slots as device
  // memory holds (tile factors dominate: c5 ~20 GB per slot), keeping 8 %
  // headroom; selected-inversion storage comes first
  {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const double tb = (double)TB * TB * 8.0;
    const double per_slot =
        ((double)A.nT + (double)A.NT * (1 + (H.links_on ? 4 : 0)) + std::max(A.ngrp, 1)) * tb +
        8.0 * ((double)npad * 5 + (double)m * 3 + (double)H.nq + (double)H.nnz_p +
               (double)std::max<int64_t>(V.ngch, 1) + (double)std::max<int64_t>(V.nch, 1)) +
        8.0 * 2 * TB * ((double)A.NT * 2 + std::max(A.n_sgrp, 1)) +
        (H.family != PINLA_FAMILY_GAUSSIAN ? 8.0 * kTries * (2.0 * npad + 3.0 * m) : 0.0) +
        4.0 * 2 * std::max<size_t>({A.factor_tasks.size(), A.solve_tasks.size(), A.selinv_tasks.size()});
    const double sel = (double)H.Ssel * ((double)A.nT + std::max(A.s_ngbuf, 1)) * tb;
    const double budget = 0.92 * (double)fr - sel - 512.0 * (1 << 20);
    const int fit = budget > per_slot ? (int)std::min<double>(budget / per_slot, 1 << 20) : 1;
    if (fit < H.S) {
      H.S = std::max(1, fit);
      H.Ssel = std::min(H.Ssel, H.S);
    }
  }
  const int S = H.S;
  const size_t TE = (size_t)TB * TB;
  H.L.alloc((size_t)S * A.nT * TE, acct);
  H.Linv.alloc((size_t)S * A.NT * TE, acct);
  if (H.links_on) H.Mlink.alloc((size_t)S * 4 * A.NT * TE, acct);
  H.Gbuf.alloc((size_t)S * std::max(A.ngrp, 1) * TE, acct);
  H.Sg.alloc((size_t)H.Ssel * A.nT * TE, acct);
  H.Gsel.alloc((size_t)H.Ssel * std::max(A.s_ngbuf, 1) * TE, acct);
  H.qv.alloc((size_t)S * H.nq, acct);
  H.pv.alloc((size_t)S * H.nnz_p, acct);
  H.gains.alloc((size_t)S * std::max<size_t>(H.gain_kind.size(), 1), acct);
  H.tau.alloc(S, acct);
  for (DBuf<double>* v : {&H.x, &H.delta, &H.b, &H.qx}) v->alloc((size_t)S * npad, acct);
  for (DBuf<double>* v : {&H.eta, &H.d1, &H.w}) v->alloc((size_t)S * m, acct);
  H.parts.alloc((size_t)S * kRedBlocks * 3, acct);
  H.red.alloc((size_t)S * 3, acct);
  CK(cudaMallocHost(&H.hpin, sizeof(double) * kPinPerSlot * S));
  CK(cudaMallocHost(&H.hpin_i, sizeof(int) * S));
  CK(cudaMallocHost(&H.hpin_x, sizeof(double) * npad));
  if (H.family != PINLA_FAMILY_GAUSSIAN) {
    for (DBuf<double>* v : {&H.tx, &H.tqx}) v->alloc((size_t)kTries * S * npad, acct);
    for (DBuf<double>* v : {&H.teta, &H.td1, &H.tw}) v->alloc((size_t)kTries * S * m, acct);
    std::vector<double> ta((size_t)kTries * S);
    for (int t = 0; t < kTries; ++t)
      for (int s2 = 0; s2 < S; ++s2) ta[(size_t)t * S + s2] = std::ldexp(1.0, -t);
    H.talpha.upload(ta, acct);
    CK(cudaMallocHost(&H.hpin_t, sizeof(double) * 7 * kTries * S));
  }
  H.ldsum.alloc(S, acct);
  H.logparts.alloc((size_t)S * kLogParts, acct);
  H.chbuf.alloc((size_t)S * std::max<int64_t>(V.nch, 1), acct);
  H.gchbuf.alloc((size_t)S * std::max<int64_t>(V.ngch, 1), acct);
  H.hbuf.alloc((size_t)S * std::max<int64_t>(H.vm.nhp, 1), acct);
  H.vm.hbuf = H.hbuf.p;
  H.llY.alloc((size_t)S * A.NT * 2 * TB, acct);
  H.llX.alloc((size_t)S * A.NT * 2 * TB, acct);
  H.llP.alloc((size_t)S * std::max(A.n_sgrp, 1) * 2 * TB, acct);
  H.llY.zero(H.st);
  H.llX.zero(H.st);
  H.llP.zero(H.st);
  H.status.alloc(S, acct);
  H.active.alloc(S, acct);
  H.sel.alloc(S, acct);
  H.counter.alloc(1, acct);
  {
    size_t qn = (size_t)S * std::max<size_t>({A.factor_tasks.size(), A.solve_tasks.size(),
                                                A.selinv_tasks.size()});
    H.qcnt.alloc(qn, acct);
    H.qcap = (int)qn;

    H.qctr.alloc(2 * kQueues + 1, acct);
    H.fq.alloc(qn, acct);
    // claim tags of the factor instances (chunk continuations of the warp-specialised kernel):
    // tag = launch epoch (>= 1), so the buffer is zeroed once
    H.fclaim.alloc((size_t)S * A.factor_tasks.size(), acct);
    H.fclaim.zero(H.st);
    H.act_slots.alloc(S, acct);
    H.sel_act.alloc(std::max(S, 1), acct);
  }
  H.lslot.alloc(H.Ssel, acct);
  for (DBuf<double>* v : {&H.x, &H.delta, &H.b, &H.qx}) v->zero(H.st);
  CK(cudaStreamSynchronize(H.st));
  clk.mark("build: workspaces");
  H.analyze_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---------------------------------------------------------------------------
// device phases

static cudaEvent_t ev_get(Handle& H) {
  if (H.ev_pool.empty()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = H.ev_pool.back();
  H.ev_pool.pop_back();
  return e;
}
// phase timer: two events on the engine stream, resolved by flush_timers()
struct Timer {
  Handle& H;
  cudaEvent_t a, b;
  double* acc;
  Timer(Handle& h, double* accum) : H(h), acc(accum) {
    a = ev_get(H);
    b = ev_get(H);
    cudaEventRecord(a, H.st);
  }
  ~Timer() {
    cudaEventRecord(b, H.st);
    H.pending.push_back({a, b, acc});
  }
};
static void flush_timers(Handle& H) {
  for (auto& p : H.pending) {
    cudaEventSynchronize(p.b);
    float ms = 0;
    cudaEventElapsedTime(&ms, p.a, p.b);
    *p.acc += ms;
    H.ev_pool.push_back(p.a);
    H.ev_pool.push_back(p.b);
  }
  H.pending.clear();
}

static int n_active(const Handle& H);
static void run_factor(Handle& H, const double* qv, int S) {
  Analysis& A = H.an;
  FactorArgs f{};
  f.S = S;
  f.n_base = (int64_t)A.factor_tasks.size();
  f.tasks = H.d_ftasks.p;
  f.rec = H.d_frec.p;
  f.upd_k = H.d_upd_k.p;
  f.L = H.L.p;
  f.Linv = H.Linv.p;
  f.nT = A.nT;
  f.NT = A.NT;
  f.tile_row = H.d_tile_row.p;
  f.tile_col = H.d_tile_col.p;
  f.tstart = H.d_tstart.p;
  f.upd_a = H.d_upd_a.p;
  f.upd_b = H.d_upd_b.p;
  f.chunk_rng = H.d_chunk_rng.p;
  f.chunk_tile = H.d_chunk_tile.p;
  f.chunk_flags = H.d_chunk_flags.p;
  f.tbsz = H.d_tbsz.p;
  f.grp_rng = H.d_grp_rng.p;
  f.grp_tile = H.d_grp_tile.p;
  f.chunk_grp_ptr = H.d_chunk_grp_ptr.p;
  f.G = H.Gbuf.p;
  f.ngrp = std::max(A.ngrp, 1);
  f.qptr = H.d_qptr.p;
  f.qloc = H.d_qloc.p;
  f.qv = qv;
  f.nq = H.nq;
  f.diagq = H.d_diagq.p;
  f.status = H.status.p;
  f.rel_tol = 1e-13;
  f.trace = nullptr;
  f.flops_per_level = (double)A.factor_flops_limited / std::max(1, A.f_depth);
  static const char* trace_path = getenv("PINLA_TRACE");
  static int traced = 0;
  unsigned long long* tbuf = nullptr;
  const size_t ntask = (size_t)f.n_base * S;
  if (trace_path && !traced && n_active(H) == S) {
    CK(cudaMalloc(&tbuf, ntask * 8 * sizeof(unsigned long long)));
    CK(cudaMemsetAsync(tbuf, 0, ntask * 8 * sizeof(unsigned long long), H.st));
    f.trace = tbuf;
  }
  {
    std::vector<int> acts;
    for (int i = 0; i < (int)H.active_h.size() && i < S; ++i)
      if (H.active_h[i]) acts.push_back(i);
    h2d(H.act_slots.p, acts.data(), acts.size(), H.st);
    f.q.ntask = (int)A.factor_tasks.size();
    f.q.ndep0 = H.d_f_ndep.p;
    f.q.succ_ptr = H.d_f_succ_ptr.p;
    f.q.succ = H.d_f_succ.p;
    f.q.ready0 = H.d_f_ready0.p;
    static const char* f_sched = getenv("PINLA_FACTOR_SCHED");
    f.q.fifo = (f_sched && f_sched[0] == 'f') ? 1 : 0;
    f.q.nlane = f.q.fifo ? 0 : A.f_nlane;
    static const int lane_ctas = getenv("PINLA_LANE_CTAS") ? atoi(getenv("PINLA_LANE_CTAS")) : kLaneCtas;  // tuning
    f.q.lane_ctas = std::max(1, std::min(lane_ctas, kLaneCtasMax));
    f.q.fqueue = H.fq.p;
    f.q.hot = nullptr;
    static const bool f_cont = !(getenv("PINLA_FACTOR_CONT") && getenv("PINLA_FACTOR_CONT")[0] == '0');  // tuning
    f.q.claimed = f_cont ? H.fclaim.p : nullptr;
    f.q.prio = H.d_f_prio.p;
    f.q.nready0 = (int)A.f_ready0.size();
    f.q.cnt = H.qcnt.p;
    f.q.queue = nullptr;
    f.q.order = H.d_f_order.p;
    f.q.ctr = H.qctr.p;
    f.q.cap = H.qcap;
    f.q.epoch = ++H.qepoch;
    f.q.act_slots = H.act_slots.p;
    f.q.nact = (int)acts.size();
  }
  set_int_kernel<<<(S + 63) / 64, 64, 0, H.st>>>(H.status.p, S, INT_MAX);
  CK(launch_factor(f, H.st));
  if (tbuf) {
    std::vector<unsigned long long> hb(ntask * 8);
    CK(cudaMemcpyAsync(hb.data(), tbuf, hb.size() * 8, cudaMemcpyDeviceToHost, H.st));
    CK(cudaStreamSynchronize(H.st));
    cudaFree(tbuf);
    FILE* fp = fopen(trace_path, "wb");
    if (fp) {
      int64_t hdr[2] = {(int64_t)f.n_base, (int64_t)S};
      fwrite(hdr, 8, 2, fp);
      std::vector<int4> tk(A.factor_tasks.size());
      for (size_t i = 0; i < tk.size(); ++i)
        tk[i] = make_int4(A.factor_tasks[i].type, 0, A.factor_tasks[i].id, A.factor_tasks[i].level);
      fwrite(tk.data(), sizeof(int4), tk.size(), fp);
      fwrite(hb.data(), 8, hb.size(), fp);
      // pairs per task: main tiles (tail) and partials
      std::vector<int64_t> np(tk.size());
      for (size_t i = 0; i < tk.size(); ++i) {
        if (tk[i].x == 1) {
          np[i] = A.grp_rng[tk[i].z + 1] - A.grp_rng[tk[i].z];
          continue;
        }
        const int c = tk[i].z, t = A.chunk_tile[c];
        np[i] = A.chunk_rng[c + 1] - A.chunk_rng[c] + 1000 * (A.tile_row[t] == A.tile_col[t]) +
                10000 * ((A.chunk_flags[c] & 2) ? 1 : 0);
      }
      fwrite(np.data(), 8, np.size(), fp);
      int64_t ns = (int64_t)A.f_succ.size();
      fwrite(&ns, 8, 1, fp);
      fwrite(A.f_succ_ptr.data(), 4, A.f_succ_ptr.size(), fp);
      fwrite(A.f_succ.data(), 4, A.f_succ.size(), fp);
      // per task: tile row, tile col, rows of I, rows of J
      std::vector<int32_t> ti(4 * tk.size());
      for (size_t i = 0; i < tk.size(); ++i) {
        const int t = tk[i].x == 1 ? A.grp_tile[tk[i].z] : A.chunk_tile[tk[i].z];
        ti[4 * i] = A.tile_row[t];
        ti[4 * i + 1] = A.tile_col[t];
        ti[4 * i + 2] = (int)(A.tstart[A.tile_row[t] + 1] - A.tstart[A.tile_row[t]]);
        ti[4 * i + 3] = (int)(A.tstart[A.tile_col[t] + 1] - A.tstart[A.tile_col[t]]);
      }
      fwrite(ti.data(), 4, ti.size(), fp);
      fclose(fp);
    }
    traced = 1;
  }
  if (H.links_on) {
    LinkArgs la{};
    la.S = S;
    la.nlink = H.nlinks;
    la.links = H.d_links.p;
    la.active = H.active.p;
    la.L = H.L.p;
    la.Linv = H.Linv.p;
    la.M = H.Mlink.p;
    la.nT = A.nT;
    la.NT = A.NT;
    la.tbsz = H.d_tbsz.p;
    CK(launch_link_tiles(la, H.st));
    H.launches += 1;
  }
  logdiag_part_kernel<<<dim3(kLogParts, S), 256, 0, H.st>>>(H.L.p, A.nT, A.NT, H.d_colptr.p,
                                                           H.logparts.p, H.active.p);
  rowsum_kernel<<<S, 32, 0, H.st>>>(H.logparts.p, kLogParts, H.ldsum.p, H.active.p);
  H.launches += 4;  // queue init, factor, log-diagonal parts, row sums
  H.n_factor += 1;
  H.factor_slot_runs += n_active(H);
}

static void run_solve(Handle& H, const double* b, double* x, int S) {
  Analysis& A = H.an;
  SolveArgs s{};
  s.S = S;
  s.n_base = (int64_t)A.solve_tasks.size();
  s.tasks = H.d_stasks.p;
  s.counter = H.counter.p;
  s.epoch = ++H.epoch;
  s.active = H.active.p;
  s.llY = H.llY.p;
  s.llX = H.llX.p;
  s.llP = H.llP.p;
  s.L = H.L.p;
  s.Linv = H.Linv.p;
  s.nT = A.nT;
  s.NT = A.NT;
  s.tile_row = H.d_tile_row.p;
  s.tile_col = H.d_tile_col.p;
  s.colptr = H.d_colptr.p;
  s.rowptr = H.d_rowptr.p;
  s.row_tid = H.d_row_tid.p;
  s.row_col = H.d_row_col.p;
  s.b = b;
  s.x = x;
  s.M = H.links_on ? H.Mlink.p : nullptr;
  s.nlinks = A.solve_links;
  s.grp = H.d_sgrp.p;
  s.n_grp = A.n_sgrp;
  s.fgp = H.d_sf_ptr.p;
  s.bgp = H.d_sb_ptr.p;
  s.trace = nullptr;
  static const char* trace_path = getenv("PINLA_TRACE_SOLVE");
  static int traced = 0;
  const size_t ntask = (size_t)s.n_base * S;
  if (trace_path && !traced && n_active(H) == S) {
    CK(cudaMalloc(&s.trace, ntask * 8 * sizeof(unsigned long long)));
    CK(cudaMemsetAsync(s.trace, 0, ntask * 8 * sizeof(unsigned long long), H.st));
  }
  {
    Timer t(H, &H.t_solvek);
    CK(launch_solve(s, H.st));
  }
  if (s.trace) {
    // dump: header (n_base, S), tasks (type, -, id, level), per-instance
    // (t_claim, t_early, t_esum, t_late, t_ready, t_end, smid, 0) with instance = base * S + slot, then
    // the tile row / col of every tile (product tasks carry tile ids)
    std::vector<unsigned long long> hb(ntask * 8);
    CK(cudaMemcpyAsync(hb.data(), s.trace, hb.size() * 8, cudaMemcpyDeviceToHost, H.st));
    CK(cudaStreamSynchronize(H.st));
    cudaFree(s.trace);
    if (FILE* fp = fopen(trace_path, "wb")) {
      int64_t hdr[3] = {(int64_t)s.n_base, (int64_t)S, (int64_t)A.nT};
      fwrite(hdr, 8, 3, fp);
      std::vector<int4> tk(A.solve_tasks.size());
      for (size_t i = 0; i < tk.size(); ++i)
        tk[i] = make_int4(A.solve_tasks[i].type, 0, A.solve_tasks[i].id, A.solve_tasks[i].level);
      fwrite(tk.data(), sizeof(int4), tk.size(), fp);
      fwrite(hb.data(), 8, hb.size(), fp);
      fwrite(A.tile_row.data(), 4, A.tile_row.size(), fp);
      fwrite(A.tile_col.data(), 4, A.tile_col.size(), fp);
      fclose(fp);
    }
    traced = 1;
  }
  H.launches += 1;
  H.n_solve += 1;
  H.solve_slot_runs += n_active(H);
}

// per-slot scalars after reduce: red[s*3 + k]
static void reduce3(Handle& H, int wdt, int maxmask, int S) {
  vk_reduce(H.parts.p, H.vm.nred, wdt, maxmask, H.red.p, H.active.p, S, H.st);
  H.launches += 1;
}

struct SlotOut {
  int status = PINLA_OK;
  int64_t badcol = -1;
  int iters = 0;
  double ll = 0, quad = 0, ldc = 0, ldp = 0;
  bool done = false;
};


static void set_active(Handle& H, const std::vector<int>& act) {
  h2d(H.active.p, act.data(), act.size(), H.st);
  H.active_h = act;
}
static int n_active(const Handle& H) {
  int c = 0;
  for (int v : H.active_h) c += v;
  return c;
}

// device time of one C-ABI call (events on the engine stream)
struct CallTimer {
  Handle& H;
  cudaEvent_t a, b;
  explicit CallTimer(Handle& h) : H(h) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, H.st);
  }
  ~CallTimer() {
    cudaEventRecord(b, H.st);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    H.last_call_ms = ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    flush_timers(H);
  }
};

// g(x) components of the active slots at x, enqueued without a host sync:
// eta = A x, likelihood (+ d1, w when `derivs`), qx = Q_prior x; the reduced
// scalars land in pinned staging: pp[2s..2s+1] = likelihood parts,
// xq[3s] = x . qx.  Overwrites eta/qx (and d1/w) of the active slots only.
static void enqueue_lik_quad_to(Handle& H, const double* x, double* eta, double* d1, double* w,
                                double* qx, bool derivs, int S, double* pp, double* xq) {
  vk_spmv_A(H.vm, x, eta, H.active.p, S, H.st);
  vk_lik(H.vm, eta, H.tau.p, derivs ? d1 : nullptr, derivs ? w : nullptr, H.parts.p, H.active.p, S,
         H.st);
  reduce3(H, 2, 0, S);
  d2h(pp, H.red.p, 2 * (size_t)S, H.st);
  vk_symv(H.vm, H.pv.p, x, qx, H.active.p, S, H.st);
  vk_dot_max(H.vm, x, qx, H.parts.p, H.active.p, S, H.st);
  reduce3(H, 3, 6, S);
  d2h(xq, H.red.p, 3 * (size_t)S, H.st);
  H.launches += 4;
}
static void enqueue_lik_quad(Handle& H, const double* x, bool derivs, int S, double* pp, double* xq) {
  enqueue_lik_quad_to(H, x, H.eta.p, H.d1.p, H.w.p, H.qx.p, derivs, S, pp, xq);
}

static double loglik(const Handle& H, double p0, double p1, double tau) {
  if (H.family == PINLA_FAMILY_GAUSSIAN)
    return 0.5 * (double)H.m * (std::log(tau) - LOG_2PI) - 0.5 * tau * p0;
  return p0 - p1 - H.lgamma_const;
}

// conditional mode for k slots (thetas k x d); leaves factor + x on device.
//
// Host round trips: one per Newton iteration (the factorization, the
// solve, the convergence scalars AND the full step alpha = 1 are enqueued
// together; the step's g(x + delta) is computed speculatively for every
// iterating slot) plus one per further halving try.  The accepted try's
// eta/d1/w/qx are those of the new iterate, so the next iteration starts
// from them instead of recomputing g(x): same kernels, same values.
// warm: one start for every slot (warm_stride 0) or slot s at warm + s * warm_stride
static void mode_batch(Handle& H, int k, const double* thetas, const double* warm,
                       std::vector<SlotOut>& out, int64_t warm_stride = 0) {
  const int S = H.S;
  const int64_t npad = H.an.npad();
  double* pR = H.hpin;            // [3S] (x.b, max|a|, max|b|) of dot_max(delta, x)
  double* pLd = pR + 3 * S;       // [S] sum log diag L
  double* pPP = pLd + S;          // [2S] likelihood parts
  double* pXQ = pPP + 2 * S;      // [3S] x . Qp x
  int* pSt = H.hpin_i;            // [S] factor status
  out.assign(S, SlotOut());
  std::vector<int> act(S, 0);
  for (int s = 0; s < k; ++s) act[s] = 1;
  std::vector<double> gains(S * std::max<size_t>(H.gain_kind.size(), 1), 0.0), tau(S, 1.0);
  for (int s = 0; s < k; ++s) {
    compute_gains(H, thetas + (size_t)s * H.d, gains.data() + s * H.gain_kind.size());
    tau[s] = H.noise_theta >= 0 ? std::exp(thetas[(size_t)s * H.d + H.noise_theta]) : H.noise_precision;
  }
  h2d(H.gains.p, gains.data(), gains.size(), H.st);
  h2d(H.tau.p, tau.data(), S, H.st);
  set_active(H, act);
  {
    Timer t(H, &H.t_assemble);
    vk_prior_values(H.vm, H.gains.p, H.pv.p, H.active.p, S, H.st);
    H.asm_bytes_done += H.asm_bytes[0] * n_active(H);
    H.launches++;
  }

  if (H.family == PINLA_FAMILY_GAUSSIAN) {
    {
      Timer t(H, &H.t_assemble);
      vk_cond_values(H.vm, H.pv.p, H.tau.p, nullptr, 0, H.qv.p, H.gchbuf.p, H.active.p, S, H.st);
      H.asm_bytes_done += H.asm_bytes[1] * n_active(H);
      H.launches++;
    }
    {
      Timer t(H, &H.t_factor);
      run_factor(H, H.qv.p, S);
    }
    {
      Timer t(H, &H.t_solve);
      // rhs = A^T (tau (y - offsets)): lik at eta = 0 gives d1 = tau (y - off)
      CK(cudaMemsetAsync(H.eta.p, 0, (size_t)S * H.m * sizeof(double), H.st));
      vk_lik(H.vm, H.eta.p, H.tau.p, H.d1.p, H.w.p, H.parts.p, H.active.p, S, H.st);
      vk_AT(H.vm, H.d1.p, nullptr, H.b.p, H.chbuf.p, H.active.p, S, H.st);
      H.launches += 3;
      run_solve(H, H.b.p, H.x.p, S);
    }
    d2h(pSt, H.status.p, S, H.st);
    d2h(pLd, H.ldsum.p, S, H.st);
    {
      Timer t(H, &H.t_other);
      enqueue_lik_quad(H, H.x.p, false, S, pPP, pXQ);
    }
    CK(cudaStreamSynchronize(H.st));
    for (int s = 0; s < k; ++s) {
      SlotOut& o = out[s];
      o.iters = 1;
      o.done = true;
      if (pSt[s] != INT_MAX) {
        o.status = PINLA_NOT_PD;
        o.badcol = H.an.perm[pSt[s]];
        continue;
      }
      o.ldc = 2.0 * pLd[s];
      o.ll = loglik(H, pPP[2 * s], pPP[2 * s + 1], tau[s]);
      o.quad = pXQ[3 * s];
    }
    flush_timers(H);
    return;
  }

  // ---------------- poisson: damped Newton (objective.py:259-296) ----------
  // warm start: one pinned upload, replicated to the slots on the device
  // (the staging buffer is only rewritten after the next host sync)
  if (warm && warm_stride > 0) {
    // per-slot warm starts (pinla_eval_batch_warm): one pinned upload
    if (!H.hpin_xs) CK(cudaMallocHost(&H.hpin_xs, sizeof(double) * (size_t)S * npad));
    std::fill(H.hpin_xs, H.hpin_xs + (size_t)k * npad, 0.0);
    for (int s = 0; s < k; ++s) {
      double* xs = H.hpin_xs + (size_t)s * npad;
      const double* ws = warm + (size_t)s * warm_stride;
      for (int64_t i = 0; i < H.n; ++i) xs[H.an.pad_of_orig[i]] = ws[i];
    }
    h2d(H.x.p, H.hpin_xs, (size_t)k * npad, H.st);
  } else {
    double* xinit = H.hpin_x;
    std::fill(xinit, xinit + npad, 0.0);
    if (warm) {
      for (int64_t i = 0; i < H.n; ++i) xinit[H.an.pad_of_orig[i]] = warm[i];
    }
    h2d(H.x.p, xinit, npad, H.st);
    for (int s = 1; s < S; ++s)
      CK(cudaMemcpyAsync(H.x.p + (size_t)s * npad, H.x.p, npad * sizeof(double),
                         cudaMemcpyDeviceToDevice, H.st));
  }
  std::vector<int> iter_act = act, search(S, 0), accepted(S, 0);
  std::vector<double> g0(S), best(S), cur_ll(S), cur_q(S);
  // g at the starting point (and d1, w, qx of the first Newton system)
  {
    Timer t(H, &H.t_other);
    enqueue_lik_quad(H, H.x.p, true, S, pPP, pXQ);
  }
  CK(cudaStreamSynchronize(H.st));
  for (int s = 0; s < k; ++s) {
    cur_ll[s] = loglik(H, pPP[2 * s], pPP[2 * s + 1], tau[s]);
    cur_q[s] = pXQ[3 * s];
  }
  // halving tries t in [t0, t1) for the active slots: x_t = x + 2^-t delta
  // (try buffers t), its g components and derivatives, and g(x_t) - g(x) as
  // sums of per-term differences (vk_gdiff) into the pinned staging of try t:
  // pp[2S] | xq[3S] | dg[2S]
  const size_t SN = (size_t)S * npad, SM = (size_t)S * H.m;
  auto pin_try = [&](int t) { return H.hpin_t + (size_t)t * 7 * S; };
  auto enqueue_tries = [&](int t0, int t1) {
    Timer t(H, &H.t_other);
    for (int tr = t0; tr < t1; ++tr) {
      double* tp = pin_try(tr);
      double* xt = H.tx.p + tr * SN;
      double* et = H.teta.p + tr * SM;
      double* qt = H.tqx.p + tr * SN;
      vk_axpy(npad, H.x.p, H.delta.p, H.talpha.p + (size_t)tr * S, xt, H.active.p, S, H.st);
      enqueue_lik_quad_to(H, xt, et, H.td1.p + tr * SM, H.tw.p + tr * SM, qt, true, S, tp, tp + 2 * S);
      vk_gdiff(H.vm, H.eta.p, et, H.tau.p, H.x.p, xt, H.qx.p, qt, H.parts.p, H.active.p, S, H.st);
      reduce3(H, 2, 0, S);
      d2h(tp + 5 * S, H.red.p, 2 * (size_t)S, H.st);
      H.launches += 2;
    }
  };
  // the ascent test of try t for slot s (objective.py:280-286): g_try and
  // g_try - g0 (the difference evaluated term by term); true = accept
  auto judge = [&](int s, int tr) {
    const double* tp = pin_try(tr);
    const double llt = loglik(H, tp[2 * s], tp[2 * s + 1], tau[s]);
    const double gt = -0.5 * tp[2 * S + 3 * s] + llt;
    const double dg = tp[5 * S + 2 * s] - 0.5 * tp[5 * S + 2 * s + 1];
    const bool fin = std::isfinite(gt) && std::isfinite(dg);
    if (fin) best[s] = std::max(best[s], dg);
    if (fin && dg >= 0.0) {
      cur_ll[s] = llt;
      cur_q[s] = tp[2 * S + 3 * s];
      return true;
    }
    return false;
  };
  // accepted tries become the iterates (x, eta, d1, w, Qp x): one launch
  std::vector<int> take(S, -1);
  auto take_tries = [&]() {
    bool any = false;
    for (int s = 0; s < S; ++s) any |= take[s] >= 0;
    if (!any) return;
    h2d(H.sel.p, take.data(), S, H.st);
    vk_take_try(npad, H.m, S, H.sel.p, H.tx.p, H.tqx.p, H.teta.p, H.td1.p, H.tw.p, H.x.p, H.qx.p,
                H.eta.p, H.d1.p, H.w.p, H.st);
    H.launches++;
  };
  for (int it = 1; it <= H.max_inner; ++it) {
    int nact = 0;
    for (int s = 0; s < S; ++s) nact += iter_act[s];
    if (!nact) break;
    set_active(H, iter_act);
    for (int s = 0; s < S; ++s)
      if (iter_act[s]) g0[s] = -0.5 * cur_q[s] + cur_ll[s];
    {
      Timer t(H, &H.t_assemble);
      vk_cond_values(H.vm, H.pv.p, H.tau.p, H.w.p, 1, H.qv.p, H.gchbuf.p, H.active.p, S, H.st);
      H.asm_bytes_done += H.asm_bytes[2] * n_active(H);
      H.launches++;
    }
    {
      Timer t(H, &H.t_factor);
      run_factor(H, H.qv.p, S);
    }
    {
      Timer t(H, &H.t_solve);
      vk_AT(H.vm, H.d1.p, H.qx.p, H.b.p, H.chbuf.p, H.active.p, S, H.st);
      H.launches += 2;
      run_solve(H, H.b.p, H.delta.p, S);
    }
    vk_dot_max(H.vm, H.delta.p, H.x.p, H.parts.p, H.active.p, S, H.st);
    H.launches++;
    reduce3(H, 3, 6, S);
    d2h(pR, H.red.p, 3 * (size_t)S, H.st);
    d2h(pSt, H.status.p, S, H.st);
    d2h(pLd, H.ldsum.p, S, H.st);
    // speculative full step (try 0) for every iterating slot
    enqueue_tries(0, 1);
    CK(cudaStreamSynchronize(H.st));
    for (int s = 0; s < S; ++s) {
      search[s] = 0;
      accepted[s] = 0;
      take[s] = -1;
      if (!iter_act[s]) continue;
      SlotOut& o = out[s];
      o.iters = it;
      if (pSt[s] != INT_MAX) {
        o.status = PINLA_NOT_PD;
        o.badcol = H.an.perm[pSt[s]];
        o.done = true;
        iter_act[s] = 0;
        continue;
      }
      const double dmax = pR[3 * s + 1], xmax = pR[3 * s + 2];
      o.ldc = 2.0 * pLd[s];
      o.ll = cur_ll[s];
      o.quad = cur_q[s];
      if (dmax <= H.inner_tol * (1.0 + xmax)) {
        o.done = true;
        iter_act[s] = 0;
        continue;
      }
      best[s] = -INFINITY;
      if (judge(s, 0)) {
        accepted[s] = 1;
        take[s] = 0;
      } else {
        search[s] = 1;
      }
    }
    // step halving: alpha = 2^-1 .. 2^-10 (objective.py:276-289, 11 tries in
    // all).  The remaining tries of the slots still searching are enqueued
    // together (one more round trip instead of up to ten) and decided in the
    // reference's order on the host: first ascent wins.
    int nsearch = 0;
    for (int s = 0; s < S; ++s) nsearch += search[s];
    if (nsearch) {
      set_active(H, search);
      enqueue_tries(1, kTries);
      CK(cudaStreamSynchronize(H.st));
      for (int s = 0; s < S; ++s) {
        if (!search[s]) continue;
        for (int tr = 1; tr < kTries; ++tr)
          if (judge(s, tr)) {
            accepted[s] = 1;
            take[s] = tr;
            break;
          }
      }
    }
    take_tries();
    for (int s = 0; s < S; ++s) {
      if (!iter_act[s] || accepted[s]) continue;
      SlotOut& o = out[s];
      // no ascent: flat floor accepts the current point (objective.py:290-295)
      o.done = true;
      iter_act[s] = 0;
      if (!(best[s] >= -1e-9 * (1.0 + std::fabs(g0[s])))) o.status = PINLA_INNER_DIVERGENCE;
    }
  }
  for (int s = 0; s < k; ++s)
    if (!out[s].done) {
      out[s].status = PINLA_INNER_DIVERGENCE;
      out[s].done = true;
    }
  set_active(H, act);
  flush_timers(H);
}

// prior log-determinant by factorizing Q_prior on the shared tile structure
static void prior_logdet(Handle& H, int k, std::vector<SlotOut>& out) {
  const int S = H.S;
  std::vector<int> act(S, 0);
  for (int s = 0; s < k; ++s) act[s] = out[s].status == PINLA_OK ? 1 : 0;
  set_active(H, act);
  {
    Timer t(H, &H.t_assemble);
    vk_cond_values(H.vm, H.pv.p, H.tau.p, nullptr, 2, H.qv.p, H.gchbuf.p, H.active.p, S, H.st);
    H.asm_bytes_done += H.asm_bytes[3] * n_active(H);
    H.launches++;
  }
  {
    Timer t(H, &H.t_factor);
    run_factor(H, H.qv.p, S);
  }
  std::vector<int> status_h(S);
  std::vector<double> ld(S);
  d2h(status_h.data(), H.status.p, S, H.st);
  d2h(ld.data(), H.ldsum.p, S, H.st);
  CK(cudaStreamSynchronize(H.st));
  for (int s = 0; s < k; ++s) {
    if (!act[s]) continue;
    if (status_h[s] != INT_MAX) {
      out[s].status = PINLA_NOT_PD;
      out[s].badcol = H.an.perm[status_h[s]];
    } else {
      out[s].ldp = 2.0 * ld[s];
    }
  }
}

// closed-form log det Q_prior(theta) (model.py lattice / AR(1) kinds)
static double lattice_logdet(int64_t nx, int64_t ny, double log_tau, double log_kappa) {
  const double k2 = std::exp(2.0 * log_kappa);
  std::vector<double> lam(nx), mu(ny);
  for (int64_t j = 0; j < nx; ++j) lam[j] = 2.0 - 2.0 * std::cos(M_PI * (double)j / (double)nx);
  for (int64_t k = 0; k < ny; ++k) mu[k] = 2.0 - 2.0 * std::cos(M_PI * (double)k / (double)ny);
  double s = 0.0;
  for (int64_t k = 0; k < ny; ++k) {
    double r = 0.0;
    for (int64_t j = 0; j < nx; ++j) r += std::log(k2 + lam[j] + mu[k]);
    s += r;
  }
  return (double)(nx * ny) * log_tau + 2.0 * s;
}
static double ar1_logdet(int64_t nt, double logit_rho) {
  const double rho = 1.0 / (1.0 + std::exp(-logit_rho));
  return -(double)(nt - 1) * std::log(1.0 - rho * rho);
}
static double analytic_prior_logdet(const Handle& H, const double* th) {
  double s = 0.0;
  for (size_t i = 0; i < H.ld_kind.size(); ++i) {
    const int k = H.ld_theta[i];
    const int64_t nx = H.ld_dims[3 * i], ny = H.ld_dims[3 * i + 1], nt = H.ld_dims[3 * i + 2];
    switch (H.ld_kind[i]) {
      case PINLA_LD_CONST: s += H.ld_value[i]; break;
      case PINLA_LD_SPDE: s += lattice_logdet(nx, ny, th[k], th[k + 1]); break;
      case PINLA_LD_ST:
        s += (double)(nx * ny) * ar1_logdet(nt, th[k + 2]) + (double)nt * lattice_logdet(nx, ny, th[k], th[k + 1]);
        break;
      default: s += (double)nt * th[k] + ar1_logdet(nt, th[k + 1]); break;
    }
  }
  return s;
}

static void to_orig(const Handle& H, const double* pad, double* orig) {
  for (int64_t i = 0; i < H.n; ++i) orig[i] = pad[H.an.pad_of_orig[i]];
}

}  // namespace pinla

// ===========================================================================
// C-ABI

using namespace pinla;

struct pinla_handle {
  Handle h;
};

#define API_BEGIN try {
#define API_END                     \
  }                                 \
  catch (const std::exception& e) { \
    g_err = e.what();               \
    return -1;                      \
  }                                 \
  return 0;

extern "C" {

const char* pinla_last_error(void) { return g_err.c_str(); }

int pinla_scalar_pattern(int64_t n, const int64_t* indptr, const int64_t* indices,
                         const int64_t* perm, int64_t* nnz_out, int64_t* Lp_out, int64_t* Li_out) {
  API_BEGIN
  std::vector<int64_t> Lp, Li;
  scalar_pattern(n, indptr, indices, perm, Lp, Li);
  if (nnz_out) *nnz_out = Lp[n];
  if (Lp_out) std::copy(Lp.begin(), Lp.end(), Lp_out);
  if (Li_out) std::copy(Li.begin(), Li.end(), Li_out);
  API_END
}

int pinla_nd_order(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t leaf_cutoff,
                   int64_t tile_max, int64_t* perm_out, int64_t* n_dense_out,
                   int64_t* tile_bounds_out, int64_t* n_bounds_out, int64_t* node_start,
                   int64_t* node_end, int64_t* node_parent, int64_t* n_nodes_out) {
  API_BEGIN
  if (tile_max < 1 || tile_max > TB) throw std::runtime_error("tile_max must be in [1, 64]");
  NDResult r = nested_dissection(n, indptr, indices, leaf_cutoff);
  std::copy(r.perm.begin(), r.perm.end(), perm_out);
  if (n_dense_out) *n_dense_out = r.n_dense;
  if (tile_bounds_out) {
    std::vector<int64_t> b = nd_tile_bounds(r, tile_max);
    std::copy(b.begin(), b.end(), tile_bounds_out);
    if (n_bounds_out) *n_bounds_out = (int64_t)b.size();
  }
  if (n_nodes_out) *n_nodes_out = (int64_t)r.nodes.size();
  for (size_t i = 0; i < r.nodes.size(); ++i) {
    if (node_start) node_start[i] = r.nodes[i].start;
    if (node_end) node_end[i] = r.nodes[i].end;
    if (node_parent) node_parent[i] = r.nodes[i].parent;
  }
  API_END
}

int pinla_analyze_pattern(int64_t n, const int64_t* indptr, const int64_t* indices,
                          const int64_t* perm, int64_t n_dense, const int64_t* tile_bounds,
                          int64_t n_tile_bounds, pinla_analysis_info* out,
                          int32_t* tile_rows_out, int32_t* tile_cols_out) {
  API_BEGIN
  Analysis A;
  analyze_tiles(A, n, indptr, indices, perm, n_dense, tile_bounds, n_tile_bounds);
  out->n_tile_rows = A.NT;
  out->n_tiles = A.nT;
  out->n_update_pairs = (int64_t)A.upd_a.size();
  out->factor_flops = A.factor_flops;
  out->selinv_flops = A.selinv_flops;
  out->solve_bytes = A.solve_bytes;
  int64_t df = 0, db = 0;
  for (int32_t J = 0; J < A.NT; ++J) {
    df = std::max<int64_t>(df, A.flevel[J] + 1);
    db = std::max<int64_t>(db, A.blevel[J] + 1);
  }
  out->depth_forward = df;
  out->depth_backward = db;
  out->factor_flops_limited = A.factor_flops_limited;
  if (tile_rows_out) std::copy(A.tile_row.begin(), A.tile_row.end(), tile_rows_out);
  if (tile_cols_out) std::copy(A.tile_col.begin(), A.tile_col.end(), tile_cols_out);
  API_END
}
const char* pinla_version(void) { return "pinla-b200 0.1 (sm_100a, fp64 tile-DAG)"; }

int pinla_create(const pinla_model* model, const pinla_options* opt, pinla_handle** out) {
  API_BEGIN
  if (!model || !opt || !out) throw std::runtime_error("null argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw std::runtime_error("no CUDA device available (the engine has no CPU fallback)");
  auto* ph = new pinla_handle();
  try {
    build(ph->h, model, opt);
  } catch (...) {
    delete ph;
    throw;
  }
  *out = ph;
  API_END
}

void pinla_destroy(pinla_handle* h) {
  if (!h) return;
  cudaSetDevice(h->h.device);
  cudaStreamSynchronize(h->h.st);
  cudaStream_t st = h->h.st;
  delete h;
  if (st) cudaStreamDestroy(st);
}

static void eval_batch_impl(Handle& H, int32_t k, const double* thetas, const double* warm,
                            int64_t warm_stride, double* f_out, double* comps_out,
                            int32_t* status_out, int64_t* badcol_out, int32_t* iters_out,
                            double* logdets_out, double* modes_out);

int pinla_eval_batch(pinla_handle* ph, int32_t k, const double* thetas, const double* warm,
                     double* f_out, double* comps_out, int32_t* status_out, int64_t* badcol_out,
                     int32_t* iters_out, double* logdets_out, double* modes_out) {
  API_BEGIN
  eval_batch_impl(ph->h, k, thetas, warm, 0, f_out, comps_out, status_out, badcol_out, iters_out,
                  logdets_out, modes_out);
  API_END
}

int pinla_eval_batch_warm(pinla_handle* ph, int32_t k, const double* thetas, const double* warms,
                          double* f_out, double* comps_out, int32_t* status_out,
                          int64_t* badcol_out, int32_t* iters_out, double* logdets_out,
                          double* modes_out) {
  API_BEGIN
  if (!warms) throw std::runtime_error("pinla_eval_batch_warm: warms is NULL");
  eval_batch_impl(ph->h, k, thetas, warms, ph->h.n, f_out, comps_out, status_out, badcol_out,
                  iters_out, logdets_out, modes_out);
  API_END
}

static void eval_batch_impl(Handle& H, int32_t k, const double* thetas, const double* warm,
                            int64_t warm_stride, double* f_out, double* comps_out,
                            int32_t* status_out, int64_t* badcol_out, int32_t* iters_out,
                            double* logdets_out, double* modes_out) {
  CK(cudaSetDevice(H.device));
  CallTimer ct(H);
  const int64_t npad = H.an.npad();
  std::vector<double> xp;
  for (int32_t base = 0; base < k; base += H.S) {
    const int kk = std::min<int32_t>(H.S, k - base);
    std::vector<SlotOut> out;
    // the closed-form prior log-dets (host, O(n) logs per slot) overlap the
    // device work of the batch
    std::vector<double> ldp(kk, 0.0);
    std::thread ld_thread;
    if (H.analytic_logdet)
      ld_thread = std::thread([&, base, kk]() {
        for (int s = 0; s < kk; ++s) ldp[s] = analytic_prior_logdet(H, thetas + (size_t)(base + s) * H.d);
      });
    try {
      mode_batch(H, kk, thetas + (size_t)base * H.d,
                 warm && warm_stride > 0 ? warm + (size_t)base * warm_stride : warm, out, warm_stride);
    } catch (...) {
      if (ld_thread.joinable()) ld_thread.join();
      throw;
    }
    if (ld_thread.joinable()) ld_thread.join();
    if (modes_out) {
      xp.resize((size_t)kk * npad);
      d2h(xp.data(), H.x.p, xp.size(), H.st);
      CK(cudaStreamSynchronize(H.st));
      for (int s = 0; s < kk; ++s)
        to_orig(H, xp.data() + (size_t)s * npad, modes_out + (size_t)(base + s) * H.n);
    }
    if (H.analytic_logdet) {
      for (int s = 0; s < kk; ++s)
        if (out[s].status == PINLA_OK) out[s].ldp = ldp[s];
    } else {
      prior_logdet(H, kk, out);
    }
    for (int s = 0; s < kk; ++s) {
      const int slot = base + s;
      const SlotOut& o = out[s];
      const double* th = thetas + (size_t)slot * H.d;
      double lph = log_prior_hyper(H, th);
      double lpl = 0.5 * o.ldp - 0.5 * (double)H.n * LOG_2PI - 0.5 * o.quad;
      double lga = 0.5 * o.ldc - 0.5 * (double)H.n * LOG_2PI;
      double f = -(lph + lpl + o.ll - lga);
      if (o.status != PINLA_OK) f = INFINITY;
      if (f_out) f_out[slot] = f;
      if (comps_out) {
        double* c = comps_out + (size_t)slot * 5;
        c[0] = f;
        c[1] = lph;
        c[2] = lpl;
        c[3] = o.ll;
        c[4] = lga;
      }
      if (status_out) status_out[slot] = o.status;
      if (badcol_out) badcol_out[slot] = o.badcol;
      if (iters_out) iters_out[slot] = o.iters;
      if (logdets_out) {
        logdets_out[2 * (size_t)slot] = o.ldc;
        logdets_out[2 * (size_t)slot + 1] = o.ldp;
      }
      H.n_evals++;
    }
  }
}

int pinla_mode(pinla_handle* ph, const double* theta, const double* warm, double* x_out,
               int32_t* iters_out, int32_t* status_out, int64_t* badcol_out, double* logdet_out) {
  API_BEGIN
  Handle& H = ph->h;
  CK(cudaSetDevice(H.device));
  std::vector<SlotOut> out;
  mode_batch(H, 1, theta, warm, out);
  if (x_out) {
    std::vector<double> xp(H.an.npad());
    d2h(xp.data(), H.x.p, xp.size(), H.st);
    CK(cudaStreamSynchronize(H.st));
    to_orig(H, xp.data(), x_out);
  }
  if (iters_out) *iters_out = out[0].iters;
  if (status_out) *status_out = out[0].status;
  if (badcol_out) *badcol_out = out[0].badcol;
  if (logdet_out) *logdet_out = out[0].ldc;
  API_END
}

static void selinv_slot0(Handle& H, double* var_out) {
  Analysis& A = H.an;
  const int64_t npad = A.npad();
  std::vector<int> ls(H.Ssel, 0), acts{0};
  h2d(H.lslot.p, ls.data(), H.Ssel, H.st);
  h2d(H.sel_act.p, acts.data(), 1, H.st);
  {
    Timer t(H, &H.t_selinv);
    SelinvArgs a{};
    a.S = H.Ssel;
    a.n_base = (int64_t)A.selinv_tasks.size();
    a.tasks = H.d_seltasks.p;
    a.lslot = H.lslot.p;
    a.L = H.L.p;
    a.Linv = H.Linv.p;
    a.Sg = H.Sg.p;
    a.tbsz = H.d_tbsz.p;
    a.nT = A.nT;
    a.NT = A.NT;
    a.tile_row = H.d_tile_row.p;
    a.tile_col = H.d_tile_col.p;
    a.pa = H.d_s_pa.p;
    a.pb = H.d_s_pb.p;
    a.mode = H.d_s_mode.p;
    a.chunk_rng = H.d_s_chunk_rng.p;
    a.chunk_tile = H.d_s_chunk_tile.p;
    a.chunk_flags = H.d_s_chunk_flags.p;
    a.grp_rng = H.d_s_grp_rng.p;
    a.grp_tile = H.d_s_grp_tile.p;
    a.tile_grp_ptr = H.d_s_tile_grp_ptr.p;
    a.G = H.Gsel.p;
    a.ngrp = std::max(A.s_ngrp, 1);
    a.gbuf = H.d_s_grp_buf.p;
    a.ngbuf = std::max(A.s_ngbuf, 1);
    a.SL = H.S;
    a.flops_per_level = (double)A.selinv_flops / std::max(1, A.f_depth);
    a.q.ntask = (int)A.selinv_tasks.size();
    a.q.ndep0 = H.d_s_ndep.p;
    a.q.succ_ptr = H.d_s_succ_ptr.p;
    a.q.succ = H.d_s_succ.p;
    a.q.cnt = H.qcnt.p;
    a.q.ctr = H.qctr.p;
    a.q.order = H.d_s_order.p;
    a.q.act_slots = H.sel_act.p;
    a.q.nact = 1;
    static const char* sel_sched = getenv("PINLA_SELINV_SCHED");
    a.q.fifo = (sel_sched && sel_sched[0] == 's') ? 0 : 1;
    a.q.fqueue = H.fq.p;
    a.q.hot = getenv("PINLA_SELINV_NOCONT") ? nullptr : H.d_s_hot.p;
    a.q.ready0 = H.d_s_ready0.p;
    a.q.nready0 = (int)A.s_ready0.size();
    a.trace = nullptr;
    static const char* sel_trace = getenv("PINLA_TRACE_SELINV");
    unsigned long long* tb = nullptr;
    const size_t nt4 = A.selinv_tasks.size() * 4;
    if (sel_trace) {
      CK(cudaMalloc(&tb, nt4 * 8));
      CK(cudaMemsetAsync(tb, 0, nt4 * 8, H.st));
      a.trace = tb;
    }
    CK(launch_selinv(a, H.st));
    if (tb) {
      std::vector<unsigned long long> hb(nt4);
      CK(cudaMemcpyAsync(hb.data(), tb, nt4 * 8, cudaMemcpyDeviceToHost, H.st));
      CK(cudaStreamSynchronize(H.st));
      cudaFree(tb);
      FILE* fp = fopen(sel_trace, "wb");
      if (fp) {
        int64_t nt = (int64_t)A.selinv_tasks.size();
        fwrite(&nt, 8, 1, fp);
        fwrite(hb.data(), 8, hb.size(), fp);
        std::vector<int32_t> info(2 * nt);  // (npairs, kind: 0 inner,1 last-off,2 last-diag,3 group)
        for (int64_t i = 0; i < nt; ++i) {
          if (i >= A.s_nchunk) { info[2*i] = (int)(A.s_grp_rng[i - A.s_nchunk + 1] - A.s_grp_rng[i - A.s_nchunk]); info[2*i+1] = 3; continue; }
          const int t = A.s_chunk_tile[i];
          info[2 * i] = (int)(A.s_chunk_rng[i + 1] - A.s_chunk_rng[i]);
          info[2 * i + 1] = (A.s_chunk_flags[i] & 2) ? (A.tile_row[t] == A.tile_col[t] ? 2 : 1) : 0;
        }
        fwrite(info.data(), 4, info.size(), fp);
        // successor lists and the (I, J) tile of every task (critical-path replay)
        const int64_t ns = (int64_t)A.s_succ.size();
        fwrite(&ns, 8, 1, fp);
        fwrite(A.s_succ_ptr.data(), 4, A.s_succ_ptr.size(), fp);
        fwrite(A.s_succ.data(), 4, A.s_succ.size(), fp);
        std::vector<int32_t> ij(2 * nt);
        for (int64_t i = 0; i < nt; ++i) {
          const int t = i >= A.s_nchunk ? A.s_grp_tile[i - A.s_nchunk] : A.s_chunk_tile[i];
          ij[2 * i] = A.tile_row[t];
          ij[2 * i + 1] = A.tile_col[t];
        }
        fwrite(ij.data(), 4, ij.size(), fp);
        fclose(fp);
      }
    }
    CK(launch_selinv_diag(H.Sg.p, A.nT, A.NT, H.d_colptr.p, H.b.p, H.st));
    H.launches += 3;
    H.n_selinv++;
  }
  std::vector<double> vp(npad);
  d2h(vp.data(), H.b.p, npad, H.st);
  CK(cudaStreamSynchronize(H.st));
  flush_timers(H);
  if (var_out) to_orig(H, vp.data(), var_out);
}

int pinla_selinv_diag(pinla_handle* ph, const double* theta, const double* warm, double* var_out,
                      double* x_out, int32_t* status_out, int64_t* badcol_out) {
  API_BEGIN
  Handle& H = ph->h;
  CK(cudaSetDevice(H.device));
  std::vector<SlotOut> out;
  mode_batch(H, 1, theta, warm, out);
  if (status_out) *status_out = out[0].status;
  if (badcol_out) *badcol_out = out[0].badcol;
  const int64_t npad = H.an.npad();
  if (x_out) {
    std::vector<double> xp(npad);
    d2h(xp.data(), H.x.p, npad, H.st);
    CK(cudaStreamSynchronize(H.st));
    to_orig(H, xp.data(), x_out);
  }
  if (out[0].status != PINLA_OK) return 0;
  selinv_slot0(H, var_out);
  API_END
}

int pinla_selinv_resident(pinla_handle* ph, double* var_out) {
  API_BEGIN
  Handle& H = ph->h;
  CK(cudaSetDevice(H.device));
  selinv_slot0(H, var_out);
  API_END
}

int pinla_solve_resident(pinla_handle* ph, const double* b, double* x_out) {
  API_BEGIN
  Handle& H = ph->h;
  CK(cudaSetDevice(H.device));
  const int64_t npad = H.an.npad();
  std::vector<double> bp(npad, 0.0);
  for (int64_t i = 0; i < H.n; ++i) bp[H.an.pad_of_orig[i]] = b[i];
  h2d(H.b.p, bp.data(), npad, H.st);
  std::vector<int> act(H.S, 0);
  act[0] = 1;
  set_active(H, act);
  run_solve(H, H.b.p, H.delta.p, H.S);
  d2h(bp.data(), H.delta.p, npad, H.st);
  CK(cudaStreamSynchronize(H.st));
  to_orig(H, bp.data(), x_out);
  API_END
}

int pinla_factor_logdet(pinla_handle* ph, const double* qvals, double* logdet_out,
                        int32_t* status_out, int64_t* badcol_out) {
  API_BEGIN
  Handle& H = ph->h;
  CK(cudaSetDevice(H.device));
  // reorder caller values (original CSC order) into tile order
  Analysis& A = H.an;
  std::vector<int64_t> etid(H.nq);
  std::vector<double> qt(H.nq);
  // rebuild the same ordering as build(): sort by (tid, loc)
  std::vector<std::pair<std::pair<int64_t, int64_t>, int64_t>> key(H.nq);
  for (int64_t c = 0; c < H.n; ++c)
    for (int64_t p = H.c_indptr[c]; p < H.c_indptr[c + 1]; ++p) {
      int64_t r = H.c_indices[p];
      int64_t pr = A.iperm[r], pc = A.iperm[c];
      int64_t PR = A.pad_of_perm(std::max(pr, pc)), PC = A.pad_of_perm(std::min(pr, pc));
      key[p] = {{A.tid_of((int32_t)(PR / TB), (int32_t)(PC / TB)), (PR % TB) * TB + PC % TB}, p};
    }
  std::sort(key.begin(), key.end());
  for (int64_t i = 0; i < H.nq; ++i) qt[i] = qvals[key[i].second];
  h2d(H.qv.p, qt.data(), H.nq, H.st);
  std::vector<int> act(H.S, 0);
  act[0] = 1;
  set_active(H, act);
  run_factor(H, H.qv.p, H.S);
  int st0;
  double ld;
  d2h(&st0, H.status.p, 1, H.st);
  d2h(&ld, H.ldsum.p, 1, H.st);
  CK(cudaStreamSynchronize(H.st));
  if (status_out) *status_out = st0 == INT_MAX ? PINLA_OK : PINLA_NOT_PD;
  if (badcol_out) *badcol_out = st0 == INT_MAX ? -1 : A.perm[st0];
  if (logdet_out) *logdet_out = 2.0 * ld;
  API_END
}

// entries of the resident factor / selected inverse at permuted (row, col)
// positions (row >= col): which 0 = L of slot `slot`, 1 = Sigma of the last
// selected inversion; positions outside the tile pattern read 0
int pinla_tile_entries(pinla_handle* ph, int32_t which, int32_t slot, int64_t k,
                       const int64_t* rows, const int64_t* cols, double* out) {
  API_BEGIN
  Handle& H = ph->h;
  CK(cudaSetDevice(H.device));
  Analysis& A = H.an;
  if (which != 0 && which != 1) throw std::runtime_error("which must be 0 (L) or 1 (Sigma)");
  const int S = which == 0 ? H.S : H.Ssel;
  if (slot < 0 || slot >= S) throw std::runtime_error("slot out of range");
  std::vector<int64_t> idx(std::max<int64_t>(k, 1));
  par_for(k, [&](int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      const int64_t r = rows[i], c = cols[i];
      if (r < c || c < 0 || r >= H.n) throw std::runtime_error("entries must satisfy 0 <= col <= row < n");
      const int64_t PR = A.pad_of_perm(r), PC = A.pad_of_perm(c);
      const int64_t tid = A.tid_of((int32_t)(PR / TB), (int32_t)(PC / TB));
      idx[i] = tid < 0 ? -1 : (((int64_t)slot * A.nT + tid) * TB + PR % TB) * TB + PC % TB;
    }
  });
  DBuf<int64_t> d_idx;
  DBuf<double> d_out;
  d_idx.upload(idx, nullptr);
  d_out.alloc(std::max<int64_t>(k, 1), nullptr);
  vk_gather(which == 0 ? H.L.p : H.Sg.p, d_idx.p, k, d_out.p, H.st);
  d2h(out, d_out.p, k, H.st);
  CK(cudaStreamSynchronize(H.st));
  API_END
}

// Q_c values of slot `slot` (the last assembled conditional precision: after
// pinla_mode, the one factorized at the returned mode) in the original-order
// lower-CSC pattern of pinla_cond_pattern
int pinla_cond_values(pinla_handle* ph, int32_t slot, double* out) {
  API_BEGIN
  Handle& H = ph->h;
  CK(cudaSetDevice(H.device));
  if (slot < 0 || slot >= H.S) throw std::runtime_error("slot out of range");
  std::vector<int64_t> idx(H.nq);
  for (int64_t p = 0; p < H.nq; ++p) idx[p] = (int64_t)slot * H.nq + H.q_newpos[p];
  DBuf<int64_t> d_idx;
  DBuf<double> d_out;
  d_idx.upload(idx, nullptr);
  d_out.alloc(std::max<int64_t>(H.nq, 1), nullptr);
  vk_gather(H.qv.p, d_idx.p, H.nq, d_out.p, H.st);
  d2h(out, d_out.p, H.nq, H.st);
  CK(cudaStreamSynchronize(H.st));
  API_END
}

// y = L x with the resident factor of slot `slot`, both in the PERMUTED order
// (factor coordinates): the building block of sample_gmrf (L^-T z = Q^-1 L z)
int pinla_factor_lmul(pinla_handle* ph, int32_t slot, const double* x, double* y) {
  API_BEGIN
  Handle& H = ph->h;
  CK(cudaSetDevice(H.device));
  Analysis& A = H.an;
  if (slot < 0 || slot >= H.S) throw std::runtime_error("slot out of range");
  const int64_t npad = A.npad();
  std::vector<double> xp(npad, 0.0), yp(npad);
  for (int64_t i = 0; i < H.n; ++i) xp[A.pad_of_perm(i)] = x[i];
  DBuf<double> dx, dy;
  dx.upload(xp, nullptr);
  dy.alloc(npad, nullptr);
  vk_tile_lmv(H.L.p + (size_t)slot * A.nT * TB * TB, A.NT, H.d_rowptr.p, H.d_row_col.p,
              H.d_row_tid.p, dx.p, dy.p, H.st);
  H.launches++;
  d2h(yp.data(), dy.p, npad, H.st);
  CK(cudaStreamSynchronize(H.st));
  for (int64_t i = 0; i < H.n; ++i) y[i] = yp[A.pad_of_perm(i)];
  API_END
}

int pinla_cond_pattern(pinla_handle* ph, int64_t* nnz_out, int64_t* indptr_out,
                       int64_t* indices_out) {
  API_BEGIN
  Handle& H = ph->h;
  if (nnz_out) *nnz_out = H.nq;
  if (indptr_out) std::copy(H.c_indptr.begin(), H.c_indptr.end(), indptr_out);
  if (indices_out) std::copy(H.c_indices.begin(), H.c_indices.end(), indices_out);
  API_END
}

int pinla_stats(pinla_handle* ph, pinla_stats_t* o) {
  API_BEGIN
  Handle& H = ph->h;
  flush_timers(H);
  o->n_evaluations = H.n_evals;
  o->n_factorizations = H.n_factor;
  o->n_solves = H.n_solve;
  o->n_selinv = H.n_selinv;
  o->nnz_cond = H.nq;
  o->n_tiles = H.an.nT;
  o->n_tile_rows = H.an.NT;
  o->factor_flops = H.an.factor_flops;
  o->selinv_flops = H.an.selinv_flops;
  o->solve_bytes = H.an.solve_bytes;
  o->assemble_bytes = H.asm_bytes[0] + H.asm_bytes[H.family == PINLA_FAMILY_POISSON ? 2 : 1];
  o->device_bytes = H.device_bytes;
  o->analyze_s = H.analyze_s;
  o->kernel_launches = H.launches;
  o->factor_launches = H.n_factor;
  o->factor_slot_runs = H.factor_slot_runs;
  o->solve_slot_runs = H.solve_slot_runs;
  o->factor_ms = H.t_factor;
  o->solve_ms = H.t_solve;
  o->assemble_ms = H.t_assemble;
  o->selinv_ms = H.t_selinv;
  o->last_call_ms = H.last_call_ms;
  o->factor_flops_limited = H.an.factor_flops_limited;
  o->slots = H.S;
  o->solve_kernel_ms = H.t_solvek;
  o->assemble_bytes_done = H.asm_bytes_done;
  o->selinv_launches = H.n_selinv;
  API_END
}

void pinla_reset_stats(pinla_handle* ph) {
  Handle& H = ph->h;
  flush_timers(H);
  H.n_evals = H.n_factor = H.n_solve = H.n_selinv = H.launches = 0;
  H.factor_slot_runs = H.solve_slot_runs = 0;
  H.t_assemble = H.t_factor = H.t_solve = H.t_selinv = H.t_other = 0;
  H.t_solvek = 0;
  H.asm_bytes_done = 0;
}

int pinla_phase_times(pinla_handle* ph, double* a, double* f, double* s, double* si, double* o) {
  Handle& H = ph->h;
  flush_timers(H);
  if (a) *a = H.t_assemble;
  if (f) *f = H.t_factor;
  if (s) *s = H.t_solve;
  if (si) *si = H.t_selinv;
  if (o) *o = H.t_other;
  return 0;
}

}  // extern "C"
