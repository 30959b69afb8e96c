/*
 * pinla.h — C-ABI of the B200 engine for the INLA hyperparameter objective
 * f(theta) and the Takahashi selected inversion that follows it.
 *
 * Plain C types only (pointers + sizes), no torch / CUDA types in any
 * signature.  All host buffers are caller-owned; device workspaces are
 * library-owned per handle and preallocated at create time for `max_slots`
 * concurrent theta slots.
 *
 * Each entry point replaces one reference interface
 * (/root/reference/pkg/src/parinla/...):
 *
 *   pinla_create        ObjectiveEvaluator.__init__        objective.py:112-173
 *                       (design, prior plan, Gram pair map, union pattern,
 *                        one-time symbolic analysis  = analyze() cholesky.py:88-137)
 *   pinla_eval_batch    [ObjectiveEvaluator.eval_objective objective.py:298-331]
 *                       x k slots as issued by run_batch   runtime.py:134-177
 *                       from fd_gradient / parallel_line_search
 *                       optimizer.py:92-140, 291-346
 *   pinla_mode          ObjectiveEvaluator.gaussian_approx objective.py:218-296
 *   pinla_selinv_diag   selected_inverse(...).marginal_variances
 *                       cholesky.py:356-400 (+ the factorization that feeds it)
 *   pinla_factor_logdet factorize(...).log_det              cholesky.py:282-322
 *                       on caller-supplied Q values (test / drop-in use)
 *   pinla_stats         ObjectiveEvaluator.stats            objective.py:180-188
 *
 * Status codes (per slot): PINLA_OK, PINLA_NOT_PD (column in the ORIGINAL
 * latent order in badcol, errors.py:22-31), PINLA_INNER_DIVERGENCE
 * (errors.py:34-42).  A failing slot never aborts the others.  Function
 * return values: 0 on success, negative on an engine error (message via
 * pinla_last_error()).
 */
#ifndef PINLA_H
#define PINLA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PINLA_OK 0
#define PINLA_NOT_PD 1
#define PINLA_INNER_DIVERGENCE 2

#define PINLA_FAMILY_GAUSSIAN 0
#define PINLA_FAMILY_POISSON 1

/* analytic log det Q_prior(theta) terms (lattice / AR(1) models) */
#define PINLA_LD_CONST 0   /* value                                            */
#define PINLA_LD_SPDE 1    /* nx*ny*log tau + 2 sum log(kappa^2 + lam_j + mu_k)  */
#define PINLA_LD_ST 2      /* n_s logdet Q_AR1(rho) + n_t logdet Q_spde        */
#define PINLA_LD_AR1 3     /* nt*log tau + logdet Q_AR1(rho)                   */

/* gain kinds of the prior plan (value = sum_t coef_t * gain[gain_t] + const) */
#define PINLA_GAIN_EXP 0   /* exp(theta[k])                                  */
#define PINLA_GAIN_SPDE 1  /* (tau k^4, 2 tau k^2, tau)[sub], theta[k..k+1]  */
#define PINLA_GAIN_AR1 2   /* exp(theta[k]) * ar1(logit rho = theta[k+1])[sub] */
#define PINLA_GAIN_ST 3    /* ar1(theta[k+2])[sub/3] * spde(theta[k],theta[k+1])[sub%3] */

typedef struct pinla_model {
  int64_t n;       /* latent dimension                                  */
  int64_t m;       /* observations                                      */
  int32_t d;       /* dim(theta)                                        */
  int32_t family;  /* PINLA_FAMILY_*                                    */
  int32_t noise_theta;      /* gaussian: theta index of log tau_y, or -1   */
  double noise_precision;   /* gaussian with fixed noise                   */
  /* prior plan, lower CSC in ORIGINAL latent order (model.py:231-282)   */
  const int64_t* p_indptr;  /* n+1 */
  const int64_t* p_indices; /* nnz_p, diagonal first, rows ascending     */
  int64_t n_terms;
  const int64_t* term_entry; /* n_terms, sorted by (entry, gain)          */
  const int32_t* term_gain;  /* n_terms */
  const double* term_coef;   /* n_terms */
  const double* p_const;     /* nnz_p  (jitter / fixed-effect precision)  */
  int32_t n_gains;
  const int32_t* gain_kind;  /* n_gains, PINLA_GAIN_*                     */
  const int32_t* gain_theta; /* n_gains, first theta index               */
  const int32_t* gain_sub;   /* n_gains                                  */
  /* design A (m x n CSR, original column order, model.py:334-356)        */
  const int64_t* a_indptr;
  const int64_t* a_indices;
  const double* a_data;
  const double* y;         /* m */
  const double* offsets;   /* m */
  const double* exposures; /* m */
  const double* hyper_shape; /* d */
  const double* hyper_rate;  /* d */
  /* fill-reducing ordering chosen by the host: perm[new] = old; the last
   * n_dense entries are dense vertices (fixed effects) forming the arrow */
  const int64_t* perm;
  int64_t n_dense;
  /* optional tile partition of the permuted index range (boundaries,
   * n_tile_bounds = NT+1 entries, each tile <= 64 rows; tiles must not
   * straddle the dense tail).  NULL: 64-row tiles + arrow tiles.        */
  const int64_t* tile_bounds;
  int64_t n_tile_bounds;
  /* optional closed-form log det Q_prior(theta) (0 terms: factorize Q_prior
   * like the reference, objective.py:308).  Lattice eigenvalues are the
   * Neumann path-graph ones, 2 - 2 cos(pi j / n). */
  int32_t n_logdet_terms;
  const int32_t* ld_kind;   /* PINLA_LD_*                                  */
  const int32_t* ld_theta;  /* first theta index of the term              */
  const int64_t* ld_dims;   /* 3 per term: nx, ny, nt                      */
  const double* ld_value;   /* PINLA_LD_CONST value                        */
} pinla_model;

typedef struct pinla_options {
  int32_t max_slots;  /* concurrent theta slots resident on the device   */
  int32_t max_inner;  /* Newton cap (objective.py:120, default 50)       */
  double inner_tol;   /* Newton tolerance (objective.py:119, 1e-8)        */
  int32_t device;     /* CUDA device ordinal                             */
  int32_t selinv_slots; /* slots with selected-inversion storage (>=1)   */
  int32_t analytic_prior_logdet; /* 1: use the model's closed-form terms  */
} pinla_options;

typedef struct pinla_handle pinla_handle;

typedef struct pinla_stats_t {
  int64_t n_evaluations;
  int64_t n_factorizations;
  int64_t n_solves;
  int64_t n_selinv;
  int64_t nnz_cond;        /* nnz of the lower conditional pattern          */
  int64_t n_tiles;         /* tiles in the factor's tile pattern            */
  int64_t n_tile_rows;     /* NT                                            */
  int64_t factor_flops;    /* algorithmic flops of one tile factorization   */
  int64_t selinv_flops;    /* algorithmic flops of one tile selinv          */
  int64_t solve_bytes;     /* algorithmic bytes of one forward+backward solve */
  int64_t assemble_bytes;  /* algorithmic bytes of one slot's Q_c assembly  */
  int64_t device_bytes;    /* device memory held by the handle              */
  double analyze_s;        /* wall time of the one-time analysis            */
  int64_t kernel_launches; /* kernels launched since create / reset         */
  int64_t factor_launches; /* factorization kernel launches since reset      */
  int64_t factor_slot_runs;/* sum over those launches of active slots        */
  int64_t solve_slot_runs; /* sum over solve launches of active slots        */
  double factor_ms;        /* device time in factorization launches (events) */
  double solve_ms;         /* device time in solve launches                  */
  double assemble_ms;      /* device time in assembly kernels                */
  double selinv_ms;        /* device time in selected-inversion launches     */
  double last_call_ms;     /* device time of the last eval/mode/selinv call  */
  int64_t factor_flops_limited; /* flops one factorization's kernels execute  */
  int64_t slots;           /* theta slots resident on the device: max_slots,
                              reduced at create to what device memory holds */
  double solve_kernel_ms;  /* device time in solve_kernel launches only      */
  int64_t assemble_bytes_done; /* algorithmic bytes of the assembly kernels
                              launched since reset (active slots x bytes)   */
  int64_t selinv_launches; /* selected-inversion launches since reset       */
} pinla_stats_t;

/* one-time: analysis + upload; returns 0 or a negative error code */
int pinla_create(const pinla_model* model, const pinla_options* opt, pinla_handle** out);
void pinla_destroy(pinla_handle* h);

/* f(theta) for k points (thetas: k x d, row-major).  warm: n (original
 * order) or NULL — the accepted-iterate warm start (fit.py:94-113); used by
 * the poisson Newton loop only, like the reference (objective.py:246-259).
 * comps_out (k x 5): f, log_prior_hyper, log_prior_latent, log_likelihood,
 * log_gaussian_approx.  logdets_out (k x 2): log det Q_c, log det Q_prior.
 * modes_out (k x n): the conditional modes x*(theta) in original order.
 * Any output pointer may be NULL. */
int pinla_eval_batch(pinla_handle* h, int32_t k, const double* thetas, const double* warm,
                     double* f_out, double* comps_out, int32_t* status_out, int64_t* badcol_out,
                     int32_t* iters_out, double* logdets_out, double* modes_out /* k x n */);

/* pinla_eval_batch with one warm start per point (warms: k x n, original
 * order) — the reference's per-point eval_objective(theta, warm_start)
 * (objective.py:298-304) batched; used for sensitivity-extrapolated starts
 * x*(theta_acc) + D (theta - theta_acc) (fit.py FitObjective). */
int pinla_eval_batch_warm(pinla_handle* h, int32_t k, const double* thetas, const double* warms,
                          double* f_out, double* comps_out, int32_t* status_out,
                          int64_t* badcol_out, int32_t* iters_out, double* logdets_out,
                          double* modes_out /* k x n */);

/* conditional mode x*(theta) (original order) and its Newton iteration
 * count; leaves the conditional factor resident in slot 0 */
int pinla_mode(pinla_handle* h, const double* theta, const double* warm, double* x_out,
               int32_t* iters_out, int32_t* status_out, int64_t* badcol_out, double* logdet_out);

/* marginal variances diag(Q_c(theta)^-1) in original order (and the mode) */
int pinla_selinv_diag(pinla_handle* h, const double* theta, const double* warm, double* var_out,
                      double* x_out, int32_t* status_out, int64_t* badcol_out);

/* factorize caller-supplied conditional-pattern values (lower CSC in the
 * ORIGINAL order, same pattern as pinla_cond_pattern) -> log det */
int pinla_factor_logdet(pinla_handle* h, const double* qvals, double* logdet_out,
                        int32_t* status_out, int64_t* badcol_out);

/* solve Q x = b with the factor resident in slot 0 (the last
 * pinla_factor_logdet / pinla_mode call); b, x in original order
 * (solve(), cholesky.py:325-336) */
int pinla_solve_resident(pinla_handle* h, const double* b, double* x_out);

/* marginal variances of the factor resident in slot 0, original order
 * (selected_inverse(), cholesky.py:356-400) */
int pinla_selinv_resident(pinla_handle* h, double* var_out);

/* the lower-CSC conditional pattern (original order): sizes then arrays */
int pinla_cond_pattern(pinla_handle* h, int64_t* nnz_out, int64_t* indptr_out /* n+1 or NULL */,
                       int64_t* indices_out /* nnz or NULL */);

/* drop-in payloads (reference hot-path types), read from the
 * device on request:
 * pinla_tile_entries: entries (rows[i], cols[i]), PERMUTED indices with
 *   row >= col, of the resident factor L of slot `slot` (which = 0; replaces
 *   CholeskyFactor.values, cholesky.py:168-190) or of the last selected
 *   inverse Sigma (which = 1; SelectedInverse.values, cholesky.py:193-214);
 *   positions outside the tile pattern read 0.
 * pinla_cond_values: the conditional precision Q_c last assembled in slot
 *   `slot` (after pinla_mode: at the returned mode) on the pattern of
 *   pinla_cond_pattern (GaussianApprox.cond_precision, objective.py:39-50).
 * pinla_factor_lmul: y = L x with slot `slot`'s factor, permuted order (with
 *   pinla_solve_resident: sample_gmrf's L^-T z = Q^-1 (L z), cholesky.py:339-353). */
int pinla_tile_entries(pinla_handle* h, int32_t which, int32_t slot, int64_t k, const int64_t* rows,
                       const int64_t* cols, double* out);
int pinla_cond_values(pinla_handle* h, int32_t slot, double* out);
int pinla_factor_lmul(pinla_handle* h, int32_t slot, const double* x, double* y);

int pinla_stats(pinla_handle* h, pinla_stats_t* out);
void pinla_reset_stats(pinla_handle* h);

/* timing of the last eval/selinv call's phases on the device (ms) */
int pinla_phase_times(pinla_handle* h, double* assemble_ms, double* factor_ms, double* solve_ms,
                      double* selinv_ms, double* other_ms);

/* host-only tile symbolic analysis of a lower-CSC pattern (no GPU needed):
 * the structure numbers an ordering produces (used by tests and by the
 * host to compare orderings).  tile_rows_out / tile_cols_out (nT each) may
 * be NULL; call once with NULL to get nT. */
typedef struct pinla_analysis_info {
  int64_t n_tile_rows;      /* NT                                        */
  int64_t n_tiles;          /* nT: tiles in the pattern of L             */
  int64_t n_update_pairs;   /* tile GEMMs of one factorization           */
  int64_t factor_flops;
  int64_t selinv_flops;
  int64_t solve_bytes;
  int64_t depth_forward;    /* longest tile-column dependency chain      */
  int64_t depth_backward;
  int64_t factor_flops_limited; /* flops executed by the row/col-limited kernels */
} pinla_analysis_info;
int pinla_analyze_pattern(int64_t n, const int64_t* indptr, const int64_t* indices,
                          const int64_t* perm, int64_t n_dense, const int64_t* tile_bounds,
                          int64_t n_tile_bounds, pinla_analysis_info* out,
                          int32_t* tile_rows_out, int32_t* tile_cols_out);

/* scalar symbolic factorization of a lower-CSC pattern under perm (host
 * only; the reference's analyze pattern, cholesky.py:88-165): call with
 * Lp_out = Li_out = NULL for *nnz_out, then with Lp_out[n+1], Li_out[nnz]
 * (per column: diagonal first, rows ascending; permuted indices). */
int pinla_scalar_pattern(int64_t n, const int64_t* indptr, const int64_t* indices,
                         const int64_t* perm, int64_t* nnz_out, int64_t* Lp_out, int64_t* Li_out);

/* nested-dissection ordering of a symmetric pattern (lower CSC, original
 * order), host only: the reference's ordering.py:206-423 (dense peel, BFS
 * level-set separators, separator shrinking, minimum-degree leaves) restated
 * natively — the permutation equals the reference's nested_dissection_order
 * (replaces ordering.py:206-274 + cholesky.py:88-137's ordering step).
 * perm_out[n] (new -> old); *n_dense_out = dense vertices peeled to the end;
 * tile_bounds_out[<= n + 1] (NULL: skipped) = separator-aligned tile starts
 * of height <= tile_max for pinla_model.tile_bounds, count in *n_bounds_out;
 * node arrays (<= n + 1 entries each, NULL: skipped) = the separator tree in
 * the reference's node order, count in *n_nodes_out. */
int pinla_nd_order(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t leaf_cutoff,
                   int64_t tile_max, int64_t* perm_out, int64_t* n_dense_out,
                   int64_t* tile_bounds_out, int64_t* n_bounds_out, int64_t* node_start,
                   int64_t* node_end, int64_t* node_parent, int64_t* n_nodes_out);

const char* pinla_last_error(void);
const char* pinla_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PINLA_H */
