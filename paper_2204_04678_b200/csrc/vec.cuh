// Device-resident model data for the vector kernels + launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pinla {

constexpr int kRedBlocks = 1184;  // max reduction partials (8 per SM); per model: VecModel::nred

struct VecModel {
  int64_t m = 0, npad = 0, nnz_p = 0, nq = 0, nch = 0;
  int family = 0, n_gains = 0;
  // reduction partials of the m- / npad-long sums: fixed per model (=>
  // deterministic), 296 .. kRedBlocks by size (one block per ~4k elements)
  int nred = 296;
  // prior plan (terms CSR by entry)
  const int64_t* term_ptr = nullptr;
  const int* term_gain = nullptr;
  const double* term_coef = nullptr;
  const double* pconst = nullptr;
  // conditional values in tile order
  const int64_t* psrc = nullptr;
  const int64_t* gptr = nullptr;
  const int* gobs = nullptr;
  const double* gcoef = nullptr;
  const double* gunit = nullptr;
  // pair layout of gram_chunk_kernel (engine.cu build): chunk positions in
  // length order, 32 per group, pair k of position 32 g + l at gbase[g] + 32 k + l
  int64_t gpos = 0;
  const int64_t* gbase = nullptr;
  const uint8_t* clen = nullptr;
  const int32_t* cperm = nullptr;  // position -> chunk id
  int64_t ngch = 0;                 // Gram chunks (each within one entry)
  const int64_t* gch_beg = nullptr;  // [ngch+1] pair ranges
  const int64_t* e_ch = nullptr;     // [nq+1] chunk range per entry
  int64_t nheavy = 0;                // entries with many chunks (fixed-effect pairs)
  const int64_t* heavy = nullptr;    // [nheavy] entry ids, reduced in parts
  int64_t nhp = 0;                   // parts of <= kHeavyPart chunks over all heavy entries
  const int64_t* hpart_ptr = nullptr;  // [nheavy+1]
  const int64_t* hp_c0 = nullptr;    // [nhp] chunk range of each part
  const int64_t* hp_c1 = nullptr;
  double* hbuf = nullptr;            // [S][nhp] part sums (scratch)
  int64_t nheavy_rows = 0;           // A^T rows with many chunks (dense design columns)
  const int64_t* heavy_rows = nullptr;
  // design
  const int64_t* ap = nullptr;
  const int* aj = nullptr;
  const double* ax = nullptr;
  const int* ch_row = nullptr;
  const int64_t* ch_beg = nullptr;  // [nch+1]
  const int* at_obs = nullptr;
  const double* at_val = nullptr;
  const int64_t* row_ch = nullptr;  // [npad+1]
  // likelihood data
  const double* y = nullptr;
  const double* off = nullptr;
  const double* logE = nullptr;
  const double* E = nullptr;
  // prior symmetric CSR over padded rows
  const int64_t* qp = nullptr;
  const int* qj = nullptr;
  const int64_t* qvi = nullptr;
};

void vk_prior_values(const VecModel& M, const double* gains, double* pv, const int* active, int S,
                     cudaStream_t st);
constexpr int64_t kGramChunk = 16;
constexpr int64_t kHeavyChunks = 32;  // entries / A^T rows with more chunks are reduced block-wise
constexpr int64_t kHeavyPart = 2048;  // chunks per block-reduced part of a heavy entry
void vk_cond_values(const VecModel& M, const double* pv, const double* tau, const double* w,
                    int mode, double* qv, double* gch_out, const int* active, int S,
                    cudaStream_t st);
void vk_spmv_A(const VecModel& M, const double* x, double* eta, const int* active, int S,
               cudaStream_t st);
void vk_lik(const VecModel& M, const double* eta, const double* tau, double* d1, double* w,
            double* parts, const int* active, int S, cudaStream_t st);
void vk_AT(const VecModel& M, const double* d1, const double* sub, double* out, double* ch_out,
           const int* active, int S, cudaStream_t st);
void vk_symv(const VecModel& M, const double* pv, const double* x, double* qx, const int* active,
             int S, cudaStream_t st);
// slots with sel[s] = t >= 0 take halving try t (buffers [t][S][..]) as the iterate
void vk_take_try(int64_t npad, int64_t m, int S, const int* sel, const double* tx, const double* tqx,
                 const double* teta, const double* td1, const double* tw, double* x, double* qx,
                 double* eta, double* d1, double* w, cudaStream_t st);
// per-slot [sum of likelihood-term differences, (x_t - x)^T Qp (x_t + x)] partials
void vk_gdiff(const VecModel& M, const double* eta, const double* eta_t, const double* tau,
              const double* x, const double* x_t, const double* qx, const double* qx_t,
              double* parts, const int* active, int S, cudaStream_t st);
void vk_dot_max(const VecModel& M, const double* a, const double* b, double* parts,
                const int* active, int S, cudaStream_t st);
void vk_reduce(const double* parts, int nblk, int wdt, int maxmask, double* out, const int* active,
               int S, cudaStream_t st);
void vk_axpy(int64_t npad, const double* x, const double* d, const double* alpha, double* y,
             const int* active, int S, cudaStream_t st);
void vk_scale(int64_t npad, const double* x, const double* alpha, double* y, const int* active,
              int S, cudaStream_t st);

void vk_gather(const double* src, const int64_t* idx, int64_t k, double* out, cudaStream_t st);
void vk_tile_lmv(const double* L, int NT, const int* rowptr, const int* row_col, const int* row_tid,
                 const double* x, double* y, cudaStream_t st);
}  // namespace pinla
