// Incremental eigen engine for the growing block-tridiagonal T_m (see eigen.cu).
#pragma once
#include "kry_internal.cuh"

namespace kry {

struct EigView {
  int s;
  int kmax;
  double *lam_old, *lam_new;
  double *F_old, *F_new;   // first s rows of Q, row r at r*kmax
  double *L_old, *L_new;   // last s rows of Q (row r <-> global row K-s+r)
  double *z, *poles, *zz, *zhat, *def_lam, *mu;
  double *org, *tau, *scal;
  int *cand, *dflag, *pflag, *pmap, *def_idx, *counts;
  unsigned* stats;   // KRY_SECULAR_STATS=1: secular iteration histogram (diagnostics)
};

struct EigEngine {
  int s = 0, kmax = 0, K = 0, cur = 0, dev = 0;
  bool deflate_attr = false;
  double* dbuf = nullptr;
  int* ibuf = nullptr;
  unsigned* ticket = nullptr;
  unsigned* cnt = nullptr;     // Cauchy per-x-tile tickets + 1 global
  size_t cnt_cap = 0;
  double *lam[2] = {nullptr, nullptr}, *F[2] = {nullptr, nullptr}, *L[2] = {nullptr, nullptr};
  double *z = nullptr, *poles = nullptr, *zz = nullptr, *zhat = nullptr, *def_lam = nullptr,
         *mu = nullptr;
  double *org = nullptr, *tau = nullptr, *u = nullptr, *w = nullptr, *scal = nullptr,
         *partials = nullptr, *res = nullptr, *vpart = nullptr, *cpart = nullptr;
  size_t cpart_cap = 0;   // x-by-y-chunk entries of cpart
  int *cand = nullptr, *dflag = nullptr, *pflag = nullptr, *pmap = nullptr,
      *def_idx = nullptr, *counts = nullptr;
  unsigned* stats = nullptr;

  int init(int s, int kmax, int device);
  void release();
  EigView view() const;
  void reset() { K = 0; cur = 0; }
  // append block row j: symmetrised diagonal block (8x8 slot) and the
  // coupling block to the previous block (nullptr for the first block)
  int append_block(cudaStream_t st, const double* dsym_blk, const double* sub_prev);
  int compute_uw(cudaStream_t st, const double* gamma, const double* tau_blk);
  int residual_lyap(cudaStream_t st, const double* gamma, const double* tau_blk);
  // grow the Cauchy stage-1 buffer for an nx x ny contraction (one-sided
  // Sylvester: nx = order of the dense side B)
  int ensure_cauchy(int nx, int ny);
  double* cpart_ext = nullptr;
  int cauchy(cudaStream_t st, int nx, const double* lx, const double* ax, int ny,
             const double* ly, const double* by, const double* cy, double* out2);
  const double* lam_cur() const { return lam[cur]; }
  const double* F_cur() const { return F[cur]; }
  const double* L_cur() const { return L[cur]; }
};

// Full eigendecomposition of the block-tridiagonal T_m (block slots dsym,
// sub as in the engine): divide and conquer on the band, lam ascending
// (device, k = s m), Q column-major k x k (device).
int dc_band_eigh(cudaStream_t st, const double* dsym, const double* sub, int s, int m,
                 double* lam, double* Q);

}  // namespace kry
