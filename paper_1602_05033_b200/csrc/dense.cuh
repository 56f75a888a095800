// Dense symmetric eigensolver and SVD of the finalisation (see dense.cu).
#pragma once
#include "kry_internal.cuh"

namespace kry {

// Symmetric eigendecomposition in place: A (k x k, symmetric, column-major)
// -> eigenvectors in the columns of A, eigenvalues ascending in w (device).
// sweeps (optional, host) receives the number of Jacobi sweeps.
// semidefinite: the caller knows the spectrum has one sign (no shift; keeps
// the absolute accuracy eps ||A|| of the small eigenvalues of a PSD matrix);
// otherwise an indefinite matrix is shifted by its upper Gershgorin bound.
int dense_syev(cudaStream_t st, double* A, int k, double* w, int* sweeps = nullptr,
               bool semidefinite = false);

// Thin SVD: A (M x N column-major, leading dimension M; any M, N >= 1)
// = U diag(sig) VT with sig descending (device, N values), U M x N
// (column-major, ld M) and VT N x N (column-major, ld N: row i = v_i^T).
// A is overwritten.
int dense_gesvd(cudaStream_t st, double* A, int M, int N, double* sig, double* U, double* VT,
                int* sweeps = nullptr);

// C (M x N, row-major, ldc) = A (M x K) B (K x N, row-major, ldb);
// A row-major (lda) or, with a_colmajor, column-major (element (i, k) at
// A[k lda + i]).  brow / crow (nullable): row index maps of B and C.
// dyn (nullable, device): the inner dimension K = dyn[0] and M = dyn[0] + 1
// are read on the device (M, K passed are upper bounds).
int dense_gemm(cudaStream_t st, int M, int N, int K, const double* A, int64_t lda, int a_colmajor,
               const double* B, int64_t ldb, const int* brow, double* C, int64_t ldc,
               const int* crow, const int* dyn = nullptr);

// Pivoted Cholesky M ~ L L^T of M_ij = (a_i . a_j) / |lam_i + lam_j| (a: k x 8
// row-major slots, s columns used; lam all of one sign): L row-major k x ldl,
// at most pmax columns; *p_host = number of columns (stops at the rounding
// level of the largest diagonal entry).
int dense_pchol_cauchy(cudaStream_t st, const double* a, const double* lam, int k, int s,
                       double* L, int ldl, int pmax, int* p_host);

// Cross factorisation R ~ Lf Uf by Gaussian elimination with complete
// pivoting, stopped at the rounding level (R ma x nb column-major, destroyed;
// Lf ma x pmax column-major; Uf pmax x nb row-major); *p_host = rank used, or
// > pmax when the matrix did not reach the rounding level within pmax steps.
int dense_gecp(cudaStream_t st, double* R, int ma, int nb, double* Lf, double* Uf, int pmax,
               int* p_host);
// Thin SVD of Lf Uf (both destroyed): sig (p, descending), left (ma x p) and
// right (nb x p), column-major with orthonormal columns.
int dense_svd_product(cudaStream_t st, double* Lf, int ma, double* Uf, int nb, int p, double* sig,
                      double* left, double* right);

}  // namespace kry
