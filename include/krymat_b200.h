/*
 * krymat_b200.h -- C-ABI of libkrymat_b200.so, the B200 (sm_100a) hot path of
 * the two-pass block-Lanczos solver for symmetric Lyapunov / Sylvester
 * equations  A X + X B + C1 C2^T = 0  (Palitta & Simoncini, arXiv 1602.05033).
 *
 * The reference (`krymat`, pure Python) has no FFI of its own; its plug-in
 * boundary is the Python solver API.  These entry points are what a ctypes /
 * cffi binding of that API binds.  Each one replaces the
 * reference code cited beside it (paths relative to pkg/src/krymat/):
 *
 *   kry_ctx_create        SparseOperator.__init__           operators.py:89-93
 *   kry_apply             SparseOperator.apply              operators.py:95-101
 *   kry_init_basis        init_basis (standard)             basis.py:192-220
 *   kry_lanczos_step      lanczos_step + mgs_twice + QR     basis.py:164-252, kernels.py:134-160
 *   kry_get_projection    ProjectionState blocks            basis.py:131-161
 *   kry_check_lyap        ctri_lyapunov                     residual.py:40-59
 *   kry_check_sylv        ctri_sylvester                    residual.py:62-84
 *   kry_solve_lyap_pass1  solve_lyapunov loop               solvers.py:216-252
 *   kry_solve_sylv_pass1  solve_sylvester_two_sided loop    solvers.py:303-347
 *   kry_finalize_lyap     finalisation + truncated_spd      solvers.py:254-264, kernels.py:309-331
 *   kry_finalize_sylv     finalisation + truncated_svd      solvers.py:349-358, kernels.py:334-345
 *   kry_recover           two_pass_recover (standard)       solvers.py:130-169
 *   kry_partial_eig       partial_eig_blocktridiag          kernels.py:296-306
 *   kry_band_eigh         np.linalg.eigh(T_m.to_dense())       solvers.py:256, :350-351
 *   kry_dense_eigh        np.linalg.eigh (dense symmetric)     kernels.py:316, solvers.py:420
 *   kry_dense_svd         np.linalg.svd (truncated_svd_factor) kernels.py:337
 *   kry_ctri_lyap_blocks  ctri_lyapunov on given blocks     residual.py:40-59
 *   kry_ctri_sylv_blocks  ctri_sylvester on given blocks    residual.py:62-84
 *   kry_true_lyap_residual true_lyapunov_residual          solvers.py:104-115
 *   kry_sylv1_setup       eigh(B), P^T C2 (one-sided)        solvers.py:405-411
 *   kry_check_sylv1       residual_one_sided                 residual.py:87-104
 *   kry_finalize_sylv1    one-sided finalisation + SVD       solvers.py:446-455
 *
 * Conventions: all arithmetic is IEEE fp64.  Host block vectors are row-major
 * n x s (C order, as numpy produces them).  s x s blocks are row-major.  Host
 * buffers are owned by the caller and copied synchronously; the library owns
 * every device allocation.  A context is not re-entrant (one host thread);
 * distinct contexts may be used concurrently.  Every call returns a status
 * code (KRY_OK = 0); kry_last_error() returns the message of the last failure
 * on the calling thread.
 */
#ifndef KRYMAT_B200_H
#define KRYMAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: 1:1 with the reference exception classes (errors.py:4-43) */
enum {
  KRY_OK = 0,
  KRY_ERR_DIMENSION = 1,     /* DimensionMismatchError */
  KRY_ERR_ASYMMETRIC = 2,    /* AsymmetricMatrixError */
  KRY_ERR_DEFLATION = 3,     /* DeflationUnsupportedError */
  KRY_ERR_INDEFINITE = 4,    /* IndefiniteMatrixError */
  KRY_ERR_FACTORIZATION = 5, /* FactorizationError */
  KRY_ERR_RECURRENCE = 6,    /* RecurrenceMismatchError */
  KRY_ERR_CUDA = 7,          /* KrymatError (device failure) */
  KRY_ERR_ARGUMENT = 8,      /* ValueError */
  KRY_ERR_NCCL = 9,          /* KrymatError (collective failure) */
  KRY_ERR_STATE = 10,        /* KrymatError (call out of order) */
  KRY_ERR_CONVERGENCE = 11   /* ConvergenceError (history is still returned) */
};

enum { KRY_OP_STENCIL = 0, KRY_OP_CSR = 1 };

/* Operator description.  A stencil operator is the symmetric 3/5/7-point
 * matrix of a Dirichlet grid (x fastest, then y, then z) whose CSR rows hold
 * the columns {i-nx*ny, i-nx, i-1, i, i+1, i+nx, i+nx*ny} (those inside the
 * grid).  Coefficients are either constant (c_*) or per point:
 *   diag[i] = A[i,i], cx[i] = A[i,i+1], cy[i] = A[i,i+nx], cz[i] = A[i,i+nx*ny]
 * Row sums are accumulated in CSR column order without FMA contraction, so
 * the product equals scipy's csr_matvecs bit for bit.
 * Multi-GPU: a rank owns z-planes [z_begin, z_end) (all planes: 0, nz). */
typedef struct kry_operator_desc {
  int32_t kind;              /* KRY_OP_STENCIL | KRY_OP_CSR */
  int32_t variable;          /* stencil: 0 constant, 1 per-point arrays */
  int64_t n;                 /* rows of the operator (global) */
  int64_t nx, ny, nz;        /* stencil grid (2-D: nz = 1; 1-D: ny = nz = 1) */
  double c_diag, c_x, c_y, c_z;
  const double *diag, *cx, *cy, *cz;   /* host, length n (variable mode) */
  int64_t nnz;                          /* CSR */
  const int64_t *indptr;
  const int32_t *indices;
  const double *values;
  int64_t z_begin, z_end;               /* slab owned by this rank */
} kry_operator_desc;

typedef struct kry_ctx kry_ctx;

/* library / device */
int kry_version(void);
const char *kry_last_error(void);
int kry_device_count(int *count);
int64_t kry_launch_count(void);          /* kernels launched by this library */
void kry_reset_launch_count(void);

/* context: one operator, one block width s, capacity max_m Lanczos steps */
int kry_ctx_create(kry_ctx **out, int device, const kry_operator_desc *op,
                   int s, int max_m);
void kry_ctx_destroy(kry_ctx *ctx);
int kry_ctx_info(kry_ctx *ctx, int64_t *n, int *s, int *m, int *exhausted);

/* multi-GPU (row slabs): NCCL communicator from a 128-byte unique id */
int kry_nccl_unique_id(void *id128);
int kry_comm_init(kry_ctx *ctx, int nranks, int rank, const void *id128);

/* in-process loopback transport for the same sharded path: several slab
 * contexts of one process (one host thread per rank, e.g. all on one GPU)
 * exchange halos and sum Gram partials through event-ordered device copies
 * and a host rendezvous instead of NCCL.  Create the group once, attach one
 * context per rank, drive every rank from its own thread; destroy the group
 * after all its contexts are destroyed. */
typedef struct kry_loop kry_loop;
int kry_loop_create(int nranks, kry_loop **out);
void kry_loop_destroy(kry_loop *group);
int kry_comm_init_loopback(kry_ctx *ctx, kry_loop *group, int rank);

/* operator apply: Y = A V for a host block V (n x ncols, row-major) */
int kry_apply(kry_ctx *ctx, const double *v, double *y, int ncols);

/* first block: V1 = C gamma^{-1}; gamma (s x s upper), beta2 = ||C||_F^2 */
int kry_init_basis(kry_ctx *ctx, const double *c, double *gamma, double *beta2);
/* same from a device pointer (n x s row-major) */
int kry_init_basis_device(kry_ctx *ctx, const double *c_dev, double *gamma,
                          double *beta2);

/* one standard block-Lanczos step (MGS twice + QR); finalize_on_zero mirrors
 * on_zero_residual="finalize" (else a zero block raises DEFLATION) */
int kry_lanczos_step(kry_ctx *ctx, int finalize_on_zero, int *exhausted);

/* projection blocks so far: m diagonal blocks (raw MGS sums, symmetrised),
 * off_mgs and the m coupling blocks tau (R factors).  Arrays are m*s*s. */
int kry_get_projection(kry_ctx *ctx, int *m, double *diag_raw, double *diag_sym,
                       double *off_mgs, double *sub);
/* copy the two newest basis blocks (orthonormal, n x s each) */
int kry_get_window(kry_ctx *ctx, double *older, double *current, int *have_older);

/* cheap residual of the current projection (requires the eigen data of T_m:
 * updated incrementally by the step functions) */
int kry_check_lyap(kry_ctx *ctx, double beta2, double *res, double *rel);
int kry_check_sylv(kry_ctx *a, kry_ctx *b, double rhs_norm, double *res,
                   double *rel);

/* pass 1: the whole iteration loop on the device.  history: max_m rows of
 * (m, space_dim, relative_residual, cum_basis_secs, cum_residual_secs).
 * Returns KRY_OK (converged), KRY_ERR_CONVERGENCE (history valid), or an
 * error.  iterations = converged m. */
int kry_solve_lyap_pass1(kry_ctx *ctx, double tol, int max_m, int check_period,
                         double *history, int *n_history, int *iterations,
                         double *final_rel, int *reason);
int kry_solve_sylv_pass1(kry_ctx *a, kry_ctx *b, double tol, int max_m,
                         int check_period, double *history, int *n_history,
                         int *iterations, double *final_rel, int *reason);
/* reason: 0 converged, 1 max_m reached, 2 Krylov space invariant (exhausted) */

/* finalisation: reduced solution in the eigenbasis, truncated factor */
int kry_finalize_lyap(kry_ctx *ctx, double trunc_eps, int *rank,
                      double *discarded);
int kry_finalize_sylv(kry_ctx *a, kry_ctx *b, double trunc_eps, int *rank,
                      double *discarded);

/* one-sided Sylvester A X + X B + C1 C2^T = 0 with B small and dense
 * (solve_sylvester_one_sided, solvers.py:386-481).  The context is the A
 * side (its block Krylov space of C1).  setup: B (n2 x n2 row-major,
 * symmetric) is eigendecomposed on the device, P^T C2 (C2: n2 x s row-major)
 * is kept; ups (n2, ascending) is returned for the definiteness check.
 * check: residual_one_sided of the current projection (after kry_init_basis
 * and the steps).  finalize: rank, discarded tail mass and the right factor
 * z2 = P * (V sqrt(sigma)) (host n2 x rank row-major; z2 may be NULL to
 * query the rank first, then call again); the left factor comes from
 * kry_recover. */
int kry_sylv1_setup(kry_ctx *ctx, int n2, const double *b, const double *c2,
                    double *ups);
int kry_check_sylv1(kry_ctx *ctx, double rhs_norm, double *res, double *rel);
int kry_finalize_sylv1(kry_ctx *ctx, double trunc_eps, int *rank,
                       double *discarded, double *z2, int z2_cap);

/* install a caller-provided reduced factor qy (k x t row-major, k = s*m) for
 * the first m blocks, as two_pass_recover(op, state, qy) does (solvers.py:130) */
int kry_set_qy(kry_ctx *ctx, int m, int t, const double *qy);

/* storage mode (SolveOptions.storage, solvers.py:49-73): stored != 0 keeps
 * every basis block of pass 1 in device memory while it fits (chunked), so
 * kry_recover assembles Z = V qy without regenerating the basis
 * (_assemble_stored, solvers.py:125-127); it falls back to the two-pass
 * regeneration when the memory runs out.  Set before kry_init_basis. */
int kry_set_storage(kry_ctx *ctx, int stored);

/* pass 2: regenerate the basis and accumulate Z = sum_i V_i qy_i.
 * z: host n x rank row-major (or NULL to keep Z on the device only). */
int kry_recover(kry_ctx *ctx, double *z);
int kry_get_factor(kry_ctx *ctx, double *z);   /* copy device Z to host */

/* standalone projected-matrix kernels (no operator needed) */
int kry_partial_eig(int device, int s, int m, const double *diag,
                    const double *sub, double *lam, double *first_rows,
                    double *last_rows);
/* the finalisation's dense LAPACK calls on the repo's own block Jacobi
 * kernels (host buffers, column-major): eigh of a symmetric k x k matrix
 * (a: matrix in, eigenvectors out; w ascending) and the thin SVD of an
 * m x n matrix (u: m x n, sig descending, vt: n x n); sweeps may be NULL;
 * semidefinite != 0: the caller knows the spectrum has one sign (no shift) */
int kry_dense_eigh(int device, int k, double *a, double *w, int *sweeps,
                   int semidefinite);
/* eigh of a block-tridiagonal matrix given by its blocks (diag: m s x s,
 * sub: m-1 s x s, T[b+1,b] = sub[b]) by divide and conquer on the band:
 * lam ascending (s m), q column-major (s m) x (s m) eigenvectors */
int kry_band_eigh(int device, int s, int m, const double *diag,
                  const double *sub, double *lam, double *q);
int kry_dense_svd(int device, int m, int n, const double *a, double *u,
                  double *sig, double *vt, int *sweeps);
int kry_ctri_lyap_blocks(int device, int s, int m, const double *diag,
                         const double *sub, const double *gamma,
                         const double *tau, double *res);
int kry_ctri_sylv_blocks(int device, int s, int m1, const double *diag1,
                         const double *sub1, int m2, const double *diag2,
                         const double *sub2, const double *gamma1,
                         const double *gamma2, const double *tau,
                         const double *iota, double *res);

/* ||A Z Z^T + Z Z^T A + C C^T||_F via small Gram matrices (device) */
int kry_true_lyap_residual(kry_ctx *ctx, const double *z, int t,
                           const double *c, double *res);

/* profiling: average duration (ms) of the fused recurrence kernel launches
 * recorded since the last reset, plus launch count */
int kry_profile_enable(kry_ctx *ctx, int enable);
int kry_profile_read(kry_ctx *ctx, double *combine_ms_total, int *combine_launches,
                     double *apply_ms_total, int *apply_launches);
/* measurement: fp64 DFMA / DMMA peak of the device (TFLOP/s, one-wave
 * microbenchmark), and the average time of the cheap residual (u, w and the
 * Cauchy contraction) on the context's current eigen data (k = its order) */
int kry_fp64_peak(int device, double *dfma_tflops, double *dmma_tflops);
int kry_profile_check(kry_ctx *ctx, int reps, double *ms, int *k);
/* pass-2 factor-accumulation launches recorded while profiling is enabled:
 * total device ms, total flops (2 n K r per chunk), launch count */
int kry_profile_zacc(kry_ctx *ctx, double *ms_total, double *flops_total, int *launches);
/* CUDA-event timer on the context's stream: op 0 records the start, op 1
 * records the stop, synchronises and returns the elapsed milliseconds */
int kry_timer(kry_ctx *ctx, int op, double *ms);

#ifdef __cplusplus
}
#endif
#endif /* KRYMAT_B200_H */
