#pragma once
#include "kry_internal.cuh"

namespace kry {
int launch_assemble_T(cudaStream_t st, const double* dsym, const double* sub, int s, int m,
                      double* Td);
int launch_first_rows_times(cudaStream_t st, const double* Q, int k, int s, const double* gamma,
                            double* u);
int launch_ytilde(cudaStream_t st, const double* u, const double* lx, int nx, const double* v,
                  const double* ly, int ny, int s, double* Y, int64_t ldy, double* mind_part,
                  int* nparts);
int launch_truncate(cudaStream_t st, const double* ev, int k, int desc, double eps,
                    const double* mind_part, int nparts, double* work, double* out);
int launch_scale_factor(cudaStream_t st, const double* W, int64_t ldw, const double* ev, int k,
                        int rank, int desc, int transposed, double* factor);
int launch_chunk_coef(cudaStream_t st, const double* S, const double* qy, int s, int rank,
                      int blk0, int nblk, double* Qc);
// pass-2 / stored factor accumulation on DMMA (zacc.cu):
// Z[i][:] (+)= sum_b V_b[i][:] Q[b s .. b s + s)[:], V_b = vbase + b vstride
// max_ctas > 0: a grid of at most that many CTAs looping over the tiles
int launch_zacc(cudaStream_t st, int s, const double* vbase, int64_t vstride, int nb,
                const double* Q, int ldq, int r, double* Z, int64_t n, int accumulate,
                int max_ctas = 0);
int launch_chunk_coef_ld(cudaStream_t st, const double* S, const double* qy, int s, int rank,
                         int blk0, int nblk, int ldq, double* Qc);
int zacc_ldq(int r);   // padded leading dimension of the Q panel
}  // namespace kry
