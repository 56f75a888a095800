// Finalisation (once per solve) and pass-2 helper kernels.
//
// Reference: solvers.py:254-264 (Lyapunov) and :349-358 (Sylvester): a full
// eigendecomposition of the projected matrix, the reduced solution in the
// eigenbasis  Ytilde = -(u u^T)/(lam_i + lam_j)  (guarded denominators,
// kernels.py:31-45), its truncated factorisation (truncated_spd_factor,
// kernels.py:309-331 / truncated_svd_factor, kernels.py:334-345) and
// qy = Q * factor.  The eigendecomposition of T_m is the band divide and
// conquer of eigen.cu, the truncated factorisations work on low-rank factors
// of Ytilde (pivoted Cholesky / cross factorisation + block Jacobi, dense.cu);
// assembly, Ytilde, the exact tail-mass truncation rule and the factor
// scaling are kernels here.  No library call anywhere.
#include "kry_internal.cuh"
#include "finalize.cuh"
#include <cmath>

namespace kry {

// dense symmetric T (k x k, column-major == row-major) from the block slots
__global__ void k_assemble_T(const double* dsym, const double* sub, int s, int m, double* Td) {
  const int k = s * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % k), c = (int)(e / k);
    const int br = r / s, bc = c / s, ir = r % s, ic = c % s;
    double v = 0.0;
    if (br == bc) v = dsym[(int64_t)br * 64 + ir * 8 + ic];
    else if (br == bc + 1) v = sub[(int64_t)bc * 64 + ir * 8 + ic];      // T[b+1, b] = tau_b
    else if (bc == br + 1) v = sub[(int64_t)br * 64 + ic * 8 + ir];      // T[b, b+1] = tau_b^T
    Td[e] = v;
  }
}

// u[i][c] = sum_r Q[r][i] gamma[r][c]   (Q column-major k x k, eigvec i = column i)
__global__ void k_first_rows_times(const double* Q, int k, int s, const double* gamma, double* u) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
    for (int c = 0; c < s; ++c) {
      double a = 0.0;
      for (int r = 0; r < s; ++r) a = fma(Q[(int64_t)i * k + r], gamma[r * 8 + c], a);
      u[(int64_t)i * 8 + c] = a;
    }
  }
}

// Y[i + j*ldy] = -(u_i . v_j) / (lx_i + ly_j) ; mind[blk] = min |den|
__global__ void k_ytilde(const double* u, const double* lx, int nx, const double* v,
                         const double* ly, int ny, int s, double* Y, int64_t ldy,
                         double* mind_part) {
  __shared__ double red[256];
  double mn = 1e300;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)nx * ny;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx), j = (int)(e / nx);
    double dot = 0.0;
    for (int c = 0; c < s; ++c) dot = fma(u[(int64_t)i * 8 + c], v[(int64_t)j * 8 + c], dot);
    const double den = lx[i] + ly[j];
    mn = fmin(mn, fabs(den));
    Y[i + j * ldy] = -(dot / den);
  }
  red[threadIdx.x] = mn;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) mind_part[blockIdx.x] = red[0];
}

// truncation rule of kernels.py:322-331 / 338-341 on a spectrum `ev` of length
// k stored ascending (desc=0: eigenvalues of an eigensolver) or descending (desc=1:
// singular values).  out[0] = rank, out[1] = discarded, out[2] = min value,
// out[3] = max |value|, out[4] = min denominator over parts.
template <bool SM>
__global__ void k_truncate(const double* ev, int k, int desc, double eps, const double* mind_part,
                           int nparts, double* work, double* out) {
  if (blockIdx.x != 0) return;
  // the squares, smallest first (the reference's lam[::-1] order), staged in
  // shared memory by the whole block (SM); the cumulative sum itself stays
  // sequential (np.cumsum order, which decides the rank at the eps boundary)
  extern __shared__ double sq[];
  if (SM) {
    for (int l = threadIdx.x; l < k; l += blockDim.x) {
      const double x = desc ? ev[k - 1 - l] : ev[l];
      sq[l] = x * x;
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  double acc = 0.0;
  for (int l = 0; l < k; ++l) {
    if (SM) {
      acc += sq[l];
    } else {
      const double x = desc ? ev[k - 1 - l] : ev[l];
      acc += x * x;
    }
    work[l] = acc;              // work[l] = sum of the l+1 smallest
  }
  int rank = 0;
  for (int i = 0; i < k; ++i) {  // tail(i) in descending order = sqrt(work[k-1-i])
    const double tail = sqrt(work[k - 1 - i]);
    if (tail > eps) ++rank;
  }
  out[0] = (double)rank;
  out[1] = (rank < k) ? sqrt(work[k - 1 - rank]) : 0.0;
  double mn = 1e300, mx = 0.0;
  for (int l = 0; l < k; ++l) {
    mn = fmin(mn, ev[l]);
    mx = fmax(mx, fabs(ev[l]));
  }
  out[2] = mn;
  out[3] = mx;
  double md = 1e300;
  for (int b = 0; b < nparts; ++b) md = fmin(md, mind_part[b]);
  out[4] = md;
}

// factor[:, c] = W[:, src(c)] * sqrt(max(val(c), 0)) for c < rank
// desc=0: W columns ascending (use column k-1-c), desc=1: already descending
// W is column-major with leading dimension ldw; factor column-major k x rank
__global__ void k_scale_factor(const double* W, int64_t ldw, const double* ev, int k, int rank,
                               int desc, int transposed, double* factor) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * rank;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % k), c = (int)(e / k);
    const int src = desc ? c : (k - 1 - c);
    const double val = ev[src];
    const double sc = sqrt(fmax(val, 0.0));
    // transposed: W holds rows as vectors (VT of an SVD): vector c = row c
    const double x = transposed ? W[(int64_t)r * ldw + src] : W[(int64_t)src * ldw + r];
    factor[e] = x * sc;
  }
}

// Qc[(b*s + a) * rank + c] = sum_q S_i[a][q] * qy[(i*s + q) * rank + c], i = blk0 + b
__global__ void k_chunk_coef(const double* S, const double* qy, int s, int rank, int blk0,
                             int nblk, double* Qc) {
  const int64_t total = (int64_t)nblk * s * rank;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % rank);
    const int64_t ra = e / rank;
    const int a = (int)(ra % s), b = (int)(ra / s);
    const int i = blk0 + b;
    double v = 0.0;
    for (int q = 0; q < s; ++q)
      v = fma(S[(int64_t)i * 64 + a * 8 + q], qy[((int64_t)i * s + q) * rank + c], v);
    Qc[e] = v;
  }
}

static int grid_for(int64_t n, int bs = 256) {
  int64_t g = (n + bs - 1) / bs;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  return (int)g;
}

int launch_assemble_T(cudaStream_t st, const double* dsym, const double* sub, int s, int m,
                      double* Td) {
  const int64_t k = (int64_t)s * m;
  k_assemble_T<<<grid_for(k * k), 256, 0, st>>>(dsym, sub, s, m, Td);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}
int launch_first_rows_times(cudaStream_t st, const double* Q, int k, int s, const double* gamma,
                            double* u) {
  k_first_rows_times<<<grid_for(k), 256, 0, st>>>(Q, k, s, gamma, u);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}
int launch_ytilde(cudaStream_t st, const double* u, const double* lx, int nx, const double* v,
                  const double* ly, int ny, int s, double* Y, int64_t ldy, double* mind_part,
                  int* nparts) {
  int g = grid_for((int64_t)nx * ny);
  if (g > 1024) g = 1024;
  k_ytilde<<<g, 256, 0, st>>>(u, lx, nx, v, ly, ny, s, Y, ldy, mind_part);
  *nparts = g;
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}
int launch_truncate(cudaStream_t st, const double* ev, int k, int desc, double eps,
                    const double* mind_part, int nparts, double* work, double* out) {
  const size_t smb = (size_t)k * sizeof(double);
  if (smb <= (size_t)200 * 1024) {
    static bool attr[64] = {false};   // the attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
      cudaFuncSetAttribute(k_truncate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr[dev & 63] = true;
    }
    k_truncate<true><<<1, 256, smb, st>>>(ev, k, desc, eps, mind_part, nparts, work, out);
  } else {
    k_truncate<false><<<1, 32, 0, st>>>(ev, k, desc, eps, mind_part, nparts, work, out);
  }
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}
int launch_scale_factor(cudaStream_t st, const double* W, int64_t ldw, const double* ev, int k,
                        int rank, int desc, int transposed, double* factor) {
  if (rank <= 0) return KRY_OK;
  k_scale_factor<<<grid_for((int64_t)k * rank), 256, 0, st>>>(W, ldw, ev, k, rank, desc,
                                                              transposed, factor);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}
int launch_chunk_coef(cudaStream_t st, const double* S, const double* qy, int s, int rank,
                      int blk0, int nblk, double* Qc) {
  if (rank <= 0 || nblk <= 0) return KRY_OK;
  k_chunk_coef<<<grid_for((int64_t)nblk * s * rank), 256, 0, st>>>(S, qy, s, rank, blk0, nblk,
                                                                   Qc);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

}  // namespace kry
