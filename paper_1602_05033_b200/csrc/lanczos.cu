// Block-Lanczos recurrence kernels for sm_100a (fp64).
//
// One standard block-Lanczos step of the reference (basis.py:223-252:
// W = A V_m; MGS twice against V_{m-1}, V_m (basis.py:164-180); economy QR
// with diag(R) >= 0 (kernels.py:134-148)) is executed as two HBM passes:
//
//   apply   (k_apply_gram):  W0 = A V_m on the fly, Gram blocks V_m^T W0 and
//                            W0^T W0 (DMMA m8n8k4 tiles), grid reduction in a
//                            fixed order; the last CTA runs the coefficient
//                            solve (MGS-twice simulated on the Gram algebra,
//                            Cholesky QR of the residual block, lazy CholQR2
//                            correction of the previous block).
//   combine (k_combine):     V_{m+1} = V_{m-1} Mo + V_m Mc + (A V_m) Mw with
//                            the stencil recomputed on the fly, plus the Gram
//                            blocks the next coefficient solve needs
//                            (V_m^T V_{m+1}, (A V_m)^T V_{m+1}, V_{m+1}^T V_{m+1}).
//
// so a step reads V_{m-1}, V_m twice-ish and writes V_{m+1} once (4 block
// transfers instead of the reference's ~12 BLAS passes).  The operator is a
// 3/5/7-point Dirichlet stencil (constant or per-point coefficients) or a CSR
// matrix; row sums use __dmul_rn/__dadd_rn in CSR column order so A*V equals
// scipy's csr_matvecs (operators.py:101) bit for bit.
#include "kry_internal.cuh"
#include <algorithm>
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <cstdlib>

namespace kry {

#define TP 128     // points per tile = threads per CTA
#define XCOLS 24   // tile columns (<= 3 groups of 8)
#define LDP (TP + 4)  // transposed tile stride: conflict-free row writes and DMMA loads
// column k of a transposed tile starts at CB(k): stride LDP plus a 4-row
// shift on every other group of 4 columns, so a half-warp storing 4 column
// pairs x 4 points (the cooperative staging order, which keeps each quarter
// warp's 16-byte global loads inside one 128-byte line) hits 16 distinct bank
// pairs; the shift is uniform per DMMA fragment load, which stays conflict-free.
#define CB(k) ((k) * LDP + ((k) & 4))

// ------------------------------------------------------------------ vector io
template <int S>
__device__ __forceinline__ void load_vec(const double* __restrict__ p, double (&v)[S]) {
  if constexpr (S % 2 == 0) {
#pragma unroll
    for (int a = 0; a < S; a += 2) {
      double2 t = __ldg(reinterpret_cast<const double2*>(p + a));
      v[a] = t.x;
      v[a + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int a = 0; a < S; ++a) v[a] = __ldg(p + a);
  }
}

template <int S>
__device__ __forceinline__ void store_vec(double* __restrict__ p, const double (&v)[S]) {
  if constexpr (S % 2 == 0) {
#pragma unroll
    for (int a = 0; a < S; a += 2)
      *reinterpret_cast<double2*>(p + a) = make_double2(v[a], v[a + 1]);
  } else {
#pragma unroll
    for (int a = 0; a < S; ++a) p[a] = v[a];
  }
}

template <int S>
__device__ __forceinline__ void axpy_rn(double (&w)[S], double coef, const double (&x)[S]) {
#pragma unroll
  for (int a = 0; a < S; ++a) w[a] = __dadd_rn(w[a], __dmul_rn(coef, x[a]));
}

// y = A x at local point i (CSR column order, no FMA contraction)
template <int S>
__device__ __forceinline__ void apply_point(const OpDev& op, const double* __restrict__ V,
                                            int64_t ld, int i, const double (&vi)[S],
                                            double (&w)[S]) {
#pragma unroll
  for (int a = 0; a < S; ++a) w[a] = 0.0;
  double nb[S];
  if (op.kind == KRY_OP_STENCIL) {
    const int x = i % op.nx;
    const int r = i / op.nx;
    const int y = r % op.ny;
    const int z = r / op.ny;
    const bool var = op.variable != 0;
    const bool hz0 = z > 0 || op.halo_lo, hy0 = y > 0, hx0 = x > 0;
    const bool hx1 = x < op.nx - 1, hy1 = y < op.ny - 1, hz1 = z < op.nzl - 1 || op.halo_hi;
    // all six gathers are issued before any use (one memory round trip);
    // a missing neighbour loads the point itself and is skipped below, so
    // the sum keeps the CSR column order exactly
    double n0[S], n1[S], n2[S], n3[S], n4[S], n5[S];
    load_vec<S>(V + (int64_t)(hz0 ? i - op.nxy : i) * ld, n0);
    load_vec<S>(V + (int64_t)(hy0 ? i - op.nx : i) * ld, n1);
    load_vec<S>(V + (int64_t)(hx0 ? i - 1 : i) * ld, n2);
    load_vec<S>(V + (int64_t)(hx1 ? i + 1 : i) * ld, n3);
    load_vec<S>(V + (int64_t)(hy1 ? i + op.nx : i) * ld, n4);
    load_vec<S>(V + (int64_t)(hz1 ? i + op.nxy : i) * ld, n5);
    if (hz0) axpy_rn<S>(w, var ? __ldg(op.ez + i - op.nxy) : op.cz, n0);
    if (hy0) axpy_rn<S>(w, var ? __ldg(op.ey + i - op.nx) : op.cy, n1);
    if (hx0) axpy_rn<S>(w, var ? __ldg(op.ex + i - 1) : op.cx, n2);
    axpy_rn<S>(w, var ? __ldg(op.d + i) : op.cd, vi);
    if (hx1) axpy_rn<S>(w, var ? __ldg(op.ex + i) : op.cx, n3);
    if (hy1) axpy_rn<S>(w, var ? __ldg(op.ey + i) : op.cy, n4);
    if (hz1) axpy_rn<S>(w, var ? __ldg(op.ez + i) : op.cz, n5);
  } else {
    const int64_t b = __ldg(op.rp + i), e = __ldg(op.rp + i + 1);
    for (int64_t jj = b; jj < e; ++jj) {
      const int j = __ldg(op.ci + jj);
      load_vec<S>(V + (int64_t)j * ld, nb);
      axpy_rn<S>(w, __ldg(op.va + jj), nb);
    }
  }
}

// ------------------------------------------------------------------ DMMA gram tile
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// acc[mt] += X[rows k0..k0+31, mt*8..mt*8+7]^T * X[rows, ycol..ycol+7]
template <int MT>
__device__ __forceinline__ void tile_gram(const double* sX, int k0, int ycol, double (&acc)[MT][2]) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int k = k0 + ks * 4 + t;   // point index inside the tile
    const double b = sX[CB(ycol + g) + k];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][0], acc[mt][1], sX[CB(mt * 8 + g) + k], b);
  }
}

// ------------------------------------------------------------------ small matrices (smem, 8x8 row-major)
__device__ __forceinline__ int tid() { return threadIdx.x; }

__device__ void m_copy(double* dst, const double* src) {
  __syncthreads();
  if (tid() < 64) dst[tid()] = src[tid()];
  __syncthreads();
}
__device__ void m_eye(double* dst, int s) {
  __syncthreads();
  if (tid() < 64) {
    int r = tid() >> 3, c = tid() & 7;
    dst[tid()] = (r == c && r < s) ? 1.0 : 0.0;
  }
  __syncthreads();
}
__device__ void m_zero(double* dst) {
  __syncthreads();
  if (tid() < 64) dst[tid()] = 0.0;
  __syncthreads();
}
// C = alpha * op(A) op(B) (+ beta * D when D != nullptr); C may alias inputs
__device__ void mm(double* C, const double* A, int ta, const double* B, int tb, int s,
                   double alpha = 1.0, const double* D = nullptr, double beta = 0.0) {
  __syncthreads();
  double v = 0.0;
  if (tid() < 64) {
    int r = tid() >> 3, c = tid() & 7;
    if (r < s && c < s) {
      for (int k = 0; k < s; ++k) {
        double a = ta ? A[k * 8 + r] : A[r * 8 + k];
        double b = tb ? B[c * 8 + k] : B[k * 8 + c];
        v = fma(a, b, v);
      }
      v *= alpha;
      if (D) v = fma(beta, D[tid()], v);
    }
  }
  __syncthreads();
  if (tid() < 64) C[tid()] = v;
  __syncthreads();
}
// C = A + beta * B
__device__ void madd(double* C, const double* A, const double* B, double beta) {
  __syncthreads();
  double v = 0.0;
  if (tid() < 64) v = A[tid()] + beta * B[tid()];
  __syncthreads();
  if (tid() < 64) C[tid()] = v;
  __syncthreads();
}
// serial Cholesky G = R^T R (upper R, positive diagonal) from the upper
// triangle of G.  Returns 0 ok, 1 breakdown / numerically singular pivot.
__device__ int chol_upper(const double* G, double* R, int s, double* min_ratio) {
  for (int i = 0; i < 64; ++i) R[i] = 0.0;
  double mr = 1e300;
  for (int k = 0; k < s; ++k) {
    double p = G[k * 8 + k];
    for (int i = 0; i < k; ++i) p -= R[i * 8 + k] * R[i * 8 + k];
    // pivots at the level of the Gram's rounding are treated as zero
    if (!(p > 1e3 * 2.220446049250313e-16 * fabs(G[k * 8 + k])) || !(p > 0.0)) return 1;
    const double rkk = sqrt(p);
    R[k * 8 + k] = rkk;
    for (int j = k + 1; j < s; ++j) {
      double v = G[k * 8 + j];
      for (int i = 0; i < k; ++i) v -= R[i * 8 + k] * R[i * 8 + j];
      R[k * 8 + j] = v / rkk;
    }
  }
  double fro = 0.0;
  for (int i = 0; i < 64; ++i) fro += R[i] * R[i];
  fro = sqrt(fro);
  for (int k = 0; k < s; ++k) mr = fmin(mr, R[k * 8 + k] / fro);
  *min_ratio = mr;
  return 0;
}
// Shifted Cholesky of shifted CholQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto,
// Yamazaki 2020): R = chol(G + sigma I), sigma = 11 (n s + s (s + 1)) u ||G||,
// with ||G|| bounded by trace(G).  The shift keeps the factorisation
// positive definite for any W with kappa(W) up to ~u^-1, and Q0 = W R^-1 is
// then well enough conditioned (kappa ~ (n s u)^-1/2) for two plain CholQR
// stages to reach Householder-level orthogonality.  That is what resolves
// the rank of ill-conditioned blocks the way economy_qr (kernels.py:134-160)
// does, instead of failing at the Gram's rounding level (kappa ~ 1e7).
__device__ int chol_shifted(const double* G, double* R, int s, double nrows) {
  double tr = 0.0;
  for (int k = 0; k < s; ++k) tr += fabs(G[k * 8 + k]);
  const double sigma = 11.0 * (nrows * s + s * (s + 1.0)) * 2.220446049250313e-16 * tr;
  for (int i = 0; i < 64; ++i) R[i] = 0.0;
  for (int k = 0; k < s; ++k) {
    double p = G[k * 8 + k] + sigma;
    for (int i = 0; i < k; ++i) p -= R[i * 8 + k] * R[i * 8 + k];
    if (!(p > 0.0)) return 1;
    const double rkk = sqrt(p);
    R[k * 8 + k] = rkk;
    for (int j = k + 1; j < s; ++j) {
      double v = G[k * 8 + j];
      for (int i = 0; i < k; ++i) v -= R[i * 8 + k] * R[i * 8 + j];
      R[k * 8 + j] = v / rkk;
    }
  }
  return 0;
}
__device__ void inv_upper(const double* R, double* Ri, int s) {
  for (int i = 0; i < 64; ++i) Ri[i] = 0.0;
  for (int j = 0; j < s; ++j) {
    Ri[j * 8 + j] = 1.0 / R[j * 8 + j];
    for (int i = j - 1; i >= 0; --i) {
      double v = 0.0;
      for (int k = i + 1; k <= j; ++k) v += R[i * 8 + k] * Ri[k * 8 + j];
      Ri[i * 8 + j] = -v / R[i * 8 + i];
    }
  }
}
// Warp-parallel Cholesky + triangular inverse for the coefficient tail (all
// threads of the CTA call it; warp 0 computes).  Same arithmetic order as
// chol_upper (right-looking form of the same left-to-right subtractions) and
// inv_upper (one lane per column).  Returns the breakdown flag uniformly;
// Ri is written only when the factorisation succeeded.
__device__ int chol_inv_par(const double* G, double* R, double* Ri, int s, double* min_ratio) {
  __shared__ double s_W[64];
  __shared__ int s_bad;
  __shared__ double s_mr;
  __syncthreads();
  if (tid() < 32) {
    const int l = tid();
    for (int q = l; q < 64; q += 32) {
      s_W[q] = G[q];
      R[q] = 0.0;
    }
    __syncwarp();
    int bad = 0;
    for (int k = 0; k < s; ++k) {
      const double p = s_W[k * 8 + k];
      if (!(p > 1e3 * 2.220446049250313e-16 * fabs(G[k * 8 + k])) || !(p > 0.0)) {
        bad = 1;
        break;
      }
      const double rkk = sqrt(p);
      if (l >= k && l < s) R[k * 8 + l] = (l == k) ? rkk : s_W[k * 8 + l] / rkk;
      __syncwarp();
      for (int q = l; q < 64; q += 32) {
        const int i = q >> 3, j = q & 7;
        if (i > k && j >= i && j < s) s_W[q] -= R[k * 8 + i] * R[k * 8 + j];
      }
      __syncwarp();
    }
    if (!bad) {
      if (l < s) {
        const int j = l;
        for (int i = 0; i < 8; ++i) Ri[i * 8 + j] = 0.0;
        Ri[j * 8 + j] = 1.0 / R[j * 8 + j];
        for (int i = j - 1; i >= 0; --i) {
          double v = 0.0;
          for (int k = i + 1; k <= j; ++k) v += R[i * 8 + k] * Ri[k * 8 + j];
          Ri[i * 8 + j] = -v / R[i * 8 + i];
        }
      } else if (l < 8) {
        for (int i = 0; i < 8; ++i) Ri[i * 8 + l] = 0.0;
      }
      if (l == 0) {
        double fro = 0.0;
        for (int i = 0; i < 64; ++i) fro += R[i] * R[i];
        fro = sqrt(fro);
        double mr = 1e300;
        for (int k = 0; k < s; ++k) mr = fmin(mr, R[k * 8 + k] / fro);
        s_mr = mr;
      }
    }
    if (l == 0) s_bad = bad;
  }
  __syncthreads();
  *min_ratio = s_mr;
  return s_bad;
}
__device__ double m_trace(const double* A, int s) {
  double t = 0.0;
  for (int k = 0; k < s; ++k) t += A[k * 8 + k];
  return t;
}

// ------------------------------------------------------------------ post routines
struct PostSmem {
  double G[12][64];
};

__device__ void set_status(DevState* st, int code) {
  if (tid() == 0 && st->status == KRY_OK) st->status = code;
}

// The new block V_{j+1} = W R1^-1 leaves the combine with one Cholesky-QR
// stage; its Gram Gcc (just reduced) gives the second stage R2 = chol(Gcc),
// which the next coefficient solve applies lazily.  The coupling the
// residual check of step j reads (T.tau1[j-1]) is finalised here to R2 R1
// -- the same product, bit for bit, that the next solve stores in T.sub --
// so the check uses the reference's final QR factor (basis.py:241-249)
// instead of the first stage (which differs by ~eps ||AV||^2 / ||W||^2).
__device__ void finalize_tau(DevState* st, const TStore& T, double (*sm)[64], const double* Gcc) {
  const int j = st->step;   // the step whose combine produced the block
  if (j < 1 || j > T.cap) return;
  __syncthreads();
  double mr;
  // scratch slots 3..5: the callers (POST_P / POST_FUSED) hold Gram blocks
  // in slots 0..2 only (the smallest post scratch has 14 slots)
  const int bad = chol_inv_par(Gcc, sm[3], sm[4], st->s, &mr);
  if (bad) return;   // the next solve takes the fallback; keep R1
  mm(sm[5], sm[3], 0, st->R1prev, 0, st->s);
  if (tid() < 64) T.tau1[(int64_t)(j - 1) * 64 + tid()] = sm[5][tid()];
  __syncthreads();
}

// total: MP x 8 reduced Gram (row = X column, col = Y column)
__device__ void extract_block(const double* total, int row0, int s, double* dst) {
  __syncthreads();
  if (tid() < 64) {
    int r = tid() >> 3, c = tid() & 7;
    dst[tid()] = (r < s && c < s) ? total[(row0 + r) * 8 + c] : 0.0;
  }
  __syncthreads();
}

// ---- warp-synchronous small-matrix helpers: the coefficient solve runs on
// ONE warp (lane l owns elements l and l + 32 of every 8 x 8 slot), with
// __syncwarp instead of block barriers.  Every element is computed with the
// same sequence of operations as mm / madd / chol_inv_par above, so the
// results are bit-identical to the block-wide versions; the ~45 dependent
// small products of a solve no longer cost block barriers on the last CTA
// of every step (the serial tail of the recurrence).
__device__ __forceinline__ void w_mm(double* C, const double* A, int ta, const double* B, int tb,
                                     int s, double alpha = 1.0, const double* D = nullptr,
                                     double beta = 0.0) {
  const int l = threadIdx.x & 31;
  double out[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int e = l + 32 * h, r = e >> 3, c = e & 7;
    double v = 0.0;
    if (r < s && c < s) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < s) {
          const double a = ta ? A[k * 8 + r] : A[r * 8 + k];
          const double b = tb ? B[c * 8 + k] : B[k * 8 + c];
          v = fma(a, b, v);
        }
      }
      v *= alpha;
      if (D) v = fma(beta, D[e], v);
    }
    out[h] = v;
  }
  __syncwarp();
  C[l] = out[0];
  C[l + 32] = out[1];
  __syncwarp();
}
__device__ __forceinline__ void w_madd(double* C, const double* A, const double* B, double beta) {
  const int l = threadIdx.x & 31;
  const double v0 = A[l] + beta * B[l];
  const double v1 = A[l + 32] + beta * B[l + 32];
  __syncwarp();
  C[l] = v0;
  C[l + 32] = v1;
  __syncwarp();
}
__device__ __forceinline__ void w_copy(double* dst, const double* src) {
  const int l = threadIdx.x & 31;
  const double v0 = src[l], v1 = src[l + 32];
  __syncwarp();
  dst[l] = v0;
  dst[l + 32] = v1;
  __syncwarp();
}
__device__ __forceinline__ void w_zero(double* dst) {
  const int l = threadIdx.x & 31;
  __syncwarp();
  dst[l] = 0.0;
  dst[l + 32] = 0.0;
  __syncwarp();
}
__device__ __forceinline__ void w_extract(const double* total, int row0, int s, double* dst) {
  const int l = threadIdx.x & 31;
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int e = l + 32 * h, r = e >> 3, c = e & 7;
    dst[e] = (r < s && c < s) ? total[(row0 + r) * 8 + c] : 0.0;
  }
  __syncwarp();
}
// chol_inv_par on the calling warp (W: 64 doubles of scratch)
__device__ int w_chol_inv(const double* G, double* R, double* Ri, int s, double* min_ratio,
                          double* W) {
  const int l = threadIdx.x & 31;
  __syncwarp();
  for (int q = l; q < 64; q += 32) {
    W[q] = G[q];
    R[q] = 0.0;
  }
  __syncwarp();
  int bad = 0;
  for (int k = 0; k < s; ++k) {
    const double p = W[k * 8 + k];
    if (!(p > 1e3 * 2.220446049250313e-16 * fabs(G[k * 8 + k])) || !(p > 0.0)) {
      bad = 1;
      break;
    }
    const double rkk = sqrt(p);
    if (l >= k && l < s) R[k * 8 + l] = (l == k) ? rkk : W[k * 8 + l] / rkk;
    __syncwarp();
    for (int q = l; q < 64; q += 32) {
      const int i = q >> 3, j = q & 7;
      if (i > k && j >= i && j < s) W[q] -= R[k * 8 + i] * R[k * 8 + j];
    }
    __syncwarp();
  }
  double mr = 1e300;
  if (!bad) {
    if (l < s) {
      const int j = l;
      for (int i = 0; i < 8; ++i) Ri[i * 8 + j] = 0.0;
      Ri[j * 8 + j] = 1.0 / R[j * 8 + j];
      for (int i = j - 1; i >= 0; --i) {
        double v = 0.0;
        for (int k = i + 1; k <= j; ++k) v += R[i * 8 + k] * Ri[k * 8 + j];
        Ri[i * 8 + j] = -v / R[i * 8 + i];
      }
    } else if (l < 8) {
      for (int i = 0; i < 8; ++i) Ri[i * 8 + l] = 0.0;
    }
    if (l == 0) {
      double fro = 0.0;
      for (int i = 0; i < 64; ++i) fro += R[i] * R[i];
      fro = sqrt(fro);
      for (int k = 0; k < s; ++k) mr = fmin(mr, R[k * 8 + k] / fro);
    }
    mr = __shfl_sync(0xffffffffu, mr, 0);
  }
  __syncwarp();
  *min_ratio = mr;
  return bad;
}

// The coefficient solve of one fused step (see file header).  Runs on warp 0
// of the last CTA of the apply reduction; `total` holds [V^T W0 ; W0^T W0].
// `row_cw` / `row_ww`: first rows of V_c^T W0 and W0^T W0 in `total`.  With
// `deferred` (the fused step kernel solves step j+1 ahead of time) a failure
// only raises KRY_FLAG_FALLBACK: the host then redoes step j+1 on the
// two-kernel path, which repeats this (idempotent up to the failure point)
// solve and reports the error at the step the reference reports it.
__device__ __noinline__ void coef_solve_w(const double* total, DevState* st, const TStore& T, double (*sm)[64],
                                        int row_cw, int row_ww, int deferred) {
  const int s = st->s;
  double* Gcc = sm[0]; double* Goc = sm[1]; double* GoW = sm[2]; double* Goo = sm[3];
  double* GcW = sm[4]; double* GWW = sm[5]; double* Sc = sm[6]; double* So = sm[7];
  double* A = sm[8]; double* B = sm[9]; double* X = sm[10]; double* Y = sm[11];
  double* Z = sm[12]; double* U = sm[13];
  const int lane = threadIdx.x & 31;
  // the five carried 8x8 blocks in one batch of loads (all in flight)
  __syncwarp();
  for (int q = lane; q < 5 * 64; q += 32) {
    const int b = q >> 6, e = q & 63;
    const double* src = b == 0 ? st->Gcc : b == 1 ? st->Goc : b == 2 ? st->GoW : b == 3 ? st->Goo : st->So;
    double* dst = b == 0 ? Gcc : b == 1 ? Goc : b == 2 ? GoW : b == 3 ? Goo : So;
    dst[e] = src[e];
  }
  w_extract(total, row_cw, s, GcW);
  w_extract(total, row_ww, s, GWW);
  const int j = st->step + 1;        // 1-based step being solved
  const int has_old = st->has_old;
  // 1. lazy CholQR2 correction of the current block: Gcc = R2^T R2, Sc = R2^-1
  {
    double mr;
    const int bad = w_chol_inv(Gcc, X, Sc, s, &mr, U);
    if (bad) {  // the stored block is not numerically full rank
      if (deferred) {
        if (lane == 0) { st->flags |= KRY_FLAG_FALLBACK; if (st->replay == 2) st->replay_err = 1e300; }
      } else {
        if (lane == 0 && st->status == KRY_OK) st->status = KRY_ERR_DEFLATION;
      }
      __syncwarp();
      return;
    }
  }
  // 2. finalise the previous coupling block (or gamma): R_hat = R2 * R1prev
  w_copy(Y, st->R1prev);
  w_mm(Z, X, 0, Y, 0, s);
  if (j == 1) {
    if (!st->replay) { st->gamma[lane] = Z[lane]; st->gamma[lane + 32] = Z[lane + 32]; }
  } else {
    double* dst = T.sub + (int64_t)(j - 2) * 64;
    if (st->replay) {
      if (lane == 0) {
        double num = 0.0, den = 0.0;
        for (int q = 0; q < 64; ++q) {
          double d = Z[q] - dst[q];
          num += d * d;
          den += dst[q] * dst[q];
        }
        double rel = sqrt(num) / fmax(sqrt(den), 1e-300);
        st->replay_err = fmax(st->replay_err, rel);
      }
    } else {
      dst[lane] = Z[lane];
      dst[lane + 32] = Z[lane + 32];
    }
  }
  for (int e = lane; e < 64; e += 32) {
    st->Sc[e] = Sc[e];
    T.S[(int64_t)(j - 1) * 64 + e] = Sc[e];
  }
  if (lane == 0) st->flags &= ~KRY_FLAG_FALLBACK;
  __syncwarp();
  // 3. Gram blocks in the orthonormal (true) basis
  w_mm(A, Sc, 1, Gcc, 0, s); w_mm(Gcc, A, 0, Sc, 0, s);    // Gcc^ = Sc^T Gcc Sc
  w_mm(A, Sc, 1, GcW, 0, s); w_mm(GcW, A, 0, Sc, 0, s);    // GcW^
  w_mm(A, Sc, 1, GWW, 0, s); w_mm(GWW, A, 0, Sc, 0, s);    // GWW^
  if (has_old) {
    w_mm(A, So, 1, Goo, 0, s); w_mm(Goo, A, 0, So, 0, s);  // Goo^
    w_mm(A, So, 1, Goc, 0, s); w_mm(Goc, A, 0, Sc, 0, s);  // Goc^
    w_mm(A, So, 1, GoW, 0, s); w_mm(GoW, A, 0, Sc, 0, s);  // GoW^
  }
  // 4. MGS performed twice on W = W0 - Vo a - Vc b  (basis.py:164-180)
  w_zero(A);  // a (off sum)
  w_zero(B);  // b (diag sum)
  for (int sweep = 0; sweep < 2; ++sweep) {
    if (has_old) {
      // alpha = GoW - Goo a - Goc b
      w_mm(X, Goo, 0, A, 0, s, -1.0, GoW, 1.0);
      w_mm(X, Goc, 0, B, 0, s, -1.0, X, 1.0);
      w_madd(A, A, X, 1.0);
    }
    // beta = GcW - Goc^T a - Gcc b
    if (has_old) {
      w_mm(X, Goc, 1, A, 0, s, -1.0, GcW, 1.0);
    } else {
      w_copy(X, GcW);
    }
    w_mm(X, Gcc, 0, B, 0, s, -1.0, X, 1.0);
    w_madd(B, B, X, 1.0);
  }
  // 5. W^T W = GWW - GcW^T b - b^T GcW + b^T Gcc b  (+ the old-block terms)
  w_mm(X, GcW, 1, B, 0, s);                 // X = GcW^T b ; Z = GWW - X - X^T
  __syncwarp();
  for (int e = lane; e < 64; e += 32) {
    int r = e >> 3, c = e & 7;
    Z[e] = GWW[e] - X[r * 8 + c] - X[c * 8 + r];
  }
  __syncwarp();
  w_mm(U, Gcc, 0, B, 0, s);                 // Gcc b
  w_mm(Z, B, 1, U, 0, s, 1.0, Z, 1.0);      // + b^T Gcc b
  if (has_old) {
    w_mm(X, GoW, 1, A, 0, s);               // GoW^T a
    __syncwarp();
    for (int e = lane; e < 64; e += 32) {
      int r = e >> 3, c = e & 7;
      Z[e] = Z[e] - X[r * 8 + c] - X[c * 8 + r];
    }
    __syncwarp();
    w_mm(U, Goo, 0, A, 0, s);               // Goo a
    w_mm(Z, A, 1, U, 0, s, 1.0, Z, 1.0);    // + a^T Goo a
    w_mm(U, Goc, 0, B, 0, s);               // Goc b
    w_mm(X, A, 1, U, 0, s);                 // a^T Goc b
    __syncwarp();
    for (int e = lane; e < 64; e += 32) {
      int r = e >> 3, c = e & 7;
      Z[e] = Z[e] + X[r * 8 + c] + X[c * 8 + r];
    }
    __syncwarp();
  }
  // symmetrise W^T W
  __syncwarp();
  for (int e = lane; e < 64; e += 32) {
    int r = e >> 3, c = e & 7;
    U[e] = 0.5 * (Z[r * 8 + c] + Z[c * 8 + r]);
  }
  __syncwarp();
  const double scale2 = m_trace(GWW, s), w2 = m_trace(U, s);
  if (lane == 0) {
    st->scale2 = scale2;
    st->w2 = w2;
  }
  // 6. zero / near-zero residual block: decided by the explicit path
  if (!(w2 > 1e-10 * scale2)) {
    if (lane == 0) { st->flags |= KRY_FLAG_FALLBACK; if (st->replay == 2) st->replay_err = 1e300; }
    return;
  }
  // 7. Cholesky QR of the residual block
  {
    double mr = 0.0;
    const int bad = w_chol_inv(U, X, Y, s, &mr, Z);
    const int fail = bad || mr < 1e-5;
    if (fail) {
      if (lane == 0) { st->flags |= KRY_FLAG_FALLBACK; if (st->replay == 2) st->replay_err = 1e300; }
      return;
    }
    for (int e = lane; e < 64; e += 32) {
      st->R1prev[e] = X[e];
      T.tau1[(int64_t)(j - 1) * 64 + e] = X[e];
    }
  }
  // 8. combine coefficients: Vn = Vo Mo + Vc Mc + W0 Mw
  w_mm(Z, Sc, 0, Y, 0, s);                   // Mw = Sc R1^-1
  for (int e = lane; e < 64; e += 32) st->M[128 + e] = Z[e];
  __syncwarp();
  w_mm(U, B, 0, Y, 0, s);                    // b R1^-1
  w_mm(Z, Sc, 0, U, 0, s, -1.0);             // Mc = -Sc b R1^-1
  for (int e = lane; e < 64; e += 32) st->M[64 + e] = Z[e];
  __syncwarp();
  if (has_old) {
    w_mm(U, A, 0, Y, 0, s);
    w_mm(Z, So, 0, U, 0, s, -1.0);           // Mo = -So a R1^-1
  } else {
    w_zero(Z);
  }
  for (int e = lane; e < 64; e += 32) st->M[e] = Z[e];
  // 9. projection blocks of step j
  for (int e = lane; e < 64; e += 32) {
    int r = e >> 3, c = e & 7;
    const int64_t o = (int64_t)(j - 1) * 64;
    if (!st->replay) {
      T.draw[o + e] = B[e];
      T.dsym[o + e] = 0.5 * (B[r * 8 + c] + B[c * 8 + r]);
      T.off[o + e] = has_old ? A[e] : 0.0;
    }
    st->So[e] = Sc[e];
    st->Goo[e] = st->Gcc[e];
  }
  __syncwarp();
  if (lane == 0) {
    st->step = j;
    st->has_old = 1;
  }
  __syncwarp();
}

__device__ __noinline__ void run_post(int post, const double* total, DevState* st, const TStore& T,
                         double (*sm)[64]) {
  const int s = st->s;
  __shared__ int s_bad;
  __shared__ double s_v;
  switch (post) {
    case POST_NONE:
      for (int e = tid(); e < 3 * 64; e += blockDim.x) st->gram[e] = total[e];
      __syncthreads();
      break;
    case POST_P:
      extract_block(total, 0, s, sm[0]);
      extract_block(total, s, s, sm[1]);
      extract_block(total, 2 * s, s, sm[2]);
      if (tid() < 64) {
        st->Goc[tid()] = sm[0][tid()];
        st->GoW[tid()] = sm[1][tid()];
        st->Gcc[tid()] = sm[2][tid()];
      }
      finalize_tau(st, T, sm, sm[2]);
      break;
    case POST_STEP:
      __syncthreads();
      if (threadIdx.x < 32) coef_solve_w(total, st, T, sm, 0, s, 0);
      __syncthreads();
      break;
    case POST_STEP8:   // [V^T W0 | W0^T W0] as two 8-row blocks (k_apply_gl)
      __syncthreads();
      if (threadIdx.x < 32) coef_solve_w(total, st, T, sm, 0, 8, 0);
      __syncthreads();
      break;
    case POST_FUSED:
      // [Goc | GoW | Gcc | GcW | GWW] as five 8x8 blocks (k_step): the
      // carried blocks of POST_P, then the coefficient solve of step j+1
      extract_block(total, 0, s, sm[0]);
      extract_block(total, 8, s, sm[1]);
      extract_block(total, 16, s, sm[2]);
      if (tid() < 64) {
        st->Goc[tid()] = sm[0][tid()];
        st->GoW[tid()] = sm[1][tid()];
        st->Gcc[tid()] = sm[2][tid()];
      }
      finalize_tau(st, T, sm, sm[2]);
      __syncthreads();
      if (threadIdx.x < 32) coef_solve_w(total, st, T, sm, 24, 32, 1);
      __syncthreads();
      break;
    case POST_INIT: {
      extract_block(total, 0, s, sm[0]);
      if (tid() == 0) {
        double mr = 0.0;
        st->beta2 = m_trace(sm[0], s);
        int shifted = 0;
        s_bad = chol_upper(sm[0], sm[1], s, &mr);
        if (s_bad) {
          // ill-conditioned C: shifted first stage, the host adds the
          // explicit middle stage (rank decided on the final gamma)
          s_bad = chol_shifted(sm[0], sm[1], s, st->nrows);
          shifted = 1;
        }
        if (s_bad) {
          if (st->status == KRY_OK) st->status = KRY_ERR_DEFLATION;
        } else {
          inv_upper(sm[1], sm[2], s);
          for (int q = 0; q < 64; ++q) {
            st->R1prev[q] = sm[1][q];
            st->gram[q] = sm[1][q];
            st->M[q] = 0.0;
            st->M[64 + q] = sm[2][q];
            st->M[128 + q] = 0.0;
            st->So[q] = ((q >> 3) == (q & 7) && (q >> 3) < s) ? 1.0 : 0.0;
          }
          st->step = 0;
          st->has_old = 0;
          st->flags = shifted ? KRY_FLAG_SHIFTED : 0;
        }
      }
      __syncthreads();
      break;
    }
    case POST_CHOL_MID:
      extract_block(total, 0, s, sm[0]);
      if (tid() == 0) {
        double mr = 0.0;
        s_bad = chol_upper(sm[0], sm[1], s, &mr);
        if (s_bad) {
          if (st->status == KRY_OK) st->status = KRY_ERR_DEFLATION;
        } else {
          inv_upper(sm[1], sm[2], s);
          for (int r = 0; r < 8; ++r)
            for (int c = 0; c < 8; ++c) {
              double v = 0.0;
              for (int k = 0; k < 8; ++k) v += sm[1][r * 8 + k] * st->gram[k * 8 + c];
              sm[3][r * 8 + c] = v;
            }
          for (int q = 0; q < 64; ++q) {
            st->M[q] = sm[2][q];
            st->gram[q] = sm[3][q];
            st->R1prev[q] = sm[3][q];
          }
          st->flags &= ~KRY_FLAG_SHIFTED;
        }
      }
      __syncthreads();
      break;
    case POST_GCC:
      extract_block(total, 0, s, sm[0]);
      if (tid() < 64) st->Gcc[tid()] = sm[0][tid()];
      __syncthreads();
      break;
    case POST_SCALE:
      extract_block(total, 0, s, sm[0]);
      if (tid() == 0) {
        st->scale2 = m_trace(sm[0], s);
        for (int q = 0; q < 64; ++q) { st->acc_a[q] = 0.0; st->acc_b[q] = 0.0; }
      }
      __syncthreads();
      break;
    case POST_MGS_OLD:
    case POST_MGS_CUR: {
      // raw g = V^T W ; true coefficient alpha = S^T g ; update matrix S alpha
      extract_block(total, 0, s, sm[0]);
      m_copy(sm[1], post == POST_MGS_OLD ? st->So : st->Sc);
      mm(sm[2], sm[1], 1, sm[0], 0, s);           // alpha
      mm(sm[3], sm[1], 0, sm[2], 0, s);           // S alpha
      if (tid() < 64) {
        double* acc = post == POST_MGS_OLD ? st->acc_a : st->acc_b;
        acc[tid()] += sm[2][tid()];
        st->M[tid()] = sm[3][tid()];
      }
      __syncthreads();
      break;
    }
    case POST_W2:
      extract_block(total, 0, s, sm[0]);
      if (tid() == 0) st->w2 = m_trace(sm[0], s);
      __syncthreads();
      break;
    case POST_CHOL1:
    case POST_CHOL2: {
      extract_block(total, 0, s, sm[0]);
      if (tid() == 0) {
        double mr = 0.0;
        s_bad = chol_upper(sm[0], sm[1], s, &mr);
        if (s_bad && post == POST_CHOL1) {
          // shifted CholQR3: the host runs POST_CHOL_MID before POST_CHOL2
          s_bad = chol_shifted(sm[0], sm[1], s, st->nrows);
          if (!s_bad) st->flags |= KRY_FLAG_SHIFTED;
        }
        if (s_bad) {
          if (st->status == KRY_OK) st->status = KRY_ERR_DEFLATION;
        } else {
          inv_upper(sm[1], sm[2], s);
          for (int q = 0; q < 64; ++q) st->M[q] = sm[2][q];
          if (post == POST_CHOL1) {
            for (int q = 0; q < 64; ++q) st->gram[q] = sm[1][q];   // R1
          } else {
            // R = R2 R1 ; rank test as kernels.py:151-160
            double fro = 0.0;
            for (int r = 0; r < 8; ++r)
              for (int c = 0; c < 8; ++c) {
                double v = 0.0;
                for (int k = 0; k < 8; ++k) v += sm[1][r * 8 + k] * st->gram[k * 8 + c];
                st->gram[64 + r * 8 + c] = v;
                fro += v * v;
              }
            fro = sqrt(fro);
            double mn = 1e300;
            for (int k = 0; k < s; ++k) mn = fmin(mn, fabs(st->gram[64 + k * 8 + k]));
            if (mn < 1e-12 * fro && st->status == KRY_OK) st->status = KRY_ERR_DEFLATION;
          }
        }
      }
      __syncthreads();
      break;
    }
    default:
      break;
  }
  (void)s_v;
}

// ------------------------------------------------------------------ grid reduction tail
template <int MP, int NW = 4>
__device__ void finish_reduction(const double (&acc)[MP / 8][2], double* sX, double* partials,
                                 unsigned* ticket, int post, DevState* st, const TStore& T) {
  constexpr int MT = MP / 8;
  constexpr int NE = MP * 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  __syncthreads();
  // per-warp tiles to smem: red[warp][m*8+n]
  double* red = sX;  // NW * NE doubles
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    red[warp * NE + (mt * 8 + g) * 8 + 2 * t] = acc[mt][0];
    red[warp * NE + (mt * 8 + g) * 8 + 2 * t + 1] = acc[mt][1];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    double v = red[e];
#pragma unroll
    for (int w = 1; w < NW; ++w) v += red[w * NE + e];
    partials[(int64_t)blockIdx.x * NE + e] = v;
  }
  __threadfence();
  __syncthreads();
  // Two-level deterministic grid reduction: the last CTA to finish in each
  // group of RG consecutive CTAs sums the group's partials in CTA order; the
  // last group to finish sums the group totals in group order.  The order of
  // every addition is fixed by the grid shape, never by arrival order (pass 2
  // reproduces pass 1 bit for bit), and each tail reads at most RG partials
  // with all loads in flight (a single-CTA sweep over ~1000 partials cost
  // 100+ us of one SM while the rest of the GPU idled).
  constexpr int RG = 32;
  __shared__ unsigned s_last;
  const int ngroups = (gridDim.x + RG - 1) / RG;
  const int grp = blockIdx.x / RG;
  const int g0 = grp * RG, gn = min(RG, (int)gridDim.x - g0);
  if (threadIdx.x == 0) {
    s_last = (atomicAdd(ticket + 1 + grp, 1u) == (unsigned)gn - 1) ? 1u : 0u;
    if (s_last) ticket[1 + grp] = 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double* gpart = partials + (int64_t)gridDim.x * NE;
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    const double* src = partials + (int64_t)g0 * NE + e;
    double v[RG];
#pragma unroll
    for (int b = 0; b < RG; ++b) v[b] = b < gn ? __ldcg(src + (int64_t)b * NE) : 0.0;
    double sum = v[0];
#pragma unroll
    for (int b = 1; b < RG; ++b) sum += v[b];
    gpart[(int64_t)grp * NE + e] = sum;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == (unsigned)ngroups - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double* total = sX;  // reuse: NE doubles
  __syncthreads();
  for (int e = threadIdx.x; e < NE; e += blockDim.x) {
    double sum = 0.0;
    for (int b0 = 0; b0 < ngroups; b0 += 16) {
      double v[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) v[b] = b0 + b < ngroups ? __ldcg(gpart + (int64_t)(b0 + b) * NE + e) : 0.0;
#pragma unroll
      for (int b = 0; b < 16; ++b) sum += v[b];
    }
    total[e] = sum;
  }
  for (int e = NE + threadIdx.x; e < 256; e += blockDim.x) total[e] = 0.0;
  constexpr int SMOFF = NE > 256 ? NE : 256;
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0u;
  // post routine on 8x8 smem scratch carved after `total`
  double(*sm)[64] = reinterpret_cast<double(*)[64]>(sX + SMOFF);
  run_post(post, total, st, T, sm);
}

// ------------------------------------------------------------------ kernels
// ------------------------------------------------------------------ fused hot kernels
// Stencil for the recurrence kernels: FMA form, constant coefficients folded
// per axis (w = cd v + cx (v_{x-1} + v_{x+1}) + cy (...) + cz (...)); the
// bit-exact CSR-order product is kept for the apply API (apply_point).
template <int S>
__device__ __forceinline__ void stencil_fast(const OpDev& op, const double* __restrict__ V,
                                             int64_t ld, int i, const double (&vi)[S],
                                             double (&w)[S]) {
  if (op.kind != KRY_OP_STENCIL) {
    apply_point<S>(op, V, ld, i, vi, w);
    return;
  }
  const int x = i % op.nx;
  const int r = i / op.nx;
  const int y = r % op.ny;
  const int z = r / op.ny;
  const bool hz0 = z > 0 || op.halo_lo, hy0 = y > 0, hx0 = x > 0;
  const bool hx1 = x < op.nx - 1, hy1 = y < op.ny - 1, hz1 = z < op.nzl - 1 || op.halo_hi;
  double n0[S], n1[S], n2[S], n3[S], n4[S], n5[S];
  load_vec<S>(V + (int64_t)(hz0 ? i - op.nxy : i) * ld, n0);
  load_vec<S>(V + (int64_t)(hy0 ? i - op.nx : i) * ld, n1);
  load_vec<S>(V + (int64_t)(hx0 ? i - 1 : i) * ld, n2);
  load_vec<S>(V + (int64_t)(hx1 ? i + 1 : i) * ld, n3);
  load_vec<S>(V + (int64_t)(hy1 ? i + op.nx : i) * ld, n4);
  load_vec<S>(V + (int64_t)(hz1 ? i + op.nxy : i) * ld, n5);
  if (!op.variable) {
#pragma unroll
    for (int a = 0; a < S; ++a) {
      const double sx = (hx0 ? n2[a] : 0.0) + (hx1 ? n3[a] : 0.0);
      const double sy = (hy0 ? n1[a] : 0.0) + (hy1 ? n4[a] : 0.0);
      const double sz = (hz0 ? n0[a] : 0.0) + (hz1 ? n5[a] : 0.0);
      w[a] = fma(op.cd, vi[a], fma(op.cz, sz, fma(op.cy, sy, op.cx * sx)));
    }
  } else {
    const double cz0 = hz0 ? __ldg(op.ez + i - op.nxy) : 0.0, cz1 = hz1 ? __ldg(op.ez + i) : 0.0;
    const double cy0 = hy0 ? __ldg(op.ey + i - op.nx) : 0.0, cy1 = hy1 ? __ldg(op.ey + i) : 0.0;
    const double cx0 = hx0 ? __ldg(op.ex + i - 1) : 0.0, cx1 = hx1 ? __ldg(op.ex + i) : 0.0;
    const double cd = __ldg(op.d + i);
#pragma unroll
    for (int a = 0; a < S; ++a) {
      double t = cd * vi[a];
      t = fma(cx0, n2[a], t);
      t = fma(cx1, n3[a], t);
      t = fma(cy0, n1[a], t);
      t = fma(cy1, n4[a], t);
      t = fma(cz0, n0[a], t);
      w[a] = fma(cz1, n5[a], t);
    }
  }
}

// L2 prefetch of a contiguous byte range by the TMA unit (no registers, no
// LSU traffic): the recurrence kernels call it for their NEXT tile, so every
// load of the current tile (centre rows and the +-x/y/z neighbours, which are
// centre rows of tiles at most one grid-stride ahead) hits L2 instead of
// waiting on DRAM.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_rows(const double* base, int64_t ld, int64_t row0,
                                              int64_t n) {
  if (base == nullptr || row0 >= n || row0 < 0) return;
  const int64_t rows = (row0 + TP <= n) ? TP : n - row0;
  const uint64_t a = reinterpret_cast<uint64_t>(base + row0 * ld);
  const uint64_t a0 = a & ~(uint64_t)15;
  const uint64_t bytes = ((a + rows * ld * 8 - a0) + 15) & ~(uint64_t)15;
  prefetch_l2(reinterpret_cast<const void*>(a0), (uint32_t)bytes);
}

// Tile order of the persistent recurrence kernels.  Default (KRY_CONTIG_TILES
// = 0): interleaved, tile = blockIdx + k * gridDim (the active tiles form a
// compact wavefront).  KRY_CONTIG_TILES = 1: each CTA walks a contiguous
// range, so the +-nx neighbour rows of a tile are rows this CTA loaded a
// moment ago (L1 hits instead of L2 fills); the +-nx*ny planes are the rows
// the CTAs a few ranges away are loading at the same time.
#ifndef KRY_CONTIG_TILES
#define KRY_CONTIG_TILES 0
#endif
struct TileOrder {
  int64_t n, per, base;
  __device__ explicit TileOrder(int64_t ntiles) : n(ntiles) {
    per = (ntiles + gridDim.x - 1) / gridDim.x;
    base = (int64_t)blockIdx.x * per;
  }
  __device__ bool valid(int64_t k) const {
    return KRY_CONTIG_TILES ? (k < per && base + k < n) : (blockIdx.x + k * (int64_t)gridDim.x < n);
  }
  __device__ int64_t at(int64_t k) const {
    return KRY_CONTIG_TILES ? base + k : blockIdx.x + k * (int64_t)gridDim.x;
  }
};

__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
// tile columns of the combine kernel: [V_{m-1} | V_m | A V_m | V_{m+1}] (+ zero padding
// read by the DMMA tiles)
__host__ __device__ constexpr int comb_cols(int S) {
  return cmax(cmax(4 * S, S + 8 * cdiv(3 * S, 8)), cmax(3 * S + 8, 4 * cdiv(3 * S, 4)));
}
__host__ __device__ constexpr int apply_cols(int S) { return cmax(cmax(2 * S, 8 * cdiv(2 * S, 8)), S + 8); }

// warp-level Gram over the warp's 32 tile rows:
// acc[mt] += X[:, x0 + 8mt .. +8]^T X[:, y0 .. y0+8]
template <int MT>
__device__ __forceinline__ void warp_gram(const double* sX, int r0, int x0, int y0,
                                          double (&acc)[MT][2]) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int k = r0 + ks * 4 + t;
    const double b = sX[CB(y0 + g) + k];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][0], acc[mt][1], sX[CB(x0 + mt * 8 + g) + k], b);
  }
}

// Cooperative, fully coalesced staging of one warp's 32 tile rows (S even,
// stencil operator): lane -> (point pp, 16-byte column pair cp); every warp
// load instruction covers 32 consecutive pieces (512 contiguous bytes when
// ld == S).  The stencil is evaluated per column pair and the results are
// written straight into the transposed smem tile:
//   column groups: [col_o: V_{m-1}] (if col_o >= 0), [col_c: V_m], [col_w: A V_m]
// `wout`: also store A V (apply kernel, for the combine that follows);
// `win`: load A V instead of gathering the stencil (combine kernel).
template <int S>
__device__ __forceinline__ void stage_warp_coop(const OpDev& op, const double* __restrict__ vc,
                                                int64_t ldc, const double* __restrict__ vo,
                                                int64_t ldo, bool load_old, bool use_op,
                                                int64_t n, int64_t tile_base, int r0,
                                                double* sX, int col_o, int col_c, int col_w,
                                                const double* __restrict__ win = nullptr,
                                                double* __restrict__ wout = nullptr) {
  constexpr int CP = S / 2;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < CP; ++e) {
    const int q = lane + 32 * e;
    const int pp = q / CP, cp = q % CP;
    const int row = r0 + pp;
    const int64_t i64 = tile_base + row;
    double2 o = make_double2(0.0, 0.0), v = make_double2(0.0, 0.0), w = make_double2(0.0, 0.0);
    if (i64 < n) {
      const int i = (int)i64;
      const int off = 2 * cp;
      v = __ldg(reinterpret_cast<const double2*>(vc + i64 * ldc + off));
      if (load_old) o = __ldg(reinterpret_cast<const double2*>(vo + i64 * ldo + off));
      if (use_op && win) {
        w = __ldg(reinterpret_cast<const double2*>(win + i64 * S + off));
      } else if (use_op) {
        const unsigned r = fdiv((unsigned)i, op.fx);
        const int x = i - (int)r * op.nx;
        const unsigned zq = fdiv(r, op.fy);
        const int y = (int)r - (int)zq * op.ny;
        const int z = (int)zq;
        const bool hz0 = z > 0 || op.halo_lo, hy0 = y > 0, hx0 = x > 0;
        const bool hx1 = x < op.nx - 1, hy1 = y < op.ny - 1, hz1 = z < op.nzl - 1 || op.halo_hi;
        // one 64-bit base, neighbours by (32-bit) element deltas
        const double2* pc = reinterpret_cast<const double2*>(vc + i64 * ldc + off);
        const int dx = (int)ldc / 2, dy = op.nx * (int)ldc / 2, dz = op.nxy * (int)ldc / 2;
        const double2 n0 = __ldg(pc - (hz0 ? dz : 0)), n1 = __ldg(pc - (hy0 ? dy : 0));
        const double2 n4 = __ldg(pc + (hy1 ? dy : 0)), n5 = __ldg(pc + (hz1 ? dz : 0));
        const double2 n2 = __ldg(pc - (hx0 ? dx : 0)), n3 = __ldg(pc + (hx1 ? dx : 0));
        if (!op.variable) {
          const double sx0 = (hx0 ? n2.x : 0.0) + (hx1 ? n3.x : 0.0);
          const double sx1 = (hx0 ? n2.y : 0.0) + (hx1 ? n3.y : 0.0);
          const double sy0 = (hy0 ? n1.x : 0.0) + (hy1 ? n4.x : 0.0);
          const double sy1 = (hy0 ? n1.y : 0.0) + (hy1 ? n4.y : 0.0);
          const double sz0 = (hz0 ? n0.x : 0.0) + (hz1 ? n5.x : 0.0);
          const double sz1 = (hz0 ? n0.y : 0.0) + (hz1 ? n5.y : 0.0);
          w.x = fma(op.cd, v.x, fma(op.cz, sz0, fma(op.cy, sy0, op.cx * sx0)));
          w.y = fma(op.cd, v.y, fma(op.cz, sz1, fma(op.cy, sy1, op.cx * sx1)));
        } else {
          const double cz0 = hz0 ? __ldg(op.ez + i - op.nxy) : 0.0, cz1 = hz1 ? __ldg(op.ez + i) : 0.0;
          const double cy0 = hy0 ? __ldg(op.ey + i - op.nx) : 0.0, cy1 = hy1 ? __ldg(op.ey + i) : 0.0;
          const double cx0 = hx0 ? __ldg(op.ex + i - 1) : 0.0, cx1 = hx1 ? __ldg(op.ex + i) : 0.0;
          const double cd = __ldg(op.d + i);
          double t0 = cd * v.x, t1 = cd * v.y;
          t0 = fma(cx0, n2.x, t0); t1 = fma(cx0, n2.y, t1);
          t0 = fma(cx1, n3.x, t0); t1 = fma(cx1, n3.y, t1);
          t0 = fma(cy0, n1.x, t0); t1 = fma(cy0, n1.y, t1);
          t0 = fma(cy1, n4.x, t0); t1 = fma(cy1, n4.y, t1);
          t0 = fma(cz0, n0.x, t0); t1 = fma(cz0, n0.y, t1);
          w.x = fma(cz1, n5.x, t0); w.y = fma(cz1, n5.y, t1);
        }
      }
    }
    const int c0 = 2 * cp;
    if (wout && use_op && i64 < n) *reinterpret_cast<double2*>(wout + i64 * S + c0) = w;
    if (col_o >= 0) {
      sX[CB(col_o + c0) + row] = o.x;
      sX[CB(col_o + c0 + 1) + row] = o.y;
    }
    sX[CB(col_c + c0) + row] = v.x;
    sX[CB(col_c + c0 + 1) + row] = v.y;
    if (col_w >= 0) {
      sX[CB(col_w + c0) + row] = w.x;
      sX[CB(col_w + c0 + 1) + row] = w.y;
    }
  }
}

// Combine: V_{m+1} = [V_{m-1} | V_m | A V_m] * [Mo; Mc; Mw]  on DMMA tensor
// cores, then the Gram [V_m | A V_m | V_{m+1}]^T V_{m+1}.  Each warp owns 32
// rows of the tile, so a tile needs only warp-level synchronisation.
template <int S, bool COOP>
#ifndef KRY_COMB_MINB
#define KRY_COMB_MINB 5
#endif
// resident CTAs per SM of the combine kernel (0 = occupancy limit); a cap
// leaves room for the eigen stream's kernels next to the HBM-bound combine
#ifndef KRY_COMB_CAP
#define KRY_COMB_CAP 0
#endif
#ifndef KRY_APPLY_MINB
#define KRY_APPLY_MINB 8
#endif
__global__ void __launch_bounds__(TP, COOP ? KRY_COMB_MINB : 2) k_combine(OpDev op, CombineCall c, DevState* st,
                                                TStore T, double* partials, unsigned* ticket) {
  constexpr int XC = comb_cols(S);
  constexpr int MTG = cdiv(3 * S, 8);   // Gram m-tiles (rows of [V_m | AV | V_{m+1}])
  constexpr int MP = 8 * MTG;
  constexpr int KS = cdiv(3 * S, 4);    // combination k-steps
  __shared__ __align__(16) double sX[XC * LDP];
  if (st->status != KRY_OK || (st->flags & (KRY_FLAG_FALLBACK | KRY_FLAG_EXHAUSTED))) {
    if (c.write_new) return;  // never combine with invalid coefficients
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  // B fragments of the stacked coefficient matrix [Mo; Mc; Mw] (3S x S)
  double bM[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int kk = 4 * ks + t;
    double v = 0.0;
    if (kk < 3 * S && g < S) v = st->M[(kk / S) * 64 + (kk % S) * 8 + g];
    bM[ks] = v;
  }
  for (int e = 0; e < XC; ++e) sX[CB(e) + threadIdx.x] = 0.0;
  double acc[MTG][2];
#pragma unroll
  for (int mt = 0; mt < MTG; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
  __syncthreads();
  const int64_t ntiles = (c.n + TP - 1) / TP;
  const int r0 = warp * 32;
  double* row = sX + threadIdx.x;   // column q at row[CB(q)]
  constexpr bool coop = COOP && (S % 2 == 0);
  // interleaved tile order: the active tiles form a compact wavefront, so the
  // +-nx*ny neighbour planes of a tile are in L2 (streamed as centre rows by
  // the CTAs ~nx*ny/TP tiles ahead / behind)
  const TileOrder ord(ntiles);
  for (int64_t k = 0; ord.valid(k); ++k) {
    const int64_t it = ord.at(k);
    const int64_t tile = c.reverse ? (ntiles - 1 - it) : it;
    const int64_t i64 = tile * TP + threadIdx.x;
    if (threadIdx.x == 0 && ord.valid(k + 1)) {
      const int64_t nx_ = ord.at(k + 1);
      const int64_t nt = c.reverse ? (ntiles - 1 - nx_) : nx_;
      prefetch_rows(c.vc, c.ldc, nt * TP, c.n);
      if (c.write_new && c.has_old) prefetch_rows(c.vo, c.ldo, nt * TP, c.n);
      if (!c.write_new) prefetch_rows(c.vn, c.ldn, nt * TP, c.n);
    }
    if constexpr (coop) {
      stage_warp_coop<(S % 2 == 0) ? S : 2>(op, c.vc, c.ldc, c.vo, c.ldo, c.write_new && c.has_old,
                                            c.use_op, c.n, tile * TP, r0, sX, 0, S, 2 * S, c.win);
      if (!c.write_new && i64 < c.n) {
        double vn[S];
        load_vec<S>(c.vn + i64 * c.ldn, vn);
#pragma unroll
        for (int a = 0; a < S; ++a) row[CB(3 * S + a)] = vn[a];
      }
    } else if (i64 < c.n) {
      const int i = (int)i64;
      if (c.write_new && c.has_old) {
        double vo[S];
        load_vec<S>(c.vo + i64 * c.ldo, vo);
#pragma unroll
        for (int a = 0; a < S; ++a) row[CB(a)] = vo[a];
      } else {
#pragma unroll
        for (int a = 0; a < S; ++a) row[CB(a)] = 0.0;
      }
      double vc[S], w[S];
      load_vec<S>(c.vc + i64 * c.ldc, vc);
      if (c.use_op) {
        stencil_fast<S>(op, c.vc, c.ldc, i, vc, w);
      } else {
#pragma unroll
        for (int a = 0; a < S; ++a) w[a] = 0.0;
      }
#pragma unroll
      for (int a = 0; a < S; ++a) {
        row[CB(S + a)] = vc[a];
        row[CB(2 * S + a)] = w[a];
      }
      if (!c.write_new) {
        double vn[S];
        load_vec<S>(c.vn + i64 * c.ldn, vn);
#pragma unroll
        for (int a = 0; a < S; ++a) row[CB(3 * S + a)] = vn[a];
      }
    } else {
#pragma unroll
      for (int a = 0; a < 4 * S; ++a) row[CB(a)] = 0.0;
    }
    __syncwarp();
    if (c.write_new) {
      // V_{m+1} for the warp's 32 rows: 4 m-tiles of 8 points x KS k-steps
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        double d0 = 0.0, d1 = 0.0;
        const int pr = r0 + mt * 8 + g;   // A row = point
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) dmma(d0, d1, sX[CB(4 * ks + t) + pr], bM[ks]);
        const int64_t pi = tile * TP + pr;
        const int c0 = 2 * t;
        if (c0 < S) {
          sX[CB(3 * S + c0) + pr] = d0;
          if (c0 + 1 < S) sX[CB(3 * S + c0 + 1) + pr] = d1;
          if (pi < c.n) {
            double* dst = c.vn + pi * c.ldn + c0;
            if constexpr (S % 2 == 0) {
              *reinterpret_cast<double2*>(dst) = make_double2(d0, d1);
            } else {
              dst[0] = d0;
              if (c0 + 1 < S) dst[1] = d1;
            }
            if (c.vn2) {
              double* d2 = c.vn2 + pi * c.ldn2 + c0;
              if constexpr (S % 2 == 0) {
                __stcs(reinterpret_cast<double2*>(d2), make_double2(d0, d1));
              } else {
                __stcs(d2, d0);
                if (c0 + 1 < S) __stcs(d2 + 1, d1);
              }
            }
          }
        }
      }
      __syncwarp();
    }
    warp_gram<MTG>(sX, r0, S, 3 * S, acc);
    __syncwarp();
  }
  finish_reduction<MP>(acc, sX, partials, ticket, c.post, st, T);
}

// Apply + Gram: X = [V | A V], Y = A V  (use_op) or X = [V], Y = V
template <int S, int USE_OP, bool COOP>
__global__ void __launch_bounds__(TP, COOP ? KRY_APPLY_MINB : 2) k_apply_gram(OpDev op, ApplyGramCall c, DevState* st,
                                                   TStore T, double* partials, unsigned* ticket) {
  constexpr int NG = USE_OP ? 2 : 1;
  constexpr int XC = apply_cols(S);
  constexpr int MT = cdiv(NG * S, 8);
  constexpr int MP = 8 * MT;
  __shared__ __align__(16) double sX[cmax(XC, 9) * LDP];
  for (int e = 0; e < XC; ++e) sX[CB(e) + threadIdx.x] = 0.0;
  double acc[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
  __syncthreads();
  const int64_t ntiles = (c.n + TP - 1) / TP;
  const int r0 = (threadIdx.x >> 5) * 32;
  double* row = sX + threadIdx.x;
  constexpr bool coop = COOP && (S % 2 == 0);
  // interleaved tile order: the active tiles form a compact wavefront, so the
  // +-nx*ny neighbour planes of a tile are in L2 (streamed as centre rows by
  // the CTAs ~nx*ny/TP tiles ahead / behind)
  const TileOrder ord(ntiles);
  for (int64_t k = 0; ord.valid(k); ++k) {
    const int64_t it = ord.at(k);
    const int64_t tile = c.reverse ? (ntiles - 1 - it) : it;
    const int64_t i64 = tile * TP + threadIdx.x;
    if (threadIdx.x == 0 && ord.valid(k + 1)) {
      const int64_t nx_ = ord.at(k + 1);
      const int64_t nt = c.reverse ? (ntiles - 1 - nx_) : nx_;
      prefetch_rows(c.v, c.ldv, nt * TP, c.n);
    }
    if constexpr (coop) {
      stage_warp_coop<(S % 2 == 0) ? S : 2>(op, c.v, c.ldv, nullptr, 0, false, USE_OP != 0, c.n,
                                            tile * TP, r0, sX, -1, 0, USE_OP ? S : -1, nullptr,
                                            c.wout);
    } else if (i64 < c.n) {
      double v[S];
      load_vec<S>(c.v + i64 * c.ldv, v);
#pragma unroll
      for (int a = 0; a < S; ++a) row[CB(a)] = v[a];
      if constexpr (USE_OP) {
        double w[S];
        stencil_fast<S>(op, c.v, c.ldv, (int)i64, v, w);
#pragma unroll
        for (int a = 0; a < S; ++a) row[CB(S + a)] = w[a];
      }
    } else {
#pragma unroll
      for (int a = 0; a < NG * S; ++a) row[CB(a)] = 0.0;
    }
    __syncwarp();
    warp_gram<MT>(sX, r0, 0, (NG - 1) * S, acc);
    __syncwarp();
  }
  finish_reduction<MP>(acc, sX, partials, ticket, c.post, st, T);
}

// Pair Gram X^T Y for two blocks (explicit path)
template <int S>
__global__ void __launch_bounds__(TP) k_pair_gram(const double* x, int64_t ldx, const double* y,
                                                  int64_t ldy, int64_t n, int post, DevState* st,
                                                  TStore T, double* partials, unsigned* ticket) {
  constexpr int W = 2 * S;
  constexpr int MP = (W + 7) / 8 * 8;
  constexpr int MT = MP / 8;
  __shared__ __align__(16) double sX[XCOLS * LDP];
  for (int e = 0; e < XCOLS; ++e) sX[CB(e) + threadIdx.x] = 0.0;
  double acc[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
  __syncthreads();
  const int64_t ntiles = (n + TP - 1) / TP;
  const int warp = threadIdx.x >> 5;
  for (int64_t it = blockIdx.x; it < ntiles; it += gridDim.x) {
    const int64_t i64 = it * TP + threadIdx.x;
    double* row = sX + threadIdx.x;   // column c at row[CB(c)]
    if (i64 < n) {
      double v[S], w[S];
      load_vec<S>(x + i64 * ldx, v);
      load_vec<S>(y + i64 * ldy, w);
#pragma unroll
      for (int a = 0; a < S; ++a) {
        row[CB(a)] = v[a];
        row[CB(S + a)] = w[a];
      }
    } else {
#pragma unroll
      for (int a = 0; a < W; ++a) row[CB(a)] = 0.0;
    }
    __syncthreads();
    tile_gram<MT>(sX, warp * 32, S, acc);
    __syncthreads();
  }
  finish_reduction<MP>(acc, sX, partials, ticket, post, st, T);
}

template <int S>
__global__ void k_apply_store(OpDev op, const double* x, int64_t ldx, double* y, int64_t ldy,
                              int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v[S], w[S];
    load_vec<S>(x + i * ldx, v);
    apply_point<S>(op, x, ldx, (int)i, v, w);
    store_vec<S>(y + i * ldy, w);
  }
}

// w = w - x M (subtract) or w = w M (x == nullptr)
template <int S>
__global__ void k_update(double* w, int64_t ldw, const double* x, int64_t ldx, const double* mdev,
                         int64_t n, int subtract) {
  __shared__ double sM[64];
  if (threadIdx.x < 64) sM[threadIdx.x] = mdev[threadIdx.x];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double wv[S], out[S];
    load_vec<S>(w + i * ldw, wv);
    if (x) {
      double xv[S];
      load_vec<S>(x + i * ldx, xv);
#pragma unroll
      for (int a = 0; a < S; ++a) {
        double t = 0.0;
#pragma unroll
        for (int b = 0; b < S; ++b) t = fma(xv[b], sM[b * 8 + a], t);
        out[a] = subtract ? wv[a] - t : wv[a] + t;
      }
    } else {
#pragma unroll
      for (int a = 0; a < S; ++a) {
        double t = 0.0;
#pragma unroll
        for (int b = 0; b < S; ++b) t = fma(wv[b], sM[b * 8 + a], t);
        out[a] = t;
      }
    }
    store_vec<S>(w + i * ldw, out);
  }
}

template <int S>
__global__ void k_copy_block(const double* x, int64_t ldx, double* y, int64_t ldy, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v[S];
    load_vec<S>(x + i * ldx, v);
    store_vec<S>(y + i * ldy, v);
  }
}

// explicit-path bookkeeping (1 CTA of 64 threads)
__global__ void k_explicit_finish(DevState* st, TStore T, int mode) {
  const int q = threadIdx.x;
  const int s = st->s;
  const int j = st->step + 1;
  const int r = q >> 3, c = q & 7;
  if (mode == 0) {
    // zero residual block: exhausted (finalize mode)
    const int64_t o = (int64_t)(j - 1) * 64;
    if (!st->replay) {
      T.draw[o + q] = st->acc_b[q];
      T.dsym[o + q] = 0.5 * (st->acc_b[r * 8 + c] + st->acc_b[c * 8 + r]);
      T.off[o + q] = st->has_old ? st->acc_a[q] : 0.0;
      T.sub[o + q] = 0.0;
      T.tau1[o + q] = 0.0;
    }
    T.S[o + q] = st->Sc[q];
    __syncthreads();
    if (q == 0) {
      st->flags = KRY_FLAG_EXHAUSTED;
      st->step = j;
    }
  } else {
    // regular explicit step: R = R2 R1 in st->gram[64..], V_new orthonormal
    const int64_t o = (int64_t)(j - 1) * 64;
    if (!st->replay) {
      T.draw[o + q] = st->acc_b[q];
      T.dsym[o + q] = 0.5 * (st->acc_b[r * 8 + c] + st->acc_b[c * 8 + r]);
      T.off[o + q] = st->has_old ? st->acc_a[q] : 0.0;
    }
    T.S[o + q] = st->Sc[q];
    st->R1prev[q] = st->gram[64 + q];
    T.tau1[o + q] = st->gram[64 + q];
    st->So[q] = st->Sc[q];
    st->Goo[q] = st->Gcc[q];
    __syncthreads();
    if (q == 0) {
      st->flags = 0;
      st->step = j;
      st->has_old = 1;
    }
  }
  (void)s;
}

// ------------------------------------------------------------------ launchers
int gram_grid_for(int64_t n) {
  int64_t tiles = (n + TP - 1) / TP;
  int64_t g = KRY_MAX_GRID;
  if (tiles < g) g = tiles;
  if (g < 1) g = 1;
  return (int)g;
}

// persistent grid = resident CTAs (occupancy x SMs), capped by the tile count,
// so the grid-stride tile loop runs in exactly one wave
template <class Kern>
static int resident_grid(Kern kernel, int64_t n, int cap_per_sm = 0) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache[64];   // per device
  int per_sm = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto& cd = cache[dev & 63];
    auto it = cd.find((const void*)kernel);
    if (it == cd.end()) {
      int sms = 148, nb = 1;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, TP, 0);
      if (cap_per_sm > 0) nb = std::min(nb, cap_per_sm);
      per_sm = std::max(1, nb) * sms;
      cd[(const void*)kernel] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  int64_t tiles = (n + TP - 1) / TP;
  int64_t g = std::min<int64_t>(std::min<int64_t>(tiles, per_sm), KRY_MAX_GRID);
  return (int)std::max<int64_t>(g, 1);
}

#define KRY_DISPATCH_S(s, F)                                        \
  switch (s) {                                                      \
    case 1: F(1); break;                                            \
    case 2: F(2); break;                                            \
    case 3: F(3); break;                                            \
    case 4: F(4); break;                                            \
    case 5: F(5); break;                                            \
    case 6: F(6); break;                                            \
    case 7: F(7); break;                                            \
    case 8: F(8); break;                                            \
    default: return fail(KRY_ERR_ARGUMENT, "block width s must be 1..8"); \
  }

int launch_combine(cudaStream_t st, int s, const OpDev& op, const CombineCall& c, DevState* dst,
                   const TStore& T, GramScratch& g, int grid, float* prof_ms, cudaEvent_t* ev) {
  (void)grid;
  if (prof_ms && ev) cudaEventRecord(ev[0], st);
  const bool coop = (s % 2 == 0) && op.kind == KRY_OP_STENCIL && (c.ldc % 2 == 0) &&
                    (!c.has_old || c.ldo % 2 == 0);
  auto capped = [&](int gr) { return c.grid_cap > 0 ? std::min(gr, c.grid_cap) : gr; };
  if (coop) {
#define L(S)                                                                 \
  k_combine<S, true><<<capped(resident_grid(k_combine<S, true>, c.n, KRY_COMB_CAP)), TP, 0, st>>>( \
      op, c, dst, T, g.partials, g.ticket + 0)
    KRY_DISPATCH_S(s, L);
#undef L
  } else {
#define L(S)                                                                   \
  k_combine<S, false><<<capped(resident_grid(k_combine<S, false>, c.n)), TP, 0, st>>>( \
      op, c, dst, T, g.partials, g.ticket + 0)
    KRY_DISPATCH_S(s, L);
#undef L
  }
  if (prof_ms && ev) cudaEventRecord(ev[1], st);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

int launch_apply_gram(cudaStream_t st, int s, const OpDev& op, const ApplyGramCall& c,
                      DevState* dst, const TStore& T, GramScratch& g, int grid) {
  (void)grid;
  const bool coop = (s % 2 == 0) && (op.kind == KRY_OP_STENCIL || !c.use_op) && (c.ldv % 2 == 0);
  auto capped = [&](int gr) { return c.grid_cap > 0 ? std::min(gr, c.grid_cap) : gr; };
#define LA(S, U, C)                                                                    \
  k_apply_gram<S, U, C><<<capped(resident_grid(k_apply_gram<S, U, C>, c.n)), TP, 0, st>>>( \
      op, c, dst, T, g.partials, g.ticket + 1 * KRY_TICKET_STRIDE)
  if (c.use_op && coop) {
#define L(S) LA(S, 1, true)
    KRY_DISPATCH_S(s, L);
#undef L
  } else if (c.use_op) {
#define L(S) LA(S, 1, false)
    KRY_DISPATCH_S(s, L);
#undef L
  } else if (coop) {
#define L(S) LA(S, 0, true)
    KRY_DISPATCH_S(s, L);
#undef L
  } else {
#define L(S) LA(S, 0, false)
    KRY_DISPATCH_S(s, L);
#undef L
  }
#undef LA
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

int launch_pair_gram(cudaStream_t st, int s, const double* x, int64_t ldx, const double* y,
                     int64_t ldy, int64_t n, int post, DevState* dst, const TStore& T,
                     GramScratch& g, int grid) {
  (void)grid;
#define L(S)                                                       \
  k_pair_gram<S><<<resident_grid(k_pair_gram<S>, n), TP, 0, st>>>( \
      x, ldx, y, ldy, n, post, dst, T, g.partials, g.ticket + 2 * KRY_TICKET_STRIDE)
  KRY_DISPATCH_S(s, L);
#undef L
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

static int ew_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

int launch_apply_store(cudaStream_t st, int s, const OpDev& op, const double* x, int64_t ldx,
                       double* y, int64_t ldy, int64_t n) {
#define L(S) k_apply_store<S><<<ew_grid(n), 256, 0, st>>>(op, x, ldx, y, ldy, n)
  KRY_DISPATCH_S(s, L);
#undef L
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

int launch_update(cudaStream_t st, int s, double* w, int64_t ldw, const double* x, int64_t ldx,
                  const double* mdev, int64_t n, int subtract) {
#define L(S) k_update<S><<<ew_grid(n), 256, 0, st>>>(w, ldw, x, ldx, mdev, n, subtract)
  KRY_DISPATCH_S(s, L);
#undef L
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

int launch_copy_block(cudaStream_t st, int s, const double* x, int64_t ldx, double* y,
                      int64_t ldy, int64_t n) {
#define L(S) k_copy_block<S><<<ew_grid(n), 256, 0, st>>>(x, ldx, y, ldy, n)
  KRY_DISPATCH_S(s, L);
#undef L
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

__global__ void __launch_bounds__(128) k_post(int post, DevState* st, TStore T) {
  __shared__ double buf[256 + 14 * 64];
  for (int e = threadIdx.x; e < 256; e += blockDim.x) buf[e] = e < 3 * 64 ? st->gram[e] : 0.0;
  __syncthreads();
  run_post(post, buf, st, T, reinterpret_cast<double(*)[64]>(buf + 256));
}

int launch_post(cudaStream_t st, int post, DevState* dst, const TStore& T) {
  k_post<<<1, 128, 0, st>>>(post, dst, T);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

int launch_explicit_finish(cudaStream_t st, DevState* dst, const TStore& T, int mode) {
  k_explicit_finish<<<1, 64, 0, st>>>(dst, T, mode);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

#include "step.cuh"



}  // namespace kry
