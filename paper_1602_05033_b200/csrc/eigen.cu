// Eigen data of the growing block-tridiagonal T_m and the cheap residual
// norm (sm_100a, fp64).
//
// Reference: partial_eig_blocktridiag (kernels.py:296-306) = band reduction
// (kernels.py:184-261, pure-Python Givens bulge chase) + tridiagonal
// eigensolver (kernels.py:264-293), recomputed from scratch at every check,
// then ctri_lyapunov / ctri_sylvester (residual.py:40-84).
//
// B200 design: T_m only ever grows by one block row (it is the leading
// principal submatrix of T_{m+1}), so its eigen data are UPDATED instead of
// recomputed.  Each scalar row k appended to T (bandwidth s, the couplings
// live in the last s rows) turns the current eigenbasis into a bordered
// (arrowhead) matrix  [diag(lam), z; z^T, d]  with z = L^T t, where L holds
// the last s rows of the eigenvector matrix.  Its eigenpairs are obtained by
// the Gu-Eisenstat scheme:
//   E1 deflation (negligible z_j; Givens rotation of numerically equal poles)
//   E2 secular equation  h(mu) = mu - d - sum z_j^2/(mu - lam_j)  for every
//      root in parallel (rational two-pole iteration, origin at the nearer
//      pole so mu - lam_j is formed without cancellation)
//   E3 recomputed zhat_j^2 = -prod_i(lam_j - mu_i)/prod_{i!=j}(lam_j - lam_i)
//      (guarantees numerically orthogonal eigenvectors)
//   E4 eigenvectors v_i = [zhat_j/(mu_i - lam_j); 1]/norm applied to the
//      tracked first s and last s rows, merged in sorted order.
// Only lam (k), the first s rows F and the last s rows L of Q are stored,
// O(s k) memory; an append costs O(s k^2) flops, fully parallel.
// The residual is the fused Cauchy contraction
//   M = ((u u^T) o C) w,  C_ij = 1/(lam_i + lam_j),  u = F^T gamma, w = L^T tau^T
#include "kry_internal.cuh"
#include "eigen.cuh"
#include "dense.cuh"
#include <cstring>
#include <mutex>
#include <cmath>
#include <vector>
#include <algorithm>

namespace kry {

static constexpr double EPS = 2.220446049250313e-16;

// ------------------------------------------------------------------ block scan helpers
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
// exclusive scan over the block; returns the prefix, *total = block sum
__device__ int block_excl_scan(int v, int* total) {
  __shared__ int s_w[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  int inc = warp_incl_scan(v);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int x = (lane < nw) ? s_w[lane] : 0;
    int xi = warp_incl_scan(x);
    if (lane < nw) s_w[lane] = xi - x;
    if (lane == 31) s_w[32] = xi;
  }
  __syncthreads();
  int res = inc - v + s_w[warp];
  *total = s_w[32];
  __syncthreads();
  return res;
}

__device__ double block_max(double v) {
  __shared__ double s_r[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) s_r[warp] = v;
  __syncthreads();
  double r = 0.0;
  const int nw = blockDim.x >> 5;
  for (int q = 0; q < nw; ++q) r = fmax(r, s_r[q]);
  __syncthreads();
  return r;
}
__device__ double block_sum(double v) {
  __shared__ double s_r[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_r[warp] = v;
  __syncthreads();
  double r = 0.0;
  const int nw = blockDim.x >> 5;
  for (int q = 0; q < nw; ++q) r += s_r[q];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ E1: coupling + deflation (1 CTA x 1024)
// The per-pole work arrays (z, candidate list, flags) live in shared memory
// when they fit (SM = true): the passes below are chains of dependent
// accesses, and each global round trip costs ~1 us on this single CTA.
// Every thread owns a contiguous segment of C = ceil(K / 1024) poles, so each
// compaction pass is ONE block scan of the per-thread counts (the first
// version scanned 1024-pole chunks one after the other: ~30 barriers per
// call, 22 us at K = 4000, barrier-stalled).
template <bool SM>
__global__ void __launch_bounds__(1024) k_eig_deflate(EigView e, int K, const double* dsym_blk,
                                                      const double* sub_prev, int a) {
  pdl_sync();
  extern __shared__ double dyn_sm[];
  if (SM) {
    e.z = dyn_sm;
    e.cand = reinterpret_cast<int*>(dyn_sm + K);
    e.dflag = e.cand + K;
    e.pflag = e.dflag + K;
  }
  const int s = e.s;
  __shared__ double t[KRY_SMAX];
  __shared__ double s_d, s_tol;
  if (threadIdx.x < s) {
    const int r = threadIdx.x;
    double v;
    if (r < s - a) v = sub_prev ? sub_prev[a * 8 + (a + r)] : 0.0;   // tau[a][a+r]
    else v = dsym_blk[a * 8 + (r - (s - a))];                          // D[a][c], c < a
    t[r] = v;
  }
  if (threadIdx.x == 0) s_d = dsym_blk[a * 8 + a];
  __syncthreads();
  const double d = s_d;
  const int C = (K + blockDim.x - 1) / blockDim.x;
  const int j0 = min(K, (int)threadIdx.x * C), j1 = min(K, j0 + C);
  double zmax = 0.0, zabs = 0.0;
  for (int j = j0; j < j1; ++j) {
    double z = 0.0;
    for (int r = 0; r < s; ++r) z = fma(e.L_old[(int64_t)r * e.kmax + j], t[r], z);
    e.z[j] = z;
    zmax = fmax(zmax, fabs(z));
    zabs += fabs(z);
  }
  zmax = block_max(zmax);
  zabs = block_sum(zabs);
  if (threadIdx.x == 0) {
    double lm = 0.0;
    if (K > 0) lm = fmax(fabs(e.lam_old[0]), fabs(e.lam_old[K - 1]));
    s_tol = 8.0 * EPS * fmax(fmax(lm, fabs(d)), zmax);
    e.scal[0] = d;
    e.scal[1] = s_tol;
    e.scal[2] = zabs;
  }
  __syncthreads();
  const double tol = s_tol;
  // pass 1: candidates = non-negligible z, compacted in eigenvalue order
  int q;
  {
    int cnt = 0;
    for (int j = j0; j < j1; ++j) cnt += (fabs(e.z[j]) > tol) ? 1 : 0;
    int pos = block_excl_scan(cnt, &q);
    for (int j = j0; j < j1; ++j) {
      const int keep = fabs(e.z[j]) > tol;
      if (keep) e.cand[pos++] = j;
      e.dflag[j] = keep ? 0 : 1;
    }
  }
  __syncthreads();
  // pass 2: pairs of consecutive candidates whose Givens rotation decouples
  // one of them (LAPACK dlaed2's rule: |t c s| <= tol)
  for (int i = 1 + threadIdx.x; i < q; i += blockDim.x) {
    const int ja = e.cand[i - 1], jb = e.cand[i];
    const double za = e.z[ja], zb = e.z[jb];
    const double r = hypot(za, zb);
    const double cth = zb / r, sth = za / r;
    const double tt = e.lam_old[jb] - e.lam_old[ja];
    e.pflag[i] = (fabs(tt * cth * sth) <= tol) ? 1 : 0;
  }
  if (threadIdx.x == 0 && q > 0) e.pflag[0] = 0;
  __syncthreads();
  // runs of flagged pairs are processed sequentially (one thread per run)
  for (int i = 1 + threadIdx.x; i < q; i += blockDim.x) {
    if (!e.pflag[i] || e.pflag[i - 1]) continue;
    if (e.stats) {
      int len = 0;
      for (int k = i; k < q && e.pflag[k]; ++k) ++len;
      atomicAdd(e.stats + 130, 1u);                       // runs
      atomicAdd(e.stats + 131, (unsigned)len);            // rotated pairs
      atomicMax(e.stats + 132, (unsigned)len);            // longest run
    }
    int prev = e.cand[i - 1];
    for (int k = i; k < q && e.pflag[k]; ++k) {
      const int cur = e.cand[k];
      const double za = e.z[prev], zb = e.z[cur];
      const double r = hypot(za, zb);
      const double cth = zb / r, sth = za / r;
      const double tt = e.lam_old[cur] - e.lam_old[prev];
      if (fabs(tt * cth * sth) <= tol) {
        const double l1 = e.lam_old[prev], l2 = e.lam_old[cur];
        e.lam_old[prev] = cth * cth * l1 + sth * sth * l2;
        e.lam_old[cur] = sth * sth * l1 + cth * cth * l2;
        e.z[prev] = 0.0;
        e.z[cur] = r;
        for (int rr = 0; rr < s; ++rr) {
          double* F = e.F_old + (int64_t)rr * e.kmax;
          double* L = e.L_old + (int64_t)rr * e.kmax;
          const double fa = F[prev], fb = F[cur];
          F[prev] = cth * fa - sth * fb;
          F[cur] = sth * fa + cth * fb;
          const double la = L[prev], lb = L[cur];
          L[prev] = cth * la - sth * lb;
          L[cur] = sth * la + cth * lb;
        }
        e.dflag[prev] = 1;
      }
      prev = cur;
    }
  }
  __syncthreads();
  // pass 3: final poles and deflated list (one scan of the packed counts)
  int pb, db;
  {
    int np = 0, nd = 0;
    for (int j = j0; j < j1; ++j) {
      if (e.dflag[j]) ++nd; else ++np;
    }
    int tot;
    const int pre = block_excl_scan(np | (nd << 16), &tot);
    int pp = pre & 0xffff, pd = pre >> 16;
    pb = tot & 0xffff;
    db = tot >> 16;
    if (K >= 65536) {   // counts do not fit 16 bits: two scans
      pp = block_excl_scan(np, &pb);
      pd = block_excl_scan(nd, &db);
    }
    for (int j = j0; j < j1; ++j) {
      if (e.dflag[j]) {
        e.def_idx[pd] = j;
        e.def_lam[pd] = e.lam_old[j];
        ++pd;
      } else {
        e.poles[pp] = e.lam_old[j];
        e.zz[pp] = e.z[j];
        e.pmap[pp] = j;
        ++pp;
      }
    }
  }
  __syncthreads();
  // rotated deflations can break the order of the deflated list locally;
  // the (usually sorted) list is checked by the whole block, and only a
  // disordered one goes through the serial insertion-sort fix-up
  int unsorted = 0;
  for (int i = 1 + threadIdx.x; i < db; i += blockDim.x)
    unsorted |= (e.def_lam[i] < e.def_lam[i - 1]) ? 1 : 0;
  unsorted = __syncthreads_or(unsorted);
  if (threadIdx.x == 0) {
    e.counts[0] = pb;
    e.counts[1] = db;
    if (e.stats) {
      atomicAdd(e.stats + 133, 1u);                       // calls
      atomicAdd(e.stats + 134, unsorted ? 1u : 0u);       // serial re-sorts
      atomicAdd(e.stats + 135, (unsigned)db);             // deflated poles
      atomicAdd(e.stats + 136, (unsigned)q);              // candidates
    }
    for (int i = 1; unsorted && i < db; ++i) {
      double v = e.def_lam[i];
      if (v >= e.def_lam[i - 1]) continue;
      int ix = e.def_idx[i];
      int k = i - 1;
      while (k >= 0 && e.def_lam[k] > v) {
        e.def_lam[k + 1] = e.def_lam[k];
        e.def_idx[k + 1] = e.def_idx[k];
        --k;
      }
      e.def_lam[k + 1] = v;
      e.def_idx[k + 1] = ix;
    }
  }
}

// ------------------------------------------------------------------ fast reciprocal
// rcp.approx (MUFU, ~23 bits) + two Newton steps: ~1 ulp, no division
// slow path.  Used where a relative error of a few ulp per term is far below
// the rounding level of the surrounding sums.
__device__ __forceinline__ double frcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  double e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  e = fma(-q, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ E2: secular roots (CTA per root)
// h(mu) = mu - d - sum_j z_j^2 / (mu - lam_j); root i lies in (lam_{i-1}, lam_i)
// (i = 0 / p: below / above all poles).  tau = mu - origin with the origin at
// the nearer pole; rational two-pole model step (LAPACK dlaed4 style) with a
// bisection safeguard.  One CTA of NT = 32 W threads per root: the sums over
// the poles are split NT ways (two independent accumulator sets per thread)
// and reduced in a fixed order, so every thread holds bit-identical sums and
// runs the (uniform) iteration logic redundantly.  The first version used
// one warp per root: ~50 serially dependent terms per lane per iteration,
// ~10 warps per SM, 48 us per call at K = 1600 (ncu); this is latency-bound
// work, so it wants short chains and many warps.
template <int W, int NV>
__device__ __forceinline__ void block_sumv(double (&v)[NV], double (*red)[W][NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  if (W == 1) return;
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) (*red)[warp][q] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double t = (*red)[0][q];
#pragma unroll
    for (int w = 1; w < W; ++w) t += (*red)[w][q];
    v[q] = t;
  }
}

// a / b for the iteration update only (the iterate's accuracy sets the
// convergence speed, not the converged root, which is decided by h)
__device__ __forceinline__ double fdivi(double a, double b) { return a * frcp(b); }

// Two-pole rational model step (LAPACK dlaed4 "middle way" style) for the
// shifted secular function at t with the left / right sums (psiL, dpsiL,
// psiR, dpsiR); da / db: shifted neighbour poles (ia / ib < 0: none);
// returns the new iterate inside (ta, tb) (bisection when the model fails).
__device__ __forceinline__ double model_step(double t, double h, double psiL, double dpsiL,
                                             double psiR, double dpsiR, double da, double db,
                                             int ia, int ib, bool near_left, double c0,
                                             double ta, double tb) {
  double tn = 0.0;
  bool ok = false;
  if (ia >= 0 && ib >= 0) {
    double w1, w2;
    if (near_left) {
      w1 = dpsiL * (t - da) * (t - da);
      w2 = (dpsiR + 1.0) * (t - db) * (t - db);
    } else {
      w1 = (dpsiL + 1.0) * (t - da) * (t - da);
      w2 = dpsiR * (t - db) * (t - db);
    }
    const double c = h + fdivi(w1, t - da) + fdivi(w2, t - db);
    const double A = c, B = c * (da + db) + w1 + w2, C = c * da * db + w1 * db + w2 * da;
    if (A != 0.0) {
      const double sq = sqrt(fmax(B * B - 4.0 * A * C, 0.0));
      double r1, r2;
      if (B >= 0.0) { r1 = fdivi(B + sq, 2.0 * A); r2 = (B + sq) != 0.0 ? fdivi(2.0 * C, B + sq) : r1; }
      else { r1 = (B - sq) != 0.0 ? fdivi(2.0 * C, B - sq) : 0.0; r2 = fdivi(B - sq, 2.0 * A); }
      if (r1 > ta && r1 < tb) { tn = r1; ok = true; }
      else if (r2 > ta && r2 < tb) { tn = r2; ok = true; }
    } else if (B != 0.0) {
      tn = fdivi(C, B);
      ok = (tn > ta && tn < tb);
    }
  } else {
    const double psi = psiL + psiR, dpsi = dpsiL + dpsiR;
    const double w = dpsi * t * t;
    const double B = c0 + psi + fdivi(w, t);
    const double sq = sqrt(B * B + 4.0 * w);
    if (ib < 0) tn = (B >= 0.0) ? fdivi(2.0 * w, B + sq) : 0.5 * (sq - B);   // top root
    else tn = (B > 0.0) ? -0.5 * (B + sq) : fdivi(2.0 * w, B - sq);          // bottom root
    ok = (tn > ta && tn < tb);
  }
  if (!ok || !isfinite(tn)) tn = 0.5 * (ta + tb);
  return tn;
}

// Per root: (1) one pass over all poles at the interval midpoint mu0 gives
// the sign of h(mu0) (the origin = nearer pole, so mu - lam_j is formed
// without cancellation) and, for the poles outside a window of SEC_WIN
// poles around the root, their left/right sums and derivatives; (2) warp 0
// solves the LOCAL model -- the window's poles exactly, the far part
// linearised at mu0 -- to convergence, one lane per window pole; (3) the
// global two-pole iteration starts from that root.  On the c5 spectra the
// far part is smooth over the interval, so (3) converges in ~2-3 passes
// where the midpoint start needed 5-11 (the model's error is dominated by
// the dense neighbourhood, which the window now takes exactly).
#define SEC_WIN 32
#define SEC_LOCAL_IT 8   // local-model iterations (more buy ~0.2 global passes, cost latency)
// Per-thread register cache of the shifted poles and z^2 (MT terms per
// thread, MT * NT >= p); MT = 0: stream them from global memory.
template <int W, int MT>
__global__ void __launch_bounds__(32 * W) k_eig_secular(EigView e) {
  pdl_sync();
  constexpr int NT = 32 * W;
  __shared__ double red[2][W][4];   // double-buffered: one barrier per reduction
  __shared__ double s_t1;
  const int p = e.counts[0];
  const int i = blockIdx.x;
  if (i > p) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const double d = e.scal[0];
  if (p == 0) {
    if (tid == 0) { e.org[0] = d; e.tau[0] = 0.0; e.mu[0] = d; }
    return;
  }
  const double* __restrict__ poles = e.poles;
  const double* __restrict__ zz = e.zz;
  const double zabs = e.scal[2];
  const double lo = fmin(poles[0], d) - zabs - 1e-300;
  const double hi = fmax(poles[p - 1], d) + zabs + 1e-300;
  int rb = 0;
  // window of poles around the root (contains the neighbours i-1, i)
  int w0 = i - SEC_WIN / 2;
  w0 = max(0, min(w0, p - SEC_WIN));
  const int w1 = min(p, w0 + SEC_WIN);
  int ia, ib;
  double mu0, org;
  if (i == 0) {
    org = poles[0]; ia = -1; ib = 0;
    mu0 = org + 0.5 * (lo - org);
  } else if (i == p) {
    org = poles[p - 1]; ia = p - 1; ib = -1;
    mu0 = org + 0.5 * (hi - org);
  } else {
    mu0 = 0.5 * (poles[i - 1] + poles[i]);
    org = 0.0;   // decided below
    ia = i - 1; ib = i;
  }
  // (1) sums over ALL poles at mu0 (left: j <= ia), absolute coordinates; the
  // window's own terms are subtracted below (the far part only feeds the
  // local model, so the cancellation of total - window costs nothing but a
  // slightly worse starting point)
  double tL, tdL, tR, tdR;
  {
    double v[4] = {0.0, 0.0, 0.0, 0.0}, u[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = tid; j < p; j += 2 * NT) {
      {
        const double zj = zz[j];
        const double r = frcp(mu0 - poles[j]);
        const double term = zj * zj * r, dterm = term * r;
        if (j <= ia) { v[0] -= term; v[1] += dterm; } else { v[2] -= term; v[3] += dterm; }
      }
      const int k = j + NT;
      if (k < p) {
        const double zk = zz[k];
        const double r = frcp(mu0 - poles[k]);
        const double term = zk * zk * r, dterm = term * r;
        if (k <= ia) { u[0] -= term; u[1] += dterm; } else { u[2] -= term; u[3] += dterm; }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] += u[q];
    block_sumv<W, 4>(v, &red[rb]);
    rb ^= 1;
    tL = v[0]; tdL = v[1]; tR = v[2]; tdR = v[3];
  }
  // window pole of this lane
  const int jw = w0 + lane;
  const bool inw = jw < w1;
  const double zw = inw ? zz[jw] : 0.0;
  const double z2w = zw * zw;
  const double plw = inw ? poles[jw] : 0.0;
  if (i > 0 && i < p) {
    // sign of h(mu0): the origin is the nearer pole
    const double hm = (mu0 - d) + tL + tR;
    org = (hm > 0.0) ? poles[i - 1] : poles[i];
  }
  double fL, fdL, fR, fdR;   // far part = total - window, at mu0
  {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (inw) {
      const double r = frcp(mu0 - plw);
      const double term = z2w * r, dterm = term * r;
      if (jw <= ia) { a0 = -term; a1 = dterm; } else { a2 = -term; a3 = dterm; }
    }
    a0 = warp_sum(a0); a1 = warp_sum(a1); a2 = warp_sum(a2); a3 = warp_sum(a3);
    fL = tL - a0; fdL = fmax(tdL - a1, 0.0); fR = tR - a2; fdR = fmax(tdR - a3, 0.0);
  }
  const double da = (ia >= 0) ? poles[ia] - org : 0.0;
  const double db = (ib >= 0) ? poles[ib] - org : 0.0;
  double ta = (ia >= 0) ? da : lo - org;
  double tb = (ib >= 0) ? db : hi - org;
  const double c0 = org - d;
  const bool near_left = (ia >= 0) && (org == poles[ia]);
  const double t0 = mu0 - org;
  // (2) local model, warp 0: g(t) = t + c0 + [window terms] + far(t0) + far'(t0) (t - t0)
  if (tid < 32) {
    const double shw = plw - org;
    const bool wleft = jw <= ia;
    double t = t0, la = ta, lb = tb;
    for (int it = 0; it < SEC_LOCAL_IT; ++it) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (inw) {
        const double r = frcp(t - shw);
        const double term = z2w * r, dterm = term * r;
        if (wleft) { a0 = -term; a1 = dterm; } else { a2 = -term; a3 = dterm; }
      }
      a0 = warp_sum(a0); a1 = warp_sum(a1); a2 = warp_sum(a2); a3 = warp_sum(a3);
      const double psiL = a0 + fL + fdL * (t - t0), dpsiL = a1 + fdL;
      const double psiR = a2 + fR + fdR * (t - t0), dpsiR = a3 + fdR;
      const double g = t + c0 + psiL + psiR;
      if (g > 0.0) lb = t; else la = t;
      if (fabs(g) <= 8.0 * EPS * (fabs(t) + fabs(c0) + fabs(psiL) + fabs(psiR))) break;
      const double tn = model_step(t, g, psiL, dpsiL, psiR, dpsiR, da, db, ia, ib, near_left, c0,
                                   la, lb);
      if (fabs(tn - t) <= 2.0 * EPS * fabs(t)) { t = tn; break; }
      t = tn;
    }
    if (tid == 0) s_t1 = t;
  }
  __syncthreads();
  // (3) global iteration from the local root
  double shc[MT > 0 ? MT : 1], z2c[MT > 0 ? MT : 1];
  if (MT > 0) {
#pragma unroll
    for (int q = 0; q < MT; ++q) {
      const int j = tid + q * NT;
      const bool in = j < p;
      const double zj = in ? zz[j] : 0.0;
      shc[q] = in ? poles[j] - org : 1.0;
      z2c[q] = zj * zj;
    }
  }
  double t = s_t1;
  if (!(t > ta && t < tb)) t = 0.5 * (ta + tb);
  int used = 80, nbis = 0;
  for (int it = 0; it < 80; ++it) {
    // v = {psiL, dpsiL, psiR, dpsiR}: poles j <= ia give positive terms,
    // j > ia negative ones, so sum |term| = psiR - psiL
    double v[4] = {0.0, 0.0, 0.0, 0.0}, u[4] = {0.0, 0.0, 0.0, 0.0};
    if (MT > 0) {
#pragma unroll
      for (int q = 0; q < MT; ++q) {
        const int j = tid + q * NT;
        const double r = frcp(t - shc[q]);
        const double term = z2c[q] * r;
        const double dterm = term * r;
        double* acc = (q & 1) ? u : v;
        if (j <= ia) { acc[0] -= term; acc[1] += dterm; }
        else { acc[2] -= term; acc[3] += dterm; }   // j >= p: z2c = 0 contributes 0
      }
    } else {
      for (int j = tid; j < p; j += 2 * NT) {
        {
          const double zj = zz[j];
          const double r = frcp(t - (poles[j] - org));
          const double term = zj * zj * r;
          const double dterm = term * r;
          if (j <= ia) { v[0] -= term; v[1] += dterm; }
          else { v[2] -= term; v[3] += dterm; }
        }
        const int k = j + NT;
        if (k < p) {
          const double zk = zz[k];
          const double r = frcp(t - (poles[k] - org));
          const double term = zk * zk * r;
          const double dterm = term * r;
          if (k <= ia) { u[0] -= term; u[1] += dterm; }
          else { u[2] -= term; u[3] += dterm; }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] += u[q];
    block_sumv<W, 4>(v, &red[rb]);
    rb ^= 1;
    const double psiL = v[0], dpsiL = v[1], psiR = v[2], dpsiR = v[3];
    const double sabs = psiR - psiL;
    const double h = t + c0 + psiL + psiR;
    const double err = 8.0 * EPS * (fabs(t) + fabs(c0) + sabs);
    if (h > 0.0) tb = t; else ta = t;
    if (fabs(h) <= err) { used = it + 1; break; }
    double tn = model_step(t, h, psiL, dpsiL, psiR, dpsiR, da, db, ia, ib, near_left, c0, ta, tb);
    if (!(tn > ta && tn < tb)) { tn = 0.5 * (ta + tb); ++nbis; }
    if (fabs(tn - t) <= 4.0 * EPS * fabs(t)) { t = tn; used = it + 1; break; }
    t = tn;
  }
  if (e.stats && tid == 0) {
    atomicAdd(e.stats + min(used, 80), 1u);
    atomicAdd(e.stats + 96 + min(nbis, 31), 1u);
  }
  if (tid == 0) {
    e.org[i] = org;
    e.tau[i] = t;
    e.mu[i] = org + t;
  }
}

// ------------------------------------------------------------------ E3: Gu-Eisenstat zhat (CTA per pole)
// zhat_j^2 = |lam_j - mu_j| |lam_j - mu_{j+1}| prod_{i<j} |lam_j - mu_i|/|lam_j - lam_i|
//            prod_{i>j} |lam_j - mu_{i+1}|/|lam_j - lam_i|
// Each thread multiplies two interleaved partial products; fixed-order
// combination across lanes and warps.
template <int W>
__global__ void __launch_bounds__(32 * W) k_eig_zhat(EigView e) {
  pdl_sync();
  constexpr int NT = 32 * W;
  __shared__ double red[W];
  const int p = e.counts[0];
  const int j = blockIdx.x;
  if (j >= p) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double lj = e.poles[j];
  double p0 = 1.0, p1 = 1.0;
  for (int i = tid; i < p; i += 2 * NT) {
    if (i != j) {
      const int ir = (i < j) ? i : i + 1;
      p0 *= fabs((lj - e.org[ir]) - e.tau[ir]) * frcp(fabs(lj - e.poles[i]));
    }
    const int k = i + NT;
    if (k < p && k != j) {
      const int kr = (k < j) ? k : k + 1;
      p1 *= fabs((lj - e.org[kr]) - e.tau[kr]) * frcp(fabs(lj - e.poles[k]));
    }
  }
  double prod = p0 * p1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) prod *= __shfl_xor_sync(0xffffffffu, prod, o);
  if (W > 1) {
    if (lane == 0) red[warp] = prod;
    __syncthreads();
    prod = red[0];
#pragma unroll
    for (int w = 1; w < W; ++w) prod *= red[w];
  }
  if (tid == 0) {
    const double a = fabs((lj - e.org[j]) - e.tau[j]);
    const double b = fabs((lj - e.org[j + 1]) - e.tau[j + 1]);
    const double zh = sqrt(prod * a * b);
    e.zhat[j] = (e.zz[j] >= 0.0) ? zh : -zh;
  }
}

// ------------------------------------------------------------------ E4: eigenvectors, tracked rows, merge
// Stage 1 (k_eig_vec_partial): CTA (root tile x pole chunk) -> partial sums of
//   nrm2 = sum_j v_ij^2, F[r] = sum_j F_old[r][j] v_ij, L[r] = sum_j L_old[r+1][j] v_ij,
//   v_ij = zhat_j / (mu_i - lam_j), written to part[chunk][root][2S].
// Stage 2 (k_eig_vec_finish): fixed-order sum over chunks, normalisation,
//   merge into sorted order; deflated columns copied unchanged.
#define E4_RT 128   // roots per CTA
#define E4_CH 64    // poles per chunk (more CTAs: this stage is latency-bound)
__device__ __forceinline__ int count_le(const double* a, int n, double v) {  // # a[k] <= v
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int count_lt(const double* a, int n, double v) {  // # a[k] < v
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int S>
__global__ void __launch_bounds__(E4_RT) k_eig_vec_partial(EigView e, double* part, int nroot_cap) {
  pdl_sync();
  const int p = e.counts[0];
  const int chunk = blockIdx.y;
  const int c0 = chunk * E4_CH;
  if (c0 >= p && !(p == 0 && chunk == 0)) return;
  const int64_t km = e.kmax;
  __shared__ double sP[E4_CH], sZ[E4_CH];
  __shared__ double sF[S][E4_CH];
  __shared__ double sL[S][E4_CH];
  for (int q = threadIdx.x; q < E4_CH; q += blockDim.x) {
    const int jj = c0 + q;
    if (jj >= p) break;
    sP[q] = e.poles[jj];
    sZ[q] = e.zhat[jj];
    const int col = e.pmap[jj];
#pragma unroll
    for (int r = 0; r < S; ++r) sF[r][q] = e.F_old[r * km + col];
#pragma unroll
    for (int r = 0; r < S - 1; ++r) sL[r][q] = e.L_old[(r + 1) * km + col];
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > p) return;
  const double org = e.org[i], tau = e.tau[i];
  double nrm2 = 0.0, aF[S], aL[S];
#pragma unroll
  for (int r = 0; r < S; ++r) aF[r] = aL[r] = 0.0;
  const int cnt = min(E4_CH, p - c0);
  for (int q = 0; q < cnt; ++q) {
    const double v = sZ[q] * frcp(tau - (sP[q] - org));   // zhat_j / (mu_i - lam_j)
    nrm2 = fma(v, v, nrm2);
#pragma unroll
    for (int r = 0; r < S; ++r) aF[r] = fma(sF[r][q], v, aF[r]);
#pragma unroll
    for (int r = 0; r < S - 1; ++r) aL[r] = fma(sL[r][q], v, aL[r]);
  }
  double* out = part + ((int64_t)chunk * nroot_cap + i) * (2 * S);
  out[0] = nrm2;
#pragma unroll
  for (int r = 0; r < S; ++r) out[1 + r] = aF[r];
#pragma unroll
  for (int r = 0; r < S - 1; ++r) out[1 + S + r] = aL[r];
}

// Stage 2: thread per (root, value); the 2S values of a root sit in 2S
// consecutive lanes, so the chunk sums are coalesced and all chunk loads of
// a thread are independent (the first version had one thread per root
// walking 16 values x all chunks: 26 CTAs, 22 us of pure latency at K=1600).
template <int S>
__global__ void __launch_bounds__(128) k_eig_vec_finish(EigView e, const double* part,
                                                        int nroot_cap, int K, int root_blocks) {
  pdl_sync();
  constexpr int NV = 2 * S;
  constexpr int NVP = NV <= 2 ? 2 : NV <= 4 ? 4 : NV <= 8 ? 8 : 16;   // lanes per root (pow2)
  constexpr int RPB = 128 / NVP;
  const int p = e.counts[0];
  const int nd = e.counts[1];
  const int64_t km = e.kmax;
  if ((int)blockIdx.x >= root_blocks) {
    // deflated columns: unchanged eigenpairs
    const int k = (blockIdx.x - root_blocks) * blockDim.x + threadIdx.x;
    if (k >= nd) return;
    const int src = e.def_idx[k];
    const double lv = e.def_lam[k];
    const int pos = k + count_lt(e.mu, p + 1, lv);
    e.lam_new[pos] = lv;
#pragma unroll
    for (int r = 0; r < S; ++r) e.F_new[r * km + pos] = e.F_old[r * km + src];
#pragma unroll
    for (int r = 0; r < S - 1; ++r) e.L_new[r * km + pos] = e.L_old[(r + 1) * km + src];
    e.L_new[(S - 1) * km + pos] = 0.0;
    if (K < S) e.F_new[K * km + pos] = 0.0;
    return;
  }
  const int i = blockIdx.x * RPB + (int)threadIdx.x / NVP;
  const int q = (int)threadIdx.x % NVP;
  const bool valid = q < NV && i <= p;
  const int nch = (p + E4_CH - 1) / E4_CH;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (valid) {
    const double* src = part + (int64_t)i * NV + q;
    const int64_t cs = (int64_t)nroot_cap * NV;
    int c = 0;
    for (; c + 4 <= nch; c += 4) {
      a0 += __ldcg(src + c * cs);
      a1 += __ldcg(src + (c + 1) * cs);
      a2 += __ldcg(src + (c + 2) * cs);
      a3 += __ldcg(src + (c + 3) * cs);
    }
    for (; c < nch; ++c) a0 += __ldcg(src + c * cs);
  }
  const double acc = (a0 + a1) + (a2 + a3);
  // the group's nrm2 (q == 0); groups never straddle a warp (NVP divides 32)
  const int lane = threadIdx.x & 31;
  const double nrm = __shfl_sync(0xffffffffu, acc, lane - q);
  if (!valid) return;
  const double inv = 1.0 / sqrt(1.0 + nrm);
  const double mu = e.mu[i];
  const int pos = i + count_le(e.def_lam, nd, mu);
  if (q == 0) {
    e.lam_new[pos] = mu;
    e.L_new[(S - 1) * km + pos] = inv;
  } else if (q <= S) {
    // row K of Q is the new unit row while K < S (it is one of the first S rows)
    e.F_new[(q - 1) * km + pos] = (q - 1 == K) ? inv : acc * inv;
  } else {
    e.L_new[(q - 1 - S) * km + pos] = acc * inv;
  }
}

// ------------------------------------------------------------------ residual kernels
// u[j][c] = sum_r F[r][j] gamma[r][c] ;  w[j][c] = sum_r L[r][j] tau[c][r]
__global__ void k_uw(const double* F, const double* L, int64_t km, int k, int s,
                     const double* gamma, const double* tau, double* u, double* w) {
  pdl_sync();
  __shared__ double g[64], tt[64];
  if (threadIdx.x < 64) {
    g[threadIdx.x] = gamma[threadIdx.x];
    tt[threadIdx.x] = tau ? tau[threadIdx.x] : 0.0;
  }
  __syncthreads();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    for (int c = 0; c < s; ++c) {
      double a = 0.0, b = 0.0;
      for (int r = 0; r < s; ++r) {
        a = fma(F[r * km + j], g[r * 8 + c], a);
        b = fma(L[r * km + j], tt[c * 8 + r], b);
      }
      u[(int64_t)j * 8 + c] = a;
      w[(int64_t)j * 8 + c] = b;
    }
  }
}

// out_x = sum_y (a_x . b_y) / (lx_x + ly_y) c_y ;  res[0] = sum_x |out_x|^2,
// res[1] = min_{x,y} |lx_x + ly_y|  (reference residual.py:52-57, the guard of
// kernels.py:31-45).
//
// One kernel, DMMA (mma.sync m8n8k4 f64) for both s-deep products, the k^2
// reciprocals on the DFMA pipe in between -- the structure of attention:
//   P  = A_x B_y^T            (8 x-rows x 8 y-cols, k = s: 1 or 2 DMMAs)
//   P' = P / (lx_x + ly_y)     (elementwise, on the accumulator fragment)
//   M += P' C_y               (k = the 8 y's: 2 DMMAs, N = s columns)
// The accumulator of the first product is directly the A operand of the
// second: lane (g, t) holds P[g][2t], P[g][2t+1], and the second product
// takes its k-steps over the y parity (k-step h <-> y = 2t + h), so no lane
// exchange is needed; the B operand of k-step h is C[y0 + 2t + h][g].
// A CTA owns 32 x-rows (four 8-row fragments per warp: four independent DMMA
// chains per loaded y-tile) and one of YS interleaved y-splits; its 8 warps take the split's
// y-tiles in a fixed stride, with the next tile's operands loaded while the
// current one is multiplied.  The warps' partial M are summed through shared
// memory in warp order; with YS > 1 the splits' partial M go to global
// memory and the last split CTA of an x-tile (per-tile ticket) adds them in
// split order, so every sum has a fixed order: the result is deterministic.
// The minimum |lx + ly| is exact and cheap because ly is sorted ascending
// (eigenvalues): per x only the two neighbours of -lx in ly can be closest.
#define CC_XR 32     // x rows per CTA (CC_XR / 8 fragments per warp)
#define CC_NW 8      // warps per CTA
#define CC_TARGET_CTAS (3 * 148)   // one wave at 3 CTAs per SM (80 registers); 2 x 148 measured 13 % slower at k = 6000
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int KS>
struct YOps {   // operands of one 8-wide y-tile held by a lane
  double b[KS], c[2], l[2];
  bool v[2];
};
template <int S, int KS>
__device__ __forceinline__ void load_y(YOps<KS>& o, int y0, int g, int t, int ny,
                                       const double* __restrict__ ly,
                                       const double* __restrict__ by,
                                       const double* __restrict__ cy) {
  const int yb = y0 + g;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int col = 4 * ks + t;
    o.b[ks] = (yb < ny && col < S) ? __ldg(by + (int64_t)yb * 8 + col) : 0.0;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int y = y0 + 2 * t + h;
    o.v[h] = y < ny;
    o.c[h] = (o.v[h] && g < S) ? __ldg(cy + (int64_t)y * 8 + g) : 0.0;
    o.l[h] = o.v[h] ? __ldg(ly + y) : 0.0;
  }
}

// part layout: [0, 2*nxt): per-x-tile (|M|^2, min);  then [nxt][YS][16][8]
// partial M of the splits.  cnt: nxt per-tile tickets + 1 global ticket.
template <int S>
__global__ void __launch_bounds__(32 * CC_NW) k_cauchy_mma(int nx, const double* __restrict__ lx,
                                                           const double* __restrict__ ax, int ny,
                                                           const double* __restrict__ ly,
                                                           const double* __restrict__ by,
                                                           const double* __restrict__ cy,
                                                           double* part, unsigned* cnt,
                                                           double* res) {
  pdl_sync();
  constexpr int KS = (S + 3) / 4;   // k-steps of the first product
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int xt = blockIdx.x, nxt = gridDim.x;
  const int split = blockIdx.y, YS = gridDim.y;
  const int x0 = xt * CC_XR;
  // A fragments of the XF 8-row x tiles: A[g][t] = a[x0 + 8f + g][4 ks + t]
  constexpr int XF = CC_XR / 8;
  double fa[XF][KS], flx[XF];
  bool vx[XF];
#pragma unroll
  for (int f = 0; f < XF; ++f) {
    const int x = x0 + 8 * f + g;
    vx[f] = x < nx;
    flx[f] = vx[f] ? lx[x] : 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int col = 4 * ks + t;
      fa[f][ks] = (vx[f] && col < S) ? ax[(int64_t)x * 8 + col] : 0.0;
    }
  }
  double m[XF][2];   // M[x0 + 8f + g][2t + j]
#pragma unroll
  for (int f = 0; f < XF; ++f) m[f][0] = m[f][1] = 0.0;
  const int nyt = (ny + 7) >> 3;
  const int ystep = CC_NW * YS;
  int yt = warp + CC_NW * split;
  YOps<KS> cur;
  if (yt < nyt) load_y<S, KS>(cur, yt * 8, g, t, ny, ly, by, cy);
  for (; yt < nyt; yt += ystep) {
    YOps<KS> nxt_ops;
    const int yn = yt + ystep;
    if (yn < nyt) load_y<S, KS>(nxt_ops, yn * 8, g, t, ny, ly, by, cy);
#pragma unroll
    for (int f = 0; f < XF; ++f) {
      double p0 = 0.0, p1 = 0.0;   // P[g][2t], P[g][2t+1]
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) dmma884(p0, p1, fa[f][ks], cur.b[ks]);
      p0 = (vx[f] && cur.v[0]) ? p0 * frcp(flx[f] + cur.l[0]) : 0.0;
      p1 = (vx[f] && cur.v[1]) ? p1 * frcp(flx[f] + cur.l[1]) : 0.0;
      dmma884(m[f][0], m[f][1], p0, cur.c[0]);
      dmma884(m[f][0], m[f][1], p1, cur.c[1]);
    }
    if (yn < nyt) cur = nxt_ops;
  }
  // fixed-order sum of the warps' partial M
  __shared__ double sm[CC_NW][CC_XR][8];
  __shared__ double s_tile[CC_XR * 8];
  __shared__ double s_min[CC_XR];
  __shared__ unsigned s_last;
#pragma unroll
  for (int f = 0; f < XF; ++f) {
    sm[warp][8 * f + g][2 * t] = m[f][0];
    sm[warp][8 * f + g][2 * t + 1] = m[f][1];
  }
  if (split == 0 && warp == 1 && lane < CC_XR) {
    // exact min |lx + ly| of this row: the neighbours of -lx in sorted ly
    const int x = x0 + lane;
    double mn = 1e300;
    if (x < nx && ny > 0) {
      const double v = lx[x];
      int lo = 0, hi = ny;   // first index with ly >= -v
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ly[mid] < -v) lo = mid + 1; else hi = mid;
      }
      if (lo < ny) mn = fmin(mn, fabs(v + ly[lo]));
      if (lo > 0) mn = fmin(mn, fabs(v + ly[lo - 1]));
    }
    s_min[lane] = mn;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < CC_XR * 8; e += blockDim.x) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < CC_NW; ++w) v += sm[w][e >> 3][e & 7];
    s_tile[e] = v;
  }
  double* tile_out = part + 2 * (int64_t)xt;
  if (YS > 1) {
    double* mine = part + 2 * (int64_t)nxt + ((int64_t)xt * YS + split) * (CC_XR * 8);
    __syncthreads();
    for (int e = threadIdx.x; e < CC_XR * 8; e += blockDim.x) mine[e] = s_tile[e];
    if (split == 0 && threadIdx.x == 0) {
      double mn = 1e300;
      for (int r = 0; r < CC_XR; ++r) mn = fmin(mn, s_min[r]);
      tile_out[1] = mn;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      s_last = (atomicAdd(cnt + xt, 1u) == (unsigned)YS - 1) ? 1u : 0u;
      if (s_last) cnt[xt] = 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const double* all = part + 2 * (int64_t)nxt + (int64_t)xt * YS * (CC_XR * 8);
    for (int e = threadIdx.x; e < CC_XR * 8; e += blockDim.x) {
      double v = 0.0;
      for (int q = 0; q < YS; ++q) v += __ldcg(all + (int64_t)q * (CC_XR * 8) + e);
      s_tile[e] = v;
    }
  } else if (threadIdx.x == 0) {
    double mn = 1e300;
    for (int r = 0; r < CC_XR; ++r) mn = fmin(mn, s_min[r]);
    tile_out[1] = mn;
  }
  __syncthreads();
  if (warp == 0) {
    double ss = 0.0;
    for (int e = lane; e < CC_XR * 8; e += 32)
      if ((e & 7) < S) ss = fma(s_tile[e], s_tile[e], ss);
    ss = warp_sum(ss);
    if (lane == 0) tile_out[0] = ss;
  }
  // last x-tile: fixed-order reduction of the tile partials
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(cnt + nxt, 1u) == (unsigned)nxt - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ double rs[32 * CC_NW], rm[32 * CC_NW];
  double tot = 0.0, mn = 1e300;
  for (int b = threadIdx.x; b < nxt; b += blockDim.x) {
    tot += __ldcg(part + 2 * b);
    mn = fmin(mn, __ldcg(part + 2 * b + 1));
  }
  rs[threadIdx.x] = tot;
  rm[threadIdx.x] = mn;
  __syncthreads();
  for (int o = blockDim.x >> 1; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      rs[threadIdx.x] += rs[threadIdx.x + o];
      rm[threadIdx.x] = fmin(rm[threadIdx.x], rm[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    res[0] = rs[0];
    res[1] = rm[0];
    cnt[nxt] = 0u;
  }
}

// ------------------------------------------------------------------ host side
static constexpr int fin_rpb(int S) {
  return 128 / (2 * S <= 2 ? 2 : 2 * S <= 4 ? 4 : 2 * S <= 8 ? 8 : 16);
}
int EigEngine::init(int s_, int kmax_, int device) {
  s = s_;
  kmax = kmax_ + 8;
  K = 0;
  cur = 0;
  dev = device;
  const size_t nk = (size_t)kmax;
  size_t doubles = 0;
  doubles += 2 * nk;              // lam
  doubles += 2 * 2 * nk * s;      // F, L ping-pong
  doubles += 6 * nk + 8;          // z, poles, zz, zhat, def_lam, mu
  doubles += 2 * (nk + 1);        // org, tau
  doubles += 2 * nk * 8;          // u, w
  doubles += 16;                  // scal
  doubles += 4096;                // partials
  doubles += 16;                  // res
  const size_t nch_max = (nk + E4_CH - 1) / E4_CH + 1;
  const size_t vpart_n = nch_max * (nk + 8) * 16;
  doubles += vpart_n;             // E4 partial sums
  // Cauchy tile sums + split partials for x up to 2 kmax
  {
    const size_t nxt = (2 * nk + CC_XR - 1) / CC_XR;
    cpart_cap = 2 * nxt + nxt * 16 * CC_XR * 8 + 64;
  }
  doubles += cpart_cap;
  KRY_CHECK(dalloc(&dbuf, doubles));
  KRY_CUDA(cudaMemset(dbuf, 0, doubles * sizeof(double)));
  double* p = dbuf;
  for (int b = 0; b < 2; ++b) { lam[b] = p; p += nk; }
  for (int b = 0; b < 2; ++b) { F[b] = p; p += nk * s; }
  for (int b = 0; b < 2; ++b) { L[b] = p; p += nk * s; }
  z = p; p += nk; poles = p; p += nk; zz = p; p += nk; zhat = p; p += nk;
  def_lam = p; p += nk; mu = p; p += nk + 8;
  org = p; p += nk + 1; tau = p; p += nk + 1;
  u = p; p += nk * 8; w = p; p += nk * 8;
  scal = p; p += 16;
  partials = p; p += 4096;
  res = p; p += 16;
  vpart = p; p += vpart_n;
  cpart = p; p += cpart_cap;
  size_t ints = 5 * nk + 8;
  KRY_CHECK(dalloc(&ibuf, ints));
  KRY_CUDA(cudaMemset(ibuf, 0, ints * sizeof(int)));
  int* q = ibuf;
  cand = q; q += nk; dflag = q; q += nk; pflag = q; q += nk; pmap = q; q += nk;
  def_idx = q; q += nk; counts = q;
  KRY_CHECK(dalloc(&ticket, 4));
  KRY_CUDA(cudaMemset(ticket, 0, sizeof(unsigned) * 4));
  cnt_cap = (2 * nk + CC_XR - 1) / CC_XR + 1;
  KRY_CHECK(dalloc(&cnt, cnt_cap));
  KRY_CUDA(cudaMemset(cnt, 0, cnt_cap * sizeof(unsigned)));
  if (const char* st = getenv("KRY_SECULAR_STATS")) {
    if (st[0] == '1') {
      KRY_CHECK(dalloc(&stats, 160));
      KRY_CUDA(cudaMemset(stats, 0, 160 * sizeof(unsigned)));
    }
  }
  return KRY_OK;
}

void EigEngine::release() {
  if (stats) {
    unsigned h[160];
    if (cudaMemcpy(h, stats, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess) {
      fprintf(stderr, "[kry] secular iterations:");
      for (int i = 0; i <= 80; ++i)
        if (h[i]) fprintf(stderr, " %d:%u", i, h[i]);
      fprintf(stderr, "\n[kry] secular bisection steps:");
      for (int i = 0; i < 32; ++i)
        if (h[96 + i]) fprintf(stderr, " %d:%u", i, h[96 + i]);
      fprintf(stderr, "\n[kry] deflate: calls %u runs %u rotated %u longest %u re-sorts %u "
              "deflated %u candidates %u\n", h[133], h[130], h[131], h[132], h[134], h[135], h[136]);
    }
    dfree(stats);
    stats = nullptr;
  }
  if (dbuf) dfree(dbuf);
  if (ibuf) dfree(ibuf);
  if (ticket) dfree(ticket);
  if (cnt) dfree(cnt);
  cnt = nullptr;
  cnt_cap = 0;
  if (cpart_ext) dfree(cpart_ext);
  dbuf = nullptr; ibuf = nullptr; ticket = nullptr; cpart_ext = nullptr;
}

EigView EigEngine::view() const {
  EigView v;
  v.s = s; v.kmax = kmax;
  v.lam_old = lam[cur]; v.lam_new = lam[1 - cur];
  v.F_old = F[cur]; v.F_new = F[1 - cur];
  v.L_old = L[cur]; v.L_new = L[1 - cur];
  v.z = z; v.poles = poles; v.zz = zz; v.zhat = zhat; v.def_lam = def_lam; v.mu = mu;
  v.org = org; v.tau = tau; v.scal = scal;
  v.cand = cand; v.dflag = dflag; v.pflag = pflag; v.pmap = pmap; v.def_idx = def_idx;
  v.counts = counts;
  v.stats = stats;
  return v;
}

int EigEngine::append_block(cudaStream_t st, const double* dsym_blk, const double* sub_prev) {
  if (K + s > kmax - 8) return fail(KRY_ERR_STATE, "eigen engine capacity exceeded");
  for (int a = 0; a < s; ++a) {
    EigView v = view();
    // programmatic dependent launch pays where the kernels are launch-bound
    // (K < 1024: c1-c3); for the large appends it gains nothing and the
    // tighter packing only takes SM time from the recurrence kernels
    PdlScope pdl_scope(K < 1024);
    const size_t dsm = (size_t)K * (sizeof(double) + 3 * sizeof(int));
    if (dsm <= 200 * 1024) {
      if (!deflate_attr) {
        KRY_CUDA(cudaFuncSetAttribute(k_eig_deflate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
        deflate_attr = true;
      }
      pdl_launch(k_eig_deflate<true>, dim3(1), dim3(1024), dsm, st, v, K, dsym_blk, sub_prev, a);
    } else {
      pdl_launch(k_eig_deflate<false>, dim3(1), dim3(1024), 0, st, v, K, dsym_blk, sub_prev, a);
    }
    // K+1 roots at most, one CTA each; threads per root grow with K
    if (K >= 1024) {
#if KRY_SECULAR_W8 == 2
      if (K <= 64 * 32) pdl_launch(k_eig_secular<2, 32>, dim3(K + 1), dim3(64), 0, st, v);
#elif KRY_SECULAR_W8
      if (K <= 256 * 8) pdl_launch(k_eig_secular<8, 8>, dim3(K + 1), dim3(256), 0, st, v);
#else
      if (K <= 128 * 16) pdl_launch(k_eig_secular<4, 16>, dim3(K + 1), dim3(128), 0, st, v);
#endif
#if KRY_SECULAR_BIG == 1
      else if (K <= 256 * 24) pdl_launch(k_eig_secular<8, 24>, dim3(K + 1), dim3(256), 0, st, v);
#elif KRY_SECULAR_BIG == 2
      else if (K <= 256 * 16) pdl_launch(k_eig_secular<8, 16>, dim3(K + 1), dim3(256), 0, st, v);
      else if (K <= 512 * 12) pdl_launch(k_eig_secular<16, 12>, dim3(K + 1), dim3(512), 0, st, v);
#endif
      else pdl_launch(k_eig_secular<4, 0>, dim3(K + 1), dim3(128), 0, st, v);
    } else if (K >= 256) {
      pdl_launch(k_eig_secular<2, 16>, dim3(K + 1), dim3(64), 0, st, v);
    } else if (K >= 64) {
      pdl_launch(k_eig_secular<1, 8>, dim3(K + 1), dim3(32), 0, st, v);
    } else {
      pdl_launch(k_eig_secular<1, 2>, dim3(K + 1), dim3(32), 0, st, v);
    }
    int nl = 2;
    if (K > 0) {
      if (K >= 1024) pdl_launch(k_eig_zhat<4>, dim3(K), dim3(128), 0, st, v);
      else if (K >= 256) pdl_launch(k_eig_zhat<2>, dim3(K), dim3(64), 0, st, v);
      else pdl_launch(k_eig_zhat<1>, dim3(K), dim3(32), 0, st, v);
      ++nl;
    }
    const int root_blocks = (K + 1 + 127) / 128;
    const int nch = std::max(1, (K + E4_CH - 1) / E4_CH);
    const int cap = kmax + 8;
    dim3 g1(root_blocks, nch);
    const int ndef_blocks = (K + 127) / 128;
#define L(S)                                                                               \
  pdl_launch(k_eig_vec_partial<S>, g1, dim3(128), 0, st, v, vpart, cap);                   \
  pdl_launch(k_eig_vec_finish<S>, dim3((K + 1 + fin_rpb(S) - 1) / fin_rpb(S) + ndef_blocks), dim3(128), 0, st, \
             v, (const double*)vpart, cap, K, (K + 1 + fin_rpb(S) - 1) / fin_rpb(S))
    switch (s) {
      case 1: L(1); break; case 2: L(2); break; case 3: L(3); break; case 4: L(4); break;
      case 5: L(5); break; case 6: L(6); break; case 7: L(7); break; case 8: L(8); break;
      default: return fail(KRY_ERR_ARGUMENT, "block width s must be 1..8");
    }
#undef L
    count_launch(nl + 2);
    KRY_CUDA(cudaGetLastError());
    cur = 1 - cur;
    K += 1;
  }
  return KRY_OK;
}

static int cauchy_splits(int nx, int ny) {
  const int nxt = std::max(1, (nx + CC_XR - 1) / CC_XR);
  const int nyt = std::max(1, (ny + 7) / 8);
  int ys = (CC_TARGET_CTAS + nxt - 1) / nxt;
  ys = std::min(ys, std::max(1, nyt / (2 * CC_NW)));   // >= 2 y-tiles per warp
  return std::max(1, std::min(ys, 16));
}

int EigEngine::ensure_cauchy(int nx, int ny) {
  const size_t nxt = (size_t)std::max(1, (nx + CC_XR - 1) / CC_XR);
  const size_t need = 2 * nxt + nxt * 16 * CC_XR * 8 + 64;   // tile sums + split partials (YS <= 16)
  (void)ny;
  if (need <= cpart_cap && nxt + 1 <= cnt_cap) return KRY_OK;
  if (cpart_ext) dfree(cpart_ext);
  cpart_ext = nullptr;
  KRY_CHECK(dalloc(&cpart_ext, need));
  cpart = cpart_ext;
  cpart_cap = need;
  if (cnt_cap < nxt + 1) {
    if (cnt) dfree(cnt);
    cnt = nullptr;
    KRY_CHECK(dalloc(&cnt, nxt + 1));
    KRY_CUDA(cudaMemset(cnt, 0, (nxt + 1) * sizeof(unsigned)));
    cnt_cap = nxt + 1;
  }
  return KRY_OK;
}

int EigEngine::cauchy(cudaStream_t st, int nx, const double* lx, const double* ax, int ny,
                      const double* ly, const double* by, const double* cy, double* out2) {
  KRY_CHECK(ensure_cauchy(nx, ny));
  const int gx = std::max(1, (nx + CC_XR - 1) / CC_XR);
  dim3 grid(gx, cauchy_splits(nx, ny));
#define L(S) \
  pdl_launch(k_cauchy_mma<S>, grid, dim3(32 * CC_NW), 0, st, nx, lx, ax, ny, ly, by, cy, cpart, cnt, out2)
  switch (s) {
    case 1: L(1); break; case 2: L(2); break; case 3: L(3); break; case 4: L(4); break;
    case 5: L(5); break; case 6: L(6); break; case 7: L(7); break; case 8: L(8); break;
    default: return fail(KRY_ERR_ARGUMENT, "block width s must be 1..8");
  }
#undef L
  count_launch(1);
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

int EigEngine::compute_uw(cudaStream_t st, const double* gamma, const double* tau_blk) {
  int grid = (K + 255) / 256;
  if (grid < 1) grid = 1;
  pdl_launch(k_uw, dim3(grid), dim3(256), 0, st, (const double*)F[cur], (const double*)L[cur], (int64_t)kmax, K, s, gamma, tau_blk, u, w);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

// Lyapunov check: res = sqrt(2 sum_j |M_j|^2) ; writes res[0..1] on device
int EigEngine::residual_lyap(cudaStream_t st, const double* gamma, const double* tau_blk) {
  KRY_CHECK(compute_uw(st, gamma, tau_blk));
  return cauchy(st, K, lam[cur], u, K, lam[cur], u, w, res);
}


// ================================================================== full eigendecomposition
// np.linalg.eigh(t_dense) of the finalisation (solvers.py:256, :350-351) for
// the block-tridiagonal T_m, by DIVIDE AND CONQUER on the band itself (no
// tridiagonalisation): a node of the tree covers a range of block rows; it
// removes its middle block row (the separator), which decouples the two
// halves, solves them recursively and then puts the s separator rows back
// ONE SCALAR ROW AT A TIME -- exactly the bordered (arrowhead) update of the
// incremental engine above (E1 deflation, E2 secular roots, E3 Gu-Eisenstat
// zhat: the same kernels), but carrying ALL rows of the eigenvector matrix:
//   X_new = W^T X_old   (X = Q^T, row = eigenvector; W = normalised
//                        zhat_j / (mu_i - lam_j), one DMMA GEMM per row)
// Leaves (<= 32 rows) are diagonalised by a two-sided Jacobi iteration in
// shared memory.  Rows of a node are ordered [left half, right half,
// separator], so the two halves of a parent are the diagonal blocks of its
// X; `pos` maps a row of T to its final position.
namespace {

struct DcAppendArgs {
  int off, K, K0, a, s, bm, nl, nr;
  int posl[KRY_SMAX], posr[KRY_SMAX];   // local positions of the coupled rows
};

// E1 of a separator row: z = X_old[:, coupled rows] t, deflation as in
// k_eig_deflate, but the Givens rotations of numerically equal poles are
// recorded (giv_i, giv_c) for k_dc_givens instead of being applied to F / L.
template <bool SM>
__global__ void __launch_bounds__(1024) k_dc_deflate(EigView e, DcAppendArgs g,
                                                     const double* __restrict__ dsym,
                                                     const double* __restrict__ sub,
                                                     double* lam, const double* __restrict__ X,
                                                     int64_t ldx, int* giv_i, double* giv_c) {
  pdl_sync();
  extern __shared__ double dyn_sm[];
  const int K = g.K, s = g.s;
  if (SM) {   // per-pole work arrays in shared memory while they fit
    e.z = dyn_sm;
    e.cand = reinterpret_cast<int*>(dyn_sm + K);
    e.dflag = e.cand + K;
    e.pflag = e.dflag + K;
  }
  __shared__ double t[3 * KRY_SMAX];
  __shared__ int tp[3 * KRY_SMAX];
  __shared__ int s_nc, s_ng;
  __shared__ double s_d, s_tol;
  if (threadIdx.x == 0) {
    int nc = 0;
    const double* D = dsym + (int64_t)g.bm * 64;
    if (g.nl > 0)
      for (int c = 0; c < s; ++c) {   // T[sep a][left last block row c] = sub[bm-1][a][c]
        t[nc] = sub[(int64_t)(g.bm - 1) * 64 + g.a * 8 + c];
        tp[nc++] = g.posl[c];
      }
    if (g.nr > 0)
      for (int c = 0; c < s; ++c) {   // T[right first block row c][sep a] = sub[bm][c][a]
        t[nc] = sub[(int64_t)g.bm * 64 + c * 8 + g.a];
        tp[nc++] = g.posr[c];
      }
    for (int c = 0; c < g.a; ++c) {   // separator rows already appended
      t[nc] = D[g.a * 8 + c];
      tp[nc++] = g.K0 + c;
    }
    s_nc = nc;
    s_d = D[g.a * 8 + g.a];
    s_ng = 0;
  }
  __syncthreads();
  const double d = s_d;
  const int nc = s_nc;
  lam += g.off;
  const int C = (K + blockDim.x - 1) / blockDim.x;
  const int j0 = min(K, (int)threadIdx.x * C), j1 = min(K, j0 + C);
  double zmax = 0.0, zabs = 0.0;
  for (int j = j0; j < j1; ++j) {
    const double* xr = X + (int64_t)(g.off + j) * ldx + g.off;
    double z = 0.0;
    for (int r = 0; r < nc; ++r) z = fma(xr[tp[r]], t[r], z);
    e.z[j] = z;
    zmax = fmax(zmax, fabs(z));
    zabs += fabs(z);
  }
  zmax = block_max(zmax);
  zabs = block_sum(zabs);
  if (threadIdx.x == 0) {
    double lm = 0.0;
    if (K > 0) lm = fmax(fabs(lam[0]), fabs(lam[K - 1]));
    s_tol = 8.0 * EPS * fmax(fmax(lm, fabs(d)), zmax);
    e.scal[0] = d;
    e.scal[1] = s_tol;
    e.scal[2] = zabs;
  }
  __syncthreads();
  const double tol = s_tol;
  int q;
  {
    int cnt = 0;
    for (int j = j0; j < j1; ++j) cnt += (fabs(e.z[j]) > tol) ? 1 : 0;
    int pos = block_excl_scan(cnt, &q);
    for (int j = j0; j < j1; ++j) {
      const int keep = fabs(e.z[j]) > tol;
      if (keep) e.cand[pos++] = j;
      e.dflag[j] = keep ? 0 : 1;
    }
  }
  __syncthreads();
  for (int i = 1 + threadIdx.x; i < q; i += blockDim.x) {
    const int ja = e.cand[i - 1], jb = e.cand[i];
    const double za = e.z[ja], zb = e.z[jb];
    const double r = hypot(za, zb);
    const double cth = zb / r, sth = za / r;
    const double tt = lam[jb] - lam[ja];
    e.pflag[i] = (fabs(tt * cth * sth) <= tol) ? 1 : 0;
  }
  if (threadIdx.x == 0 && q > 0) e.pflag[0] = 0;
  __syncthreads();
  // runs of flagged pairs: one thread per run, rotations recorded in run order
  for (int i = 1 + threadIdx.x; i < q; i += blockDim.x) {
    if (!e.pflag[i] || e.pflag[i - 1]) continue;
    int len = 0;
    for (int k = i; k < q && e.pflag[k]; ++k) ++len;
    int slot = atomicAdd(&s_ng, len);
    int prev = e.cand[i - 1];
    for (int k = i; k < q && e.pflag[k]; ++k) {
      const int cur = e.cand[k];
      const double za = e.z[prev], zb = e.z[cur];
      const double r = hypot(za, zb);
      const double cth = zb / r, sth = za / r;
      const double tt = lam[cur] - lam[prev];
      int gp = -1, gc = -1;
      double oc = 1.0, os = 0.0;
      if (fabs(tt * cth * sth) <= tol) {
        const double l1 = lam[prev], l2 = lam[cur];
        lam[prev] = cth * cth * l1 + sth * sth * l2;
        lam[cur] = sth * sth * l1 + cth * cth * l2;
        e.z[prev] = 0.0;
        e.z[cur] = r;
        e.dflag[prev] = 1;
        gp = prev; gc = cur; oc = cth; os = sth;
      }
      giv_i[2 * slot] = gp;
      giv_i[2 * slot + 1] = gc;
      giv_c[2 * slot] = oc;
      giv_c[2 * slot + 1] = os;
      ++slot;
      prev = cur;
    }
  }
  __syncthreads();
  int pb, db;
  {
    int np = 0, nd = 0;
    for (int j = j0; j < j1; ++j) {
      if (e.dflag[j]) ++nd; else ++np;
    }
    int pp = block_excl_scan(np, &pb);
    int pd = block_excl_scan(nd, &db);
    for (int j = j0; j < j1; ++j) {
      if (e.dflag[j]) {
        e.def_idx[pd] = j;
        e.def_lam[pd] = lam[j];
        ++pd;
      } else {
        e.poles[pp] = lam[j];
        e.zz[pp] = e.z[j];
        e.pmap[pp] = j;
        ++pp;
      }
    }
  }
  __syncthreads();
  int unsorted = 0;
  for (int i = 1 + threadIdx.x; i < db; i += blockDim.x)
    unsorted |= (e.def_lam[i] < e.def_lam[i - 1]) ? 1 : 0;
  unsorted = __syncthreads_or(unsorted);
  if (threadIdx.x == 0) {
    e.counts[0] = pb;
    e.counts[1] = db;
    e.counts[2] = s_ng;
    for (int i = 1; unsorted && i < db; ++i) {
      double v = e.def_lam[i];
      if (v >= e.def_lam[i - 1]) continue;
      int ix = e.def_idx[i];
      int k = i - 1;
      while (k >= 0 && e.def_lam[k] > v) {
        e.def_lam[k + 1] = e.def_lam[k];
        e.def_idx[k + 1] = e.def_idx[k];
        --k;
      }
      e.def_lam[k + 1] = v;
      e.def_idx[k + 1] = ix;
    }
  }
}

// the recorded rotations on the rows of X (thread per column; the rotations
// of a run chain through shared rows, so they are applied in list order --
// different runs touch disjoint rows)
__global__ void k_dc_givens(const int* __restrict__ counts, const int* __restrict__ giv_i,
                            const double* __restrict__ giv_c, double* X, int64_t ldx, int off,
                            int K) {
  pdl_sync();
  const int ng = counts[2];
  if (ng == 0) return;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= K) return;
  double* xc = X + (int64_t)off * ldx + off + col;
  for (int r = 0; r < ng; ++r) {
    const int prev = giv_i[2 * r], cur = giv_i[2 * r + 1];
    if (prev < 0) continue;
    const double c = giv_c[2 * r], sn = giv_c[2 * r + 1];
    const double a = xc[(int64_t)prev * ldx], b = xc[(int64_t)cur * ldx];
    xc[(int64_t)prev * ldx] = c * a - sn * b;
    xc[(int64_t)cur * ldx] = sn * a + c * b;
  }
}

// rows of W^T (root i: zhat_j / (mu_i - lam_j), normalised), the sorted
// positions of the new eigenpairs, the new coordinate, and the deflated
// eigenpairs copied through.  grid = 2 K + 1 CTAs: [0, K] roots, then deflated.
__global__ void __launch_bounds__(128) k_dc_wbuild(EigView e, int off, int K, double* Wt,
                                                   int64_t ldw, int* crow, int* brow,
                                                   const double* __restrict__ lam_old_unused,
                                                   double* lam_new, const double* __restrict__ Xo,
                                                   double* Xn, int64_t ldx) {
  pdl_sync();
  const int p = e.counts[0], nd = e.counts[1];
  const int tid = threadIdx.x;
  __shared__ double red[4];
  if ((int)blockIdx.x <= K) {
    const int i = blockIdx.x;
    if (i > p) return;
    const double org = e.org[i], tau = e.tau[i];
    double nrm2 = 0.0;
    double* wr = Wt + (int64_t)i * ldw;
    for (int j = tid; j < p; j += 128) {
      const double v = e.zhat[j] * frcp(tau - (e.poles[j] - org));
      wr[j] = v;
      nrm2 = fma(v, v, nrm2);
    }
    nrm2 = warp_sum(nrm2);
    if ((tid & 31) == 0) red[tid >> 5] = nrm2;
    __syncthreads();
    const double inv = 1.0 / sqrt(1.0 + ((red[0] + red[1]) + (red[2] + red[3])));
    for (int j = tid; j < p; j += 128) wr[j] *= inv;
    if (i < p && tid == 32) brow[i] = off + e.pmap[i];
    if (tid == 0) {
      const double mu = e.mu[i];
      const int pos = i + count_le(e.def_lam, nd, mu);
      lam_new[off + pos] = mu;
      crow[i] = off + pos;
      Xn[(int64_t)(off + pos) * ldx + off + K] = inv;
    }
    return;
  }
  const int k = blockIdx.x - (K + 1);
  if (k >= nd) return;
  const int src = e.def_idx[k];
  const double lv = e.def_lam[k];
  const int pos = k + count_lt(e.mu, p + 1, lv);
  if (tid == 0) lam_new[off + pos] = lv;
  const double* xs = Xo + (int64_t)(off + src) * ldx + off;
  double* xd = Xn + (int64_t)(off + pos) * ldx + off;
  for (int c = tid; c < K; c += 128) xd[c] = xs[c];
  if (tid == 0) xd[K] = 0.0;
}

// leaves: two-sided cyclic Jacobi on the n <= PW rows of one leaf (CTA each;
// PW / 2 disjoint rotations per round, every thread applies J^T G J to whole
// 2 x 2 blocks, so one barrier separates the rounds)
struct DcLeaf { int b0, nb, off; };
template <int PW>
__global__ void __launch_bounds__(PW == 32 ? 256 : 1024) k_dc_leaf(const DcLeaf* __restrict__ leaves,
                                                                  int s,
                                                                  const double* __restrict__ dsym,
                                                                  const double* __restrict__ sub,
                                                                  double* lam, double* X,
                                                                  int64_t ldx) {
  constexpr int GS = PW + 1, NPAIR = PW / 2;
  extern __shared__ double leaf_sm[];
  double* sG = leaf_sm;
  double* sR = sG + PW * GS;
  double* s_c = sR + PW * GS;
  double* s_s = s_c + NPAIR;
  double* s_ev = s_s + NPAIR;
  int* s_rank = reinterpret_cast<int*>(s_ev + PW);
  const DcLeaf lf = leaves[blockIdx.x];
  const int n = lf.nb * s, tid = threadIdx.x, NT = blockDim.x;
  for (int e = tid; e < PW * GS; e += NT) { sG[e] = 0.0; sR[e] = 0.0; }
  __syncthreads();
  for (int e = tid; e < n * n; e += NT) {
    const int r = e / n, c = e % n;
    const int br = r / s, bc = c / s, ir = r % s, ic = c % s;
    double v = 0.0;
    if (br == bc) v = dsym[(int64_t)(lf.b0 + br) * 64 + ir * 8 + ic];
    else if (br == bc + 1) v = sub[(int64_t)(lf.b0 + bc) * 64 + ir * 8 + ic];
    else if (bc == br + 1) v = sub[(int64_t)(lf.b0 + br) * 64 + ic * 8 + ir];
    sG[r * GS + c] = v;
  }
  if (tid < PW) sR[tid * GS + tid] = 1.0;
  __syncthreads();
  const double tol = 2.0 * EPS;
  auto pair_of = [](int rr, int j, int* p, int* q) {
    if (j == 0) { *p = PW - 1; *q = rr; }
    else { *p = (rr + j) % (PW - 1); *q = (rr - j + (PW - 1)) % (PW - 1); }
  };
  for (int sweep = 0; sweep < 40; ++sweep) {
    int need = 0;
    for (int e = tid; e < PW * PW; e += NT) {
      const int i = e / PW, j = e % PW;
      if (i < j) {
        const double o = sG[i * GS + j];
        if (o != 0.0 && o * o > tol * tol * fabs(sG[i * GS + i] * sG[j * GS + j])) need = 1;
      }
    }
    if (!__syncthreads_or(need)) break;
    for (int rr = 0; rr < PW - 1; ++rr) {
      if (tid < NPAIR) {
        int pc, qc;
        pair_of(rr, tid, &pc, &qc);
        const double gpp = sG[pc * GS + pc], gqq = sG[qc * GS + qc], gpq = sG[pc * GS + qc];
        double c = 1.0, sn = 0.0;
        if (gpq != 0.0 && gpq * gpq > tol * tol * fabs(gpp * gqq)) {
          const double d = gqq - gpp, b2 = 2.0 * gpq;
          const double tt = (d >= 0.0 ? b2 : -b2) / (fabs(d) + sqrt(fma(d, d, b2 * b2)));
          c = rsqrt(fma(tt, tt, 1.0));
          sn = tt * c;
        }
        s_c[tid] = c;
        s_s[tid] = sn;
      }
      __syncthreads();
      for (int blk = tid; blk < NPAIR * NPAIR; blk += NT) {
        const int jc = blk % NPAIR, jr = blk / NPAIR;
        const double cc = s_c[jc], sc = s_s[jc];
        const double cr = s_c[jr], sr = s_s[jr];
        if (sc != 0.0 || sr != 0.0) {
          int pc, qc, pr, qr;
          pair_of(rr, jc, &pc, &qc);
          pair_of(rr, jr, &pr, &qr);
          const double a = sG[pr * GS + pc], b = sG[pr * GS + qc];
          const double c = sG[qr * GS + pc], d = sG[qr * GS + qc];
          const double a1 = cc * a - sc * b, b1 = sc * a + cc * b;
          const double c1 = cc * c - sc * d, d1 = sc * c + cc * d;
          sG[pr * GS + pc] = cr * a1 - sr * c1;
          sG[qr * GS + pc] = sr * a1 + cr * c1;
          sG[pr * GS + qc] = cr * b1 - sr * d1;
          sG[qr * GS + qc] = sr * b1 + cr * d1;
        }
      }
      for (int e = tid; e < PW * NPAIR; e += NT) {   // R <- R J
        const int jc = e % NPAIR, r = e / NPAIR;
        const double cc = s_c[jc], sc = s_s[jc];
        if (sc != 0.0) {
          int pc, qc;
          pair_of(rr, jc, &pc, &qc);
          const double u = sR[r * GS + pc], v = sR[r * GS + qc];
          sR[r * GS + pc] = cc * u - sc * v;
          sR[r * GS + qc] = sc * u + cc * v;
        }
      }
      __syncthreads();
    }
  }
  // eigenvalues = diag(G) of the first n indices (the padding never rotates),
  // ascending; eigenvector j = column j of R
  if (tid < n) s_ev[tid] = sG[tid * GS + tid];
  __syncthreads();
  if (tid < n) {
    const double v = s_ev[tid];
    int r = 0;
    for (int j = 0; j < n; ++j) r += (s_ev[j] < v || (s_ev[j] == v && j < tid)) ? 1 : 0;
    s_rank[tid] = r;
    lam[lf.off + r] = v;
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += NT) {
    const int j = e / n, i = e % n;   // eigenvector j, row i
    X[(int64_t)(lf.off + s_rank[j]) * ldx + lf.off + i] = sR[i * GS + j];
  }
}

// sorted union of the two halves of a node: eigenvalues merged (ties: left
// first), rows of X copied into place with the other half's columns zeroed
__global__ void __launch_bounds__(128) k_dc_merge(int off, int nl, int nr, const double* lam_src,
                                                  double* lam_dst, const double* Xs, double* Xd,
                                                  int64_t ldx) {
  const int j = blockIdx.x, n = nl + nr;
  if (j >= n) return;
  const bool left = j < nl;
  const double v = lam_src[off + j];
  int pos;
  if (left) pos = j + count_lt(lam_src + off + nl, nr, v);
  else pos = (j - nl) + count_le(lam_src + off, nl, v);
  if (threadIdx.x == 0) lam_dst[off + pos] = v;
  const double* xs = Xs + (int64_t)(off + j) * ldx + off;
  double* xd = Xd + (int64_t)(off + pos) * ldx + off;
  for (int c = threadIdx.x; c < n; c += 128) {
    const bool mine = left ? (c < nl) : (c >= nl);
    xd[c] = mine ? xs[c] : 0.0;
  }
}

__global__ void k_dc_copy(int off, int n, const double* lam_src, double* lam_dst, const double* Xs,
                          double* Xd, int64_t ldx) {
  const int j = blockIdx.x;
  if (threadIdx.x == 0) lam_dst[off + j] = lam_src[off + j];
  for (int c = threadIdx.x; c < n; c += blockDim.x)
    Xd[(int64_t)(off + j) * ldx + off + c] = Xs[(int64_t)(off + j) * ldx + off + c];
}

// Q[row + j k] = X[j][pos[row]]
__global__ void k_dc_output(const double* X, int64_t ldx, const int* pos, int k, double* Q) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e % k), j = (int)(e / k);
    Q[e] = X[(int64_t)j * ldx + pos[row]];
  }
}

struct DcNode { int b0, b1, left, right, bm, off, n, nl, nr, buf; };

int dc_build(std::vector<DcNode>& nodes, std::vector<int>& pos, int b0, int b1, int off, int s,
             int leaf_blocks) {
  DcNode nd;
  nd.b0 = b0; nd.b1 = b1; nd.off = off; nd.n = (b1 - b0) * s;
  nd.left = nd.right = -1; nd.bm = -1; nd.nl = nd.nr = 0; nd.buf = 0;
  if (b1 - b0 <= leaf_blocks) {
    for (int r = 0; r < nd.n; ++r) pos[b0 * s + r] = off + r;
    nodes.push_back(nd);
    return (int)nodes.size() - 1;
  }
  const int bm = (b0 + b1) / 2;
  nd.bm = bm;
  nd.nl = (bm - b0) * s;
  nd.nr = (b1 - bm - 1) * s;
  if (nd.nl > 0) nd.left = dc_build(nodes, pos, b0, bm, off, s, leaf_blocks);
  if (nd.nr > 0) nd.right = dc_build(nodes, pos, bm + 1, b1, off + nd.nl, s, leaf_blocks);
  for (int a = 0; a < s; ++a) pos[bm * s + a] = off + nd.nl + nd.nr + a;
  nodes.push_back(nd);
  return (int)nodes.size() - 1;
}

}  // namespace

int dc_band_eigh(cudaStream_t st, const double* dsym, const double* sub, int s, int m, double* lam_out,
                 double* Q) {
  const int k = s * m;
  if (k < 1) return KRY_OK;
  // leaf width: leaves are solved in parallel (one CTA each), the
  // merges one after the other (~35 us per separator row): pick the width
  // with the smaller estimate
  int PW = 32;
  {
    double best = 1e300;
    for (int w : {32, 64, 96}) {
      const int lb = std::max(1, w / s);
      const int nleaf = (m + lb - 1) / lb;
      const double leaf_us = w == 32 ? 250.0 : (w == 64 ? 1800.0 : 5000.0);   // measured
      const double cost = leaf_us + (double)(nleaf - 1) * s * 35.0;
      if (cost < best) { best = cost; PW = w; }
    }
    if (const char* e = getenv("KRY_DC_LEAF")) {
      const int w = atoi(e);
      if (w == 32 || w == 64 || w == 96) PW = w;
    }
  }
  const int leaf_blocks = std::max(1, PW / s);
  std::vector<DcNode> nodes;
  std::vector<int> pos(k);
  const int root = dc_build(nodes, pos, 0, m, 0, s, leaf_blocks);
  const int64_t ldx = (k + 2) & ~1;
  const int64_t ldw = ldx;
  // workspace
  double *X[2] = {nullptr, nullptr}, *lam[2] = {nullptr, nullptr}, *Wt = nullptr, *dws = nullptr,
         *giv_c = nullptr;
  int *iws = nullptr, *giv_i = nullptr, *pos_d = nullptr, *node_counts = nullptr;
  double* node_scal = nullptr;
  DcLeaf* leaves_d = nullptr;
  const size_t nk = (size_t)k + 16;
  auto cleanup = [&]() {
    for (double* q : {X[0], X[1], lam[0], lam[1], Wt, dws, giv_c, node_scal})
      if (q) dfree(q);
    for (int* q : {iws, giv_i, pos_d, node_counts})
      if (q) dfree(q);
    if (leaves_d) dfree(leaves_d);
  };
  int rc;
  if ((rc = dalloc(&X[0], (size_t)k * ldx)) || (rc = dalloc(&X[1], (size_t)k * ldx)) ||
      (rc = dalloc(&lam[0], nk)) || (rc = dalloc(&lam[1], nk)) ||
      (rc = dalloc(&Wt, (size_t)(k + 1) * ldw)) || (rc = dalloc(&dws, 9 * nk + 64)) ||
      (rc = dalloc(&giv_c, 2 * nk)) || (rc = dalloc(&iws, 7 * nk + 16)) ||
      (rc = dalloc(&giv_i, 2 * nk)) || (rc = dalloc(&pos_d, nk)) ||
      (rc = dalloc(&node_counts, 16 * nodes.size() + 16)) ||
      (rc = dalloc(&node_scal, 16 * nodes.size() + 16))) {
    cleanup();
    return rc;
  }
  cudaMemsetAsync(Wt, 0, (size_t)(k + 1) * ldw * sizeof(double), st);
  cudaMemsetAsync(X[0], 0, (size_t)k * ldx * sizeof(double), st);
  cudaMemsetAsync(X[1], 0, (size_t)k * ldx * sizeof(double), st);
  EigView v;
  memset(&v, 0, sizeof(v));
  v.s = s;
  v.kmax = k;
  {
    double* p = dws;
    v.poles = p; p += nk; v.zz = p; p += nk; v.zhat = p; p += nk; v.def_lam = p; p += nk;
    v.mu = p; p += nk; v.org = p; p += nk; v.tau = p; p += nk; v.scal = p; p += 16;
    int* q = iws;
    v.pmap = q; q += nk; v.def_idx = q; q += nk; v.counts = q; q += 16;
  }
  int* crow = iws + 2 * nk + 16;
  int* brow = crow + nk;
  // global work arrays of the deflation for orders beyond the shared-memory limit
  v.z = dws + 8 * nk + 32;
  v.cand = brow + nk;
  v.dflag = v.cand + nk;
  v.pflag = v.dflag + nk;
  cudaMemcpyAsync(pos_d, pos.data(), (size_t)k * sizeof(int), cudaMemcpyHostToDevice, st);
  // leaves
  std::vector<DcLeaf> leaves;
  for (const DcNode& nd : nodes)
    if (nd.bm < 0) leaves.push_back(DcLeaf{nd.b0, nd.b1 - nd.b0, nd.off});
  if ((rc = dalloc(&leaves_d, leaves.size()))) { cleanup(); return rc; }
  cudaMemcpyAsync(leaves_d, leaves.data(), leaves.size() * sizeof(DcLeaf), cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);   // host vectors are read by the copies above
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    cudaFuncSetAttribute(k_dc_deflate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_dc_leaf<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_dc_leaf<96>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr[dev & 63] = true;
  }
  {
    const size_t lsm = (size_t)(2 * PW * (PW + 1) + 2 * (PW / 2) + PW) * sizeof(double) + PW * sizeof(int) + 16;
    const unsigned nl = (unsigned)leaves.size();
    if (PW == 32) k_dc_leaf<32><<<nl, 256, lsm, st>>>(leaves_d, s, dsym, sub, lam[0], X[0], ldx);
    else if (PW == 64) k_dc_leaf<64><<<nl, 1024, lsm, st>>>(leaves_d, s, dsym, sub, lam[0], X[0], ldx);
    else k_dc_leaf<96><<<nl, 1024, lsm, st>>>(leaves_d, s, dsym, sub, lam[0], X[0], ldx);
    count_launch();
  }
  // Internal nodes in post-order (dc_build pushes children first).  Sibling
  // subtrees are independent and, below the root, latency-bound (few CTAs per
  // kernel): nodes are spread over NS streams, a parent waits for the events
  // of its two children.  Every per-node work array is the shared array
  // offset by the node's position range [off, off + n) (disjoint between
  // nodes that can run at the same time: neither is an ancestor of the other).
  constexpr int NS = 4;
  static cudaStream_t xs[64][NS] = {{nullptr}};
  cudaStream_t streams[NS];
  streams[0] = st;
  {
    static std::mutex xs_mu;
    std::lock_guard<std::mutex> lock(xs_mu);
    for (int q = 1; q < NS; ++q) {
      if (!xs[dev & 63][q]) cudaStreamCreateWithFlags(&xs[dev & 63][q], cudaStreamNonBlocking);
      streams[q] = xs[dev & 63][q];
    }
  }
  const bool multi = getenv("KRY_DC_SERIAL") == nullptr;
  std::vector<cudaEvent_t> ev(nodes.size(), nullptr);
  std::vector<int> nstream(nodes.size(), 0);
  cudaEvent_t ev_leaves = nullptr;
  cudaEventCreateWithFlags(&ev_leaves, cudaEventDisableTiming);
  cudaEventRecord(ev_leaves, st);
  auto destroy_events = [&]() {
    for (cudaStream_t q : streams) cudaStreamSynchronize(q);
    for (cudaEvent_t e2 : ev)
      if (e2) cudaEventDestroy(e2);
    cudaEventDestroy(ev_leaves);
  };
  int next_stream = 0;
  for (size_t ni = 0; ni < nodes.size(); ++ni) {
    DcNode& nd = nodes[ni];
    if (nd.bm < 0) continue;
    // the root (and every node on the caller's critical path) may use any
    // stream; the last node must end on `st`
    const int sid = ((int)ni == root || !multi) ? 0 : (next_stream++ % NS);
    nstream[ni] = sid;
    cudaStream_t ns = streams[sid];
    cudaStreamWaitEvent(ns, ev_leaves, 0);
    for (int ch : {nd.left, nd.right})
      if (ch >= 0 && ev[ch]) cudaStreamWaitEvent(ns, ev[ch], 0);
    // per-node views of the work arrays
    EigView vn = v;
    const int off = nd.off;
    vn.poles += off; vn.zz += off; vn.zhat += off; vn.def_lam += off; vn.mu += off;
    vn.org += off; vn.tau += off; vn.z += off;
    vn.pmap += off; vn.def_idx += off; vn.cand += off; vn.dflag += off; vn.pflag += off;
    vn.counts = node_counts + 16 * (int64_t)ni;
    vn.scal = node_scal + 16 * (int64_t)ni;
    int* n_crow = crow + off;
    int* n_brow = brow + off;
    int* n_giv_i = giv_i + 2 * (int64_t)off;
    double* n_giv_c = giv_c + 2 * (int64_t)off;
    double* n_Wt = Wt + (int64_t)off * ldw;
    const int K0 = nd.nl + nd.nr;
    // both halves in one buffer
    int src = 0;
    if (nd.left >= 0) src = nodes[nd.left].buf;
    else if (nd.right >= 0) src = nodes[nd.right].buf;
    for (int ch : {nd.left, nd.right}) {
      if (ch < 0 || nodes[ch].buf == src) continue;
      k_dc_copy<<<nodes[ch].n, 128, 0, ns>>>(nodes[ch].off, nodes[ch].n, lam[1 - src], lam[src],
                                             X[1 - src], X[src], ldx);
      count_launch();
    }
    int cur = 1 - src;
    if (K0 > 0) {
      k_dc_merge<<<K0, 128, 0, ns>>>(nd.off, nd.nl, nd.nr, lam[src], lam[cur], X[src], X[cur], ldx);
      count_launch();
    }
    for (int a = 0; a < s; ++a) {
      const int K = K0 + a;
      DcAppendArgs g;
      g.off = nd.off; g.K = K; g.K0 = K0; g.a = a; g.s = s; g.bm = nd.bm; g.nl = nd.nl; g.nr = nd.nr;
      for (int c = 0; c < s; ++c) {
        g.posl[c] = nd.nl > 0 ? pos[(nd.bm - 1) * s + c] - nd.off : 0;
        g.posr[c] = nd.nr > 0 ? pos[(nd.bm + 1) * s + c] - nd.off : 0;
      }
      const size_t dsm = (size_t)K * (sizeof(double) + 3 * sizeof(int)) + 16;
      if (dsm <= 200 * 1024 && !getenv("KRY_DC_NOSMEM"))   // (the variable forces the large-order path: tests)
        pdl_launch(k_dc_deflate<true>, dim3(1), dim3(1024), dsm, ns, vn, g, dsym, sub, lam[cur], (const double*)X[cur], ldx, n_giv_i, n_giv_c);
      else
        pdl_launch(k_dc_deflate<false>, dim3(1), dim3(1024), 0, ns, vn, g, dsym, sub, lam[cur], (const double*)X[cur], ldx, n_giv_i, n_giv_c);
      if (K > 0) pdl_launch(k_dc_givens, dim3((K + 127) / 128), dim3(128), 0, ns, (const int*)vn.counts, (const int*)n_giv_i, (const double*)n_giv_c, X[cur], ldx, nd.off, K);
      if (K >= 1024) {
        if (K <= 128 * 16) pdl_launch(k_eig_secular<4, 16>, dim3(K + 1), dim3(128), 0, ns, vn);
        else pdl_launch(k_eig_secular<4, 0>, dim3(K + 1), dim3(128), 0, ns, vn);
      } else if (K >= 256) {
        pdl_launch(k_eig_secular<2, 16>, dim3(K + 1), dim3(64), 0, ns, vn);
      } else if (K >= 64) {
        pdl_launch(k_eig_secular<1, 8>, dim3(K + 1), dim3(32), 0, ns, vn);
      } else {
        pdl_launch(k_eig_secular<1, 2>, dim3(K + 1), dim3(32), 0, ns, vn);
      }
      if (K > 0) {
        if (K >= 1024) pdl_launch(k_eig_zhat<4>, dim3(K), dim3(128), 0, ns, vn);
        else if (K >= 256) pdl_launch(k_eig_zhat<2>, dim3(K), dim3(64), 0, ns, vn);
        else pdl_launch(k_eig_zhat<1>, dim3(K), dim3(32), 0, ns, vn);
      }
      pdl_launch(k_dc_wbuild, dim3(2 * K + 1), dim3(128), 0, ns, vn, nd.off, K, n_Wt, ldw, n_crow, n_brow,
                 (const double*)nullptr, lam[1 - cur], (const double*)X[cur], X[1 - cur], ldx);
      count_launch(5);
      if (K > 0) {
        rc = dense_gemm(ns, K + 1, K, K, n_Wt, ldw, 0, X[cur] + nd.off, ldx, n_brow,
                        X[1 - cur] + nd.off, ldx, n_crow, vn.counts);
        if (rc != KRY_OK) { destroy_events(); cleanup(); return rc; }
      }
      cur = 1 - cur;
    }
    nd.buf = cur;
    cudaEventCreateWithFlags(&ev[ni], cudaEventDisableTiming);
    cudaEventRecord(ev[ni], ns);
  }
  // (the root ran on `st`, which waited for its children)
  const int rb = nodes[root].buf;
  k_dc_output<<<(int)std::min<int64_t>(((int64_t)k * k + 255) / 256, 148 * 16), 256, 0, st>>>(
      X[rb], ldx, pos_d, k, Q);
  count_launch();
  cudaMemcpyAsync(lam_out, lam[rb], (size_t)k * sizeof(double), cudaMemcpyDeviceToDevice, st);
  cudaError_t e = cudaStreamSynchronize(st);
  destroy_events();
  cleanup();
  if (e != cudaSuccess) return fail(KRY_ERR_CUDA, std::string("dc_band_eigh: ") + cudaGetErrorString(e));
  return KRY_OK;
}

}  // namespace kry
