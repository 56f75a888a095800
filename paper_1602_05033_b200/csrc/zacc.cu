// Pass-2 factor accumulation on DMMA (sm_100a, fp64).
//
// Reference: two_pass_recover (solvers.py:130-169), `z += v_new @ qy[block]`
// for every regenerated block, and _assemble_stored (solvers.py:125-127).
//
//   Z[i][j] (+)= sum_{b < nb} sum_{c < s} V_b[i][c] * Q[b s + c][j]
//
// V_b are consecutive basis blocks of one pass-2 chunk, each stored once,
// point-major (n x s, ld s) at a fixed stride `vstride` (the ring layout of
// pass 1: no second, interleaved copy), Q = the chunk's rows of S qy
// (row-major, ld ldq >= r), Z row-major n x r.  This is a tall-skinny GEMM
// (M = n = 8e6 points at c4, N = r = 231, K = G s = 512 per chunk) that is
// bound by the fp64 tensor rate: 2 n k r flops per solve (7.6 TFLOP at c4).
//
// Tiling: a CTA computes a 64 x (32 NT) tile of Z, NT = 2..8 chosen from the
// rank so that one panel covers r (c4: r = 231 -> 64 x 256; 8 warps as 2 x 4,
// each warp 32 x 8 NT = 4 x NT m8n8 DMMA tiles, 8 NT accumulator doubles per
// lane; A is then read from HBM once and every loaded fragment feeds 4 or NT
// DMMAs) and
// walks the K dimension a few basis blocks per pipeline stage (>= 8 k values
// between barriers): each block's 64 point rows (64 s contiguous doubles)
// and its s rows of the Q panel arrive by cp.async (16-byte, zero-filled
// outside the matrix) in a 3-stage ring.  Shared-memory strides are padded so that the A fragments
// (8 rows x 4 k per warp) and the B fragments (4 k x 8 columns) are read
// without bank conflicts.  CTAs are ordered panel-fastest, so the panels of
// one 64-point tile read its A rows from L2.
#include "kry_internal.cuh"
#include "finalize.cuh"
#include <algorithm>
#include <cstdlib>

namespace kry {

namespace {
constexpr int ZBM = 64, ZST = 3, ZWARPS = 8, ZNTMAX = 8;
constexpr int ZTPC = 1;   // tiles per CTA (4 and a resident persistent grid measured slower)
// B row stride (doubles) for a panel of BN columns: conflict-free B fragments
__host__ __device__ constexpr int zbst(int bn) { return bn + 4; }

__device__ __forceinline__ void zdmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp8(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// A row stride (doubles): s values padded to the k-steps, + 4 so that the 8
// rows of a fragment land in distinct banks
template <int S>
__host__ __device__ constexpr int zast() { return (S <= 4 ? 4 : 8) + 4; }
// basis blocks per pipeline stage: >= 8 k values between barriers
__host__ __device__ constexpr int zbps(int s) { return s >= 8 ? 2 : (s >= 4 ? 4 : 8); }
}  // namespace

template <int S, int NT>
__global__ void __launch_bounds__(32 * ZWARPS) k_zacc(const double* __restrict__ vbase,
                                                      int64_t vstride, int nb,
                                                      const double* __restrict__ Q, int ldq,
                                                      int r, double* __restrict__ Z, int64_t n,
                                                      int accumulate, int npanels,
                                                      int64_t ntiles) {
  constexpr int KS = (S + 3) / 4;      // k4-steps per block
  constexpr int AST = zast<S>();
  constexpr int KP = 4 * KS;           // padded k rows of a B stage
  constexpr int BPS = zbps(S);         // basis blocks per pipeline stage
  constexpr int ZBN = 32 * NT, ZBST = zbst(32 * NT);
  constexpr int ASZ = ZBM * AST, BSZ = KP * ZBST;   // per block of a stage
  extern __shared__ __align__(16) double zsm[];
  double* sA = zsm;                                  // [ZST][BPS][ASZ]
  double* sB = zsm + ZST * BPS * ASZ;                // [ZST][BPS][BSZ]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  // zero the padding once (k columns >= s of A, k rows >= s of B)
  for (int e = tid; e < ZST * BPS * ASZ; e += blockDim.x) sA[e] = 0.0;
  for (int e = tid; e < ZST * BPS * BSZ; e += blockDim.x) sB[e] = 0.0;
  __syncthreads();
  // stage `st` <- blocks grp*BPS .. grp*BPS+BPS-1 of tile (i0, j0), zero-
  // filled past nb
  auto load_stage = [&](int64_t i0, int j0, int grp, int st) {
#pragma unroll
    for (int bb = 0; bb < BPS; ++bb) {
      const int b = grp * BPS + bb;
      const bool bok = b < nb;
      double* dA = sA + ((int64_t)st * BPS + bb) * ASZ;
      double* dB = sB + ((int64_t)st * BPS + bb) * BSZ;
      const double* vb = vbase + (int64_t)(bok ? b : 0) * vstride + i0 * S;
      if ((S & 1) == 0) {
        // 64 rows x S doubles contiguous: 16-byte pieces
        constexpr int PR = (S / 2) > 0 ? S / 2 : 1;   // pieces per row
        for (int q = tid; q < ZBM * PR; q += blockDim.x) {
          const int row = q / PR, pc = q % PR;
          const bool ok = bok && i0 + row < n;
          cp16(&dA[row * AST + 2 * pc], ok ? vb + (int64_t)row * S + 2 * pc : vbase, ok);
        }
      } else {
        for (int q = tid; q < ZBM * S; q += blockDim.x) {
          const int row = q / S, c = q % S;
          const bool ok = bok && i0 + row < n;
          cp8(&dA[row * AST + c], ok ? vb + (int64_t)row * S + c : vbase, ok);
        }
      }
      const double* qb = Q + (int64_t)(bok ? b : 0) * S * ldq + j0;
      constexpr int PB = ZBN / 2;   // 16-byte pieces per Q row
      for (int q = tid; q < S * PB; q += blockDim.x) {
        const int row = q / PB, pc = q % PB;
        cp16(&dB[row * ZBST + 2 * pc], qb + (int64_t)row * ldq + 2 * pc, bok);
      }
    }
  };
  const int ng = (nb + BPS - 1) / BPS;
  auto prologue = [&](int64_t tl) {
    const int64_t i0 = (tl / npanels) * ZBM;
    const int j0 = (int)(tl % npanels) * ZBN;
#pragma unroll
    for (int st = 0; st < ZST - 1; ++st) {
      if (st < ng) load_stage(i0, j0, st, st);
      cp_commit();
    }
  };
  // Tiles in a grid-stride loop.  The next tile's first stages are issued
  // (cp.async) BEFORE this tile's epilogue, so the Z read-modify-write -- a
  // latency-bound strided access, 25 % of the stall samples when it ran
  // alone -- overlaps the copies of the next tile.
  int64_t tile = blockIdx.x;
  if (tile < ntiles) prologue(tile);
  while (tile < ntiles) {
    const int64_t i0 = (tile / npanels) * ZBM;
    const int j0 = (int)(tile % npanels) * ZBN;
    double acc[4][NT][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // n-tiles of this warp that hold real columns (the last panel pads the
    // rank to a multiple of 32 NT: r = 231 -> 25 of its 128 columns are
    // padding; their DMMAs and B fragments are skipped, warp-uniformly)
    const int ntl = min(NT, max(0, (r - (j0 + wn * 8 * NT) + 7) / 8));
    for (int gi = 0; gi < ng; ++gi) {
      cp_wait<ZST - 2>();
      __syncthreads();
      {   // prefetch group gi + ZST - 1 into the stage freed by group gi - 1
        const int gn = gi + ZST - 1;
        if (gn < ng) load_stage(i0, j0, gn, gn % ZST);
        cp_commit();
      }
#pragma unroll
      for (int bb = 0; bb < BPS; ++bb) {
        const double* A = sA + ((int64_t)(gi % ZST) * BPS + bb) * ASZ;
        const double* B = sB + ((int64_t)(gi % ZST) * BPS + bb) * BSZ;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          double fa[4], fb[NT];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) fa[mt] = A[(wm * 32 + mt * 8 + g) * AST + 4 * ks + t];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            if (nt < ntl) fb[nt] = B[(4 * ks + t) * ZBST + wn * 8 * NT + nt * 8 + g];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (nt < ntl) {
#pragma unroll
              for (int mt = 0; mt < 4; ++mt) zdmma(acc[mt][nt][0], acc[mt][nt][1], fa[mt], fb[nt]);
            }
          }
        }
      }
    }
    cp_wait<0>();
    __syncthreads();   // every warp is done with the stages
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) prologue(next);
    // epilogue: Z (+)= acc; lane (g, t) holds rows ..+g, columns ..+2t, +2t+1
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int64_t i = i0 + wm * 32 + mt * 8 + g;
      if (i >= n) continue;
      double* zr = Z + i * r;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int j = j0 + wn * 8 * NT + nt * 8 + 2 * t;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (j + e < r) {
            const double v = acc[mt][nt][e];
            zr[j + e] = accumulate ? zr[j + e] + v : v;
          }
        }
      }
    }
    tile = next;
  }
}

// Variant with the 8 warps stacked along M (warp = 8 rows x the whole panel,
// up to 16 n-tiles of 8 columns, `ntp` of them used): the panel width is
// then any multiple of 8, so the rank is padded to 8 npanels columns at most
// instead of to a multiple of 128 (r = 231: 2 panels of 15 n-tiles = 240
// columns against 256, 6 % fewer DMMAs).  One A fragment and ntp B fragments
// per k4-step feed ntp DMMAs.
constexpr int ZNTW = 16;
template <int S>
__global__ void __launch_bounds__(32 * ZWARPS) k_zacc8(const double* __restrict__ vbase,
                                                       int64_t vstride, int nb,
                                                       const double* __restrict__ Q, int ldq,
                                                       int r, double* __restrict__ Z, int64_t n,
                                                       int accumulate, int npanels, int ntp,
                                                       int64_t ntiles) {
  constexpr int KS = (S + 3) / 4;
  constexpr int AST = zast<S>();
  constexpr int KP = 4 * KS;
  constexpr int BPS = zbps(S);
  constexpr int ZBST = 8 * ZNTW + 8;   // == 8 mod 32: conflict-free B fragments
  constexpr int ASZ = ZBM * AST, BSZ = KP * ZBST;
  extern __shared__ __align__(16) double zsm[];
  double* sA = zsm;
  double* sB = zsm + ZST * BPS * ASZ;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int bnp = 8 * ntp;   // panel width
  for (int e = tid; e < ZST * BPS * ASZ; e += blockDim.x) sA[e] = 0.0;
  for (int e = tid; e < ZST * BPS * BSZ; e += blockDim.x) sB[e] = 0.0;
  __syncthreads();
  auto load_stage = [&](int64_t i0, int j0, int grp, int st) {
#pragma unroll
    for (int bb = 0; bb < BPS; ++bb) {
      const int b = grp * BPS + bb;
      const bool bok = b < nb;
      double* dA = sA + ((int64_t)st * BPS + bb) * ASZ;
      double* dB = sB + ((int64_t)st * BPS + bb) * BSZ;
      const double* vb = vbase + (int64_t)(bok ? b : 0) * vstride + i0 * S;
      if ((S & 1) == 0) {
        constexpr int PR = (S / 2) > 0 ? S / 2 : 1;
        for (int q = tid; q < ZBM * PR; q += blockDim.x) {
          const int row = q / PR, pc = q % PR;
          const bool ok = bok && i0 + row < n;
          cp16(&dA[row * AST + 2 * pc], ok ? vb + (int64_t)row * S + 2 * pc : vbase, ok);
        }
      } else {
        for (int q = tid; q < ZBM * S; q += blockDim.x) {
          const int row = q / S, c = q % S;
          const bool ok = bok && i0 + row < n;
          cp8(&dA[row * AST + c], ok ? vb + (int64_t)row * S + c : vbase, ok);
        }
      }
      const double* qb = Q + (int64_t)(bok ? b : 0) * S * ldq + j0;
      const int pb = bnp / 2;   // 16-byte pieces per Q row
      for (int q = tid; q < S * pb; q += blockDim.x) {
        const int row = q / pb, pc = q % pb;
        cp16(&dB[row * ZBST + 2 * pc], qb + (int64_t)row * ldq + 2 * pc, bok);
      }
    }
  };
  const int ng = (nb + BPS - 1) / BPS;
  auto prologue = [&](int64_t tl) {
    const int64_t i0 = (tl / npanels) * ZBM;
    const int j0 = (int)(tl % npanels) * bnp;
#pragma unroll
    for (int st = 0; st < ZST - 1; ++st) {
      if (st < ng) load_stage(i0, j0, st, st);
      cp_commit();
    }
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) prologue(tile);
  while (tile < ntiles) {
    const int64_t i0 = (tile / npanels) * ZBM;
    const int j0 = (int)(tile % npanels) * bnp;
    double acc[ZNTW][2];
#pragma unroll
    for (int b = 0; b < ZNTW; ++b) acc[b][0] = acc[b][1] = 0.0;
    for (int gi = 0; gi < ng; ++gi) {
      cp_wait<ZST - 2>();
      __syncthreads();
      {
        const int gn = gi + ZST - 1;
        if (gn < ng) load_stage(i0, j0, gn, gn % ZST);
        cp_commit();
      }
#pragma unroll
      for (int bb = 0; bb < BPS; ++bb) {
        const double* A = sA + ((int64_t)(gi % ZST) * BPS + bb) * ASZ;
        const double* B = sB + ((int64_t)(gi % ZST) * BPS + bb) * BSZ;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const double fa = A[(warp * 8 + g) * AST + 4 * ks + t];
          const double* brow = B + (4 * ks + t) * ZBST + g;
#pragma unroll
          for (int nt = 0; nt < ZNTW; ++nt)
            if (nt < ntp) zdmma(acc[nt][0], acc[nt][1], fa, brow[nt * 8]);
        }
      }
    }
    cp_wait<0>();
    __syncthreads();
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) prologue(next);
    const int64_t i = i0 + warp * 8 + g;
    if (i < n) {
      double* zr = Z + i * r;
#pragma unroll
      for (int nt = 0; nt < ZNTW; ++nt) {
        if (nt >= ntp) continue;
        const int j = j0 + nt * 8 + 2 * t;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (j + e < r) {
            const double v = acc[nt][e];
            zr[j + e] = accumulate ? zr[j + e] + v : v;
          }
        }
      }
    }
    tile = next;
  }
}

// panels of the stacked-warp variant: the fewest panels of <= 16 n-tiles, then
// the narrowest width that covers the rank
static void zacc8_shape(int r, int* npanels, int* ntp) {
  const int nt = (r + 7) / 8;
  *npanels = (nt + ZNTW - 1) / ZNTW;
  *ntp = (nt + *npanels - 1) / *npanels;
}
// KRY_ZACC8: 0 (default) 2 x 4 warps (32 x 8 NT tiles per warp), 1: 8 x 1
// warps, -1: the stacked variant where it saves at least 4 % of the padded
// columns.  Measured on c4 (r = 231): the stacked variant issues 6 % fewer
// DMMAs but one B-fragment load per DMMA instead of one per two, and runs at
// 16.0 TF/s against 17.2 (pass 2 0.521 s against 0.493 s) -- off.
static int zacc_variant(int r) {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("KRY_ZACC8");
    mode = e ? atoi(e) : 0;
  }
  if (mode == 0 || mode == 1) return mode;
  int np, ntp;
  zacc8_shape(r, &np, &ntp);
  const int cols8 = np * ntp * 8;
  const int bn = 32 * (((r + 31) / 32) <= 2 ? 2 : 4);
  const int cols4 = ((r + bn - 1) / bn) * bn;
  return cols8 * 100 <= cols4 * 96 ? 1 : 0;
}

template <int S>
static int zacc8_go(cudaStream_t st, const double* vbase, int64_t vstride, int nb, const double* Q,
                    int ldq, int r, double* Z, int64_t n, int accumulate, int max_ctas) {
  constexpr int KP = 4 * ((S + 3) / 4);
  constexpr int BPS = zbps(S);
  int npanels, ntp;
  zacc8_shape(r, &npanels, &ntp);
  const int64_t ntiles = ((n + ZBM - 1) / ZBM) * npanels;
  int64_t grid = ntiles;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (grid > 0x7fffffffLL) return fail(KRY_ERR_DIMENSION, "pass-2 factor too large");
  const size_t smem = (size_t)ZST * BPS * (ZBM * zast<S>() + KP * (8 * ZNTW + 8)) * sizeof(double);
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    KRY_CUDA(cudaFuncSetAttribute(k_zacc8<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[dev & 63] = true;
  }
  k_zacc8<S><<<(unsigned)grid, 32 * ZWARPS, smem, st>>>(vbase, vstride, nb, Q, ldq, r, Z, n,
                                                         accumulate, npanels, ntp, ntiles);
  return KRY_OK;
}

// panel width 32 NT: NT = 8 (one panel for r <= 256) measured slower on c4
// (84 vs 65 ms per chunk: 1 CTA of 168 registers per SM, 12 % warps active),
// so panels stop at 128 columns (2 CTAs per SM)
static int zacc_nt(int r) {
  const int nt = (r + 31) / 32;
  if (nt <= 2) return 2;
  return 4;
}

template <int S, int NT>
static int zacc_go(cudaStream_t st, const double* vbase, int64_t vstride, int nb,
                   const double* Q, int ldq, int r, double* Z, int64_t n, int accumulate,
                   int max_ctas) {
  constexpr int KP = 4 * ((S + 3) / 4);
  constexpr int BN = 32 * NT;
  constexpr int BPS = zbps(S);
  const int npanels = (r + BN - 1) / BN;
  const int64_t ntiles = ((n + ZBM - 1) / ZBM) * npanels;
  int64_t grid = ntiles;
  // a few tiles per CTA (not one resident wave): the epilogue of one tile
  // overlaps the copies of the next, and the CTAs stay short enough for the
  // regeneration kernels on the other stream to be scheduled between them
  // (a resident persistent grid measured 22 TF/s and serialised pass 2)
  if (max_ctas == 0) max_ctas = (int)std::min<int64_t>((ntiles + ZTPC - 1) / ZTPC, 0x7fffffff);
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (grid > 0x7fffffffLL) return fail(KRY_ERR_DIMENSION, "pass-2 factor too large");
  const size_t smem = (size_t)ZST * BPS * (ZBM * zast<S>() + KP * zbst(BN)) * sizeof(double);
  static bool attr[64] = {false};   // per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    KRY_CUDA(cudaFuncSetAttribute(k_zacc<S, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr[dev & 63] = true;
  }
  k_zacc<S, NT><<<(unsigned)grid, 32 * ZWARPS, smem, st>>>(vbase, vstride, nb, Q, ldq, r, Z, n,
                                                            accumulate, npanels, ntiles);
  return KRY_OK;
}

template <int S>
static int zacc_s(cudaStream_t st, const double* vbase, int64_t vstride, int nb, const double* Q,
                  int ldq, int r, double* Z, int64_t n, int accumulate, int max_ctas) {
  if (zacc_variant(r) == 1)
    return zacc8_go<S>(st, vbase, vstride, nb, Q, ldq, r, Z, n, accumulate, max_ctas);
  switch (zacc_nt(r)) {
    case 2: return zacc_go<S, 2>(st, vbase, vstride, nb, Q, ldq, r, Z, n, accumulate, max_ctas);
    default: return zacc_go<S, 4>(st, vbase, vstride, nb, Q, ldq, r, Z, n, accumulate, max_ctas);
  }
}



int launch_zacc(cudaStream_t st, int s, const double* vbase, int64_t vstride, int nb,
                const double* Q, int ldq, int r, double* Z, int64_t n, int accumulate,
                int max_ctas) {
  if (nb < 1 || r < 1) return KRY_OK;
#define L(S) KRY_CHECK(zacc_s<S>(st, vbase, vstride, nb, Q, ldq, r, Z, n, accumulate, max_ctas))
  switch (s) {
    case 1: L(1); break; case 2: L(2); break; case 3: L(3); break; case 4: L(4); break;
    case 5: L(5); break; case 6: L(6); break; case 7: L(7); break; case 8: L(8); break;
    default: return fail(KRY_ERR_ARGUMENT, "block width s must be 1..8");
  }
#undef L
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

// Q panel of a chunk with a padded leading dimension: Q[(b s + a) ldq + c] =
// sum_q S_i[a][q] qy[(i s + q) r + c] for c < r, 0 for r <= c < ldq (i = blk0 + b)
__global__ void k_chunk_coef_ld(const double* S, const double* qy, int s, int rank, int blk0,
                                int nblk, int ldq, double* Qc) {
  const int64_t total = (int64_t)nblk * s * ldq;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % ldq);
    const int64_t ra = e / ldq;
    const int a = (int)(ra % s), b = (int)(ra / s);
    const int i = blk0 + b;
    double v = 0.0;
    if (c < rank)
      for (int q = 0; q < s; ++q)
        v = fma(S[(int64_t)i * 64 + a * 8 + q], qy[((int64_t)i * s + q) * rank + c], v);
    Qc[e] = v;
  }
}

int launch_chunk_coef_ld(cudaStream_t st, const double* S, const double* qy, int s, int rank,
                         int blk0, int nblk, int ldq, double* Qc) {
  const int64_t total = (int64_t)nblk * s * ldq;
  int64_t g = (total + 255) / 256;
  g = std::max<int64_t>(1, std::min<int64_t>(g, 148 * 8));
  k_chunk_coef_ld<<<(int)g, 256, 0, st>>>(S, qy, s, rank, blk0, nblk, ldq, Qc);
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

int zacc_ldq(int r) {
  const int bn = 32 * zacc_nt(r);
  int np, ntp;
  zacc8_shape(r, &np, &ntp);
  return std::max(((r + bn - 1) / bn) * bn, np * ntp * 8);
}

}  // namespace kry
