// TMA-staged fused block-Lanczos step (even block widths; included by
// lanczos.cu after step.cuh, whose NbOff / stencil helpers, POST_FUSED and
// ticket / flag protocol it shares).
//
// Same work decomposition as k_step (chunk t is produced by ticket t and
// consumed by ticket t + lag, static round robin over a cooperative grid),
// but every operand of a chunk comes from shared memory filled by 1-D bulk
// TMA copies (cp.async.bulk, mbarrier completion), two iterations ahead:
//   production  : V_{m-1}[c0, c0+CH), V_m[c0-1, c0+CH+1) and the +-nx, +-nx*ny
//                 shifted ranges of V_m;
//   consumption : V_m[c0, c0+CH) and the same five ranges of V_{m+1}.
// The profile of the register-gather version showed the L1 data pipe as the
// limiter (~20 LSU wavefronts per point: the L2->L1 fills of the stencil
// gathers cost as much as the loads themselves); bulk copies land in shared
// memory without using the LSU pipe, so a point costs ~9 wavefronts (its
// eight operand reads and the store), and the copies of a whole chunk stay
// in flight while the previous chunk is computed.
//
// Missing x / y neighbours read a zero row in shared memory; missing z
// neighbours read the zero halo planes that bracket every ring block (the
// copies of the shifted ranges simply include them).

#ifndef TMA_TP
#define TMA_TP 512
#endif
#define TMA_NW (TMA_TP / 32)
#define TMA_CH 128
#ifndef TMA_PF
#define TMA_PF 3   // L2 prefetch distance (iterations)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// shared-memory footprint of one half stage (production or consumption):
// 5 ranges of CH points + the centre range of CH + 2 points
__host__ __device__ constexpr int tma_half(int S) { return (6 * TMA_CH + 2) * S; }
__host__ __device__ constexpr size_t tma_smem_bytes(int S) {
  return (size_t)(4 * tma_half(S) + 8) * sizeof(double) + 8 * sizeof(uint64_t);
}

struct TmaHalf {    // offsets (doubles) of the six ranges inside a half stage
  double *a, *c, *ym, *yp, *zm, *zp;   // a = V_{m-1} (prod) or V_m (cons); c = centre +-1
};
template <int S>
__device__ __forceinline__ TmaHalf tma_half_ptrs(double* base) {
  TmaHalf h;
  h.a = base;
  h.c = base + TMA_CH * S;
  h.ym = h.c + (TMA_CH + 2) * S;
  h.yp = h.ym + TMA_CH * S;
  h.zm = h.yp + TMA_CH * S;
  h.zp = h.zm + TMA_CH * S;
  return h;
}

// issue the bulk copies of one half stage: `a` block rows [c0, c0+CH),
// `v` block rows [c0-1, c0+CH+1) and the four shifted ranges
template <int S>
__device__ __forceinline__ void tma_issue_half(const OpDev& op, const TmaHalf& h, uint64_t* bar,
                                               const double* a, const double* v, int64_t c0) {
  constexpr unsigned RB = TMA_CH * S * 8;
  const bool has_y = op.ny > 1;
  mbar_arrive_tx(bar, RB * (has_y ? 5 : 3) + (TMA_CH + 2) * S * 8);
  tma_load_1d(h.a, a + c0 * S, RB, bar);
  tma_load_1d(h.c, v + (c0 - 1) * S, (TMA_CH + 2) * S * 8, bar);
  if (has_y) {
    tma_load_1d(h.ym, v + (c0 - op.nx) * S, RB, bar);
    tma_load_1d(h.yp, v + (c0 + op.nx) * S, RB, bar);
  }
  tma_load_1d(h.zm, v + (c0 - op.nxy) * S, RB, bar);
  tma_load_1d(h.zp, v + (c0 + op.nxy) * S, RB, bar);
}

__device__ __forceinline__ void mbar_arrive_empty(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// x / y neighbour existence of global point p
__device__ __forceinline__ void xy_mask(const OpDev& op, int p, bool& x0, bool& x1, bool& y0,
                                        bool& y1) {
  const unsigned r = fdiv((unsigned)p, op.fx);
  const int x = p - (int)r * op.nx;
  const unsigned zq = fdiv(r, op.fy);
  const int y = (int)r - (int)zq * op.ny;
  x0 = x > 0;
  x1 = x < op.nx - 1;
  y0 = y > 0;
  y1 = y < op.ny - 1;
}

// production of this warp's groups of the chunk at c0 (operands in smem)
template <int S>
__device__ __forceinline__ void tma_produce(const OpDev& op, const StepCall& c, const TmaHalf& h,
                                            const double* zero, int c0,
                                            const double (&aM)[3][2]) {
  constexpr bool PAIR = step_pair(S);
  constexpr int NV = PAIR ? 2 : 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int n = (int)c.n;
  const int col = PAIR ? min(2 * t, S - 2) : min(t, S - 1);
  const int ld = (int)c.ld;
#pragma unroll
  for (int j = 0; j < TMA_CH / 8 / TMA_NW; ++j) {
    const int r0 = (warp + j * TMA_NW) * 8;
    // B column g <-> point perm(g) = [0,5,1,6,2,7,3,4]: each quarter warp of
    // the 16-byte shared loads reads two rows 64 or 320 bytes apart (no bank
    // conflict), and the accumulator columns 2t / 2t+1 are the points t and
    // 4 + (t+1)%4 (two fully coalesced 256-byte stores)
    const int r = r0 + ((g & 1) ? 4 + (((g >> 1) + 1) & 3) : (g >> 1));
    const int p = c0 + r;
    bool mx0, mx1, my0, my1;
    xy_mask(op, min(p, n - 1), mx0, mx1, my0, my1);
    const double* src[8] = {h.a + r * S, h.c + (r + 1) * S, h.zm + r * S,
                            my0 ? h.ym + r * S : zero, mx0 ? h.c + r * S : zero,
                            mx1 ? h.c + (r + 2) * S : zero, my1 ? h.yp + r * S : zero,
                            h.zp + r * S};
    double xv[8][NV];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      if constexpr (PAIR) {
        const double2 d = *reinterpret_cast<const double2*>(src[v] + col);
        xv[v][0] = d.x;
        xv[v][1] = d.y;
      } else {
        xv[v][0] = src[v][col];
      }
    }
    double w[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q)
      w[q] = stencil_val(op, min(p, n - 1), xv[1][q], xv[2][q], xv[3][q], xv[4][q], xv[5][q],
                         xv[6][q], xv[7][q]);
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      dmma(d0, d1, aM[0][q], xv[0][q]);
      dmma(e0, e1, aM[2][q], w[q]);
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) dmma(d0, d1, aM[1][q], xv[1][q]);
    d0 += e0;
    d1 += e1;
    if (g < S) {
      const int q0 = c0 + r0 + t, q1 = c0 + r0 + 4 + ((t + 1) & 3);
      if (q0 < n) {
        c.vn[(int64_t)q0 * ld + g] = d0;
        if (c.vn2) __stcs(c.vn2 + (int64_t)q0 * c.ldn2 + g, d0);
      }
      if (q1 < n) {
        c.vn[(int64_t)q1 * ld + g] = d1;
        if (c.vn2) __stcs(c.vn2 + (int64_t)q1 * c.ldn2 + g, d1);
      }
    }
  }
}

// consumption of this warp's groups of the chunk at c0 (operands in smem)
template <int S>
__device__ __forceinline__ void tma_consume(const OpDev& op, const StepCall& c, const TmaHalf& h,
                                            const double* zero, int c0,
                                            double (&acc)[STEP_NBLK][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int n = (int)c.n;
  const int col = min(g, S - 1);
#pragma unroll
  for (int j = 0; j < TMA_CH / 8 / TMA_NW; ++j) {
    const int r0 = (warp + j * TMA_NW) * 8;
    double x[2][8];
    int pp[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int r = r0 + t + 4 * k;
      const int p = c0 + r;
      pp[k] = p;
      bool mx0, mx1, my0, my1;
      xy_mask(op, min(p, n - 1), mx0, mx1, my0, my1);
      x[k][0] = h.a[r * S + col];
      x[k][1] = h.c[(r + 1) * S + col];
      x[k][2] = h.zm[r * S + col];
      x[k][3] = (my0 ? h.ym + r * S : zero)[col];
      x[k][4] = (mx0 ? h.c + r * S : zero)[col];
      x[k][5] = (mx1 ? h.c + (r + 2) * S : zero)[col];
      x[k][6] = (my1 ? h.yp + r * S : zero)[col];
      x[k][7] = h.zp[r * S + col];
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      double w = stencil_val(op, min(pp[k], n - 1), x[k][1], x[k][2], x[k][3], x[k][4], x[k][5],
                             x[k][6], x[k][7]);
      w = pp[k] < n ? w : 0.0;
      dmma(acc[0][0], acc[0][1], x[k][0], x[k][1]);   // V_m^T V_{m+1}
      dmma(acc[1][0], acc[1][1], x[k][0], w);         // V_m^T W0
      dmma(acc[2][0], acc[2][1], x[k][1], x[k][1]);   // V_{m+1}^T V_{m+1}
      dmma(acc[3][0], acc[3][1], x[k][1], w);         // V_{m+1}^T W0
      dmma(acc[4][0], acc[4][1], w, w);               // W0^T W0
    }
  }
}

// Warp-specialised: TMA_NW compute warps and two control warps (production
// copies + completion flags; dependency waits + consumption copies), two
// iterations ahead, so the compute warps never stop at a CTA barrier inside
// the loop.  Per stage:
// full_p / full_c (copies landed; armed by the control warp with the byte
// count) and empty (the 8 compute warps are done with the stage and have
// issued the stores of its production chunk).
template <int S>
__global__ void __launch_bounds__(TMA_TP + 64, 1) k_step_tma(OpDev op, StepCall c, DevState* st,
                                                             TStore T, StepScratch sc) {
  constexpr bool PAIR = step_pair(S);
  extern __shared__ __align__(128) double smem[];
  double* zero = smem + 4 * tma_half(S);
  uint64_t* bars = reinterpret_cast<uint64_t*>(zero + 8);   // full_p[2], full_c[2], empty[2]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  if (threadIdx.x < 8) zero[threadIdx.x] = 0.0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) mbar_init(bars + q, 1);
    mbar_init(bars + 4, TMA_NW);
    mbar_init(bars + 5, TMA_NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double acc[STEP_NBLK][2];
#pragma unroll
  for (int b = 0; b < STEP_NBLK; ++b) acc[b][0] = acc[b][1] = 0.0;
  __syncthreads();
  const int64_t G = gridDim.x;
  const int64_t L = (int64_t)c.lag * G;   // consumption lag in chunks
  const int64_t kend = (c.nch + L + G - 1 - blockIdx.x) / G;   // iterations of this CTA
  auto chunk_of = [&](int64_t tk) { return c.reverse ? c.nch - 1 - tk : tk; };
  if (warp >= TMA_NW) {
    // ---------------- control warps: TMA_NW issues the production copies and
    // publishes the produced chunks; TMA_NW + 1 waits for the chunks the
    // consumption copies read and issues them.  Both re-arm a stage only
    // after the compute warps released it (empty of iteration k - 2).
    const bool prod_warp = warp == TMA_NW;
    for (int64_t k = 0; k < kend; ++k) {
      const int stg = (int)(k & 1);
      if (k >= 2) {
        mbar_wait(bars + 4 + stg, (unsigned)(((k - 2) >> 1) & 1));
        const int64_t tr = blockIdx.x + (k - 2) * G;
        // the compute warps' stores of chunk tr are ordered before their
        // arrival on `empty` (release.cta) and our wait (acquire.cta); the
        // gpu-scope release below is cumulative over them
        if (prod_warp && lane == 0 && tr < c.nch) red_release_add(sc.flags + chunk_of(tr), 1u);
      }
      const int64_t tk = blockIdx.x + k * G;
      if (prod_warp) {
        // L2 prefetch PF iterations ahead of the ranges that are first
        // touched from DRAM by this CTA (V_{m-1} and V_m rows around the
        // chunk, the far z neighbour plane); by the time the bulk copies are
        // issued they hit L2
        const int64_t tp = tk + (int64_t)TMA_PF * G;
        if (lane < 4 && tp < c.nch) {
          const int64_t p0 = chunk_of(tp) * TMA_CH;
          const double* src = lane == 0 ? c.vo + p0 * S
                             : lane == 1 ? c.vc + p0 * S
                             : lane == 2 ? c.vc + (p0 + op.nxy) * S
                                         : c.vc + (p0 - op.nxy) * S;
          prefetch_l2(src, TMA_CH * S * 8);
        }
        if (lane == 0) {
          TmaHalf hp = tma_half_ptrs<S>(smem + (2 * stg) * tma_half(S));
          if (tk < c.nch)
            tma_issue_half<S>(op, hp, bars + stg, c.vo, c.vc, chunk_of(tk) * TMA_CH);
          else
            mbar_arrive_empty(bars + stg);
        }
      } else {
        const int64_t tc = tk - L;
        const bool cv = tc >= 0 && tc < c.nch;
        if (cv) step_wait(op, c, chunk_of(tc), sc.flags);
        if (lane == 0) {
          if (cv) {
            // generic-proxy writes of other CTAs (acquired above) -> async-proxy reads
            asm volatile("fence.proxy.async.global;" ::: "memory");
            TmaHalf hc = tma_half_ptrs<S>(smem + (2 * stg + 1) * tma_half(S));
            tma_issue_half<S>(op, hc, bars + 2 + stg, c.vc, c.vn, chunk_of(tc) * TMA_CH);
          } else {
            mbar_arrive_empty(bars + 2 + stg);
          }
        }
      }
      __syncwarp();
    }
    if (prod_warp) {
      for (int64_t k = kend >= 2 ? kend - 2 : 0; k < kend; ++k) {
        mbar_wait(bars + 4 + (k & 1), (unsigned)((k >> 1) & 1));
        const int64_t tr = blockIdx.x + k * G;
        if (lane == 0 && tr < c.nch) red_release_add(sc.flags + chunk_of(tr), 1u);
        __syncwarp();
      }
    }
  } else {
    // ---------------- compute warps
    double aM[3][2];
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int k = PAIR ? 2 * t + q : t;
        aM[b][q] = (k < S && g < S && (PAIR || q == 0)) ? st->M[b * 64 + k * 8 + g] : 0.0;
      }
    for (int64_t k = 0; k < kend; ++k) {
      const int stg = (int)(k & 1);
      const unsigned par = (unsigned)((k >> 1) & 1);
      const int64_t tk = blockIdx.x + k * G;
      const int64_t tc = tk - L;
      // both full barriers are waited on in every iteration (the control
      // warp arms them even when a half has no work), so the compute warps
      // never run more than one phase ahead of the control warp's waits on
      // `empty` (a barrier two phases ahead would alias the parity)
      mbar_wait(bars + stg, par);
      if (tk < c.nch) {
        TmaHalf hp = tma_half_ptrs<S>(smem + (2 * stg) * tma_half(S));
        tma_produce<S>(op, c, hp, zero, (int)(chunk_of(tk) * TMA_CH), aM);
      }
      mbar_wait(bars + 2 + stg, par);
      if (tc >= 0 && tc < c.nch) {
        TmaHalf hc = tma_half_ptrs<S>(smem + (2 * stg + 1) * tma_half(S));
        tma_consume<S>(op, c, hc, zero, (int)(chunk_of(tc) * TMA_CH), acc);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_empty(bars + 4 + stg);
    }
  }
  __syncthreads();
  // fixed-order grid reduction (by CTA index; the control warp adds zeros)
  // + the carried blocks and the next coefficient solve on the last CTA
  finish_reduction<STEP_NBLK * 8, TMA_NW + 2>(acc, smem, sc.part, sc.gcnt, POST_FUSED, st, T);
}


// ---------------------------------------------------------------- apply kernel, TMA-staged
// [V^T W0 | W0^T W0] with W0 = A V (stored for the combine), like k_apply_gl
// but with every stencil operand staged in shared memory by bulk copies (the
// centre range +-1 point and the four +-nx, +-nx*ny shifted ranges of a
// 128-point tile, two tiles ahead), so the LSU pipe only serves the operand
// reads and the stores, not the L2 fills of the gathers.  One control warp
// issues the copies; the compute warps never meet at a CTA barrier.
#ifndef APT_NW
#define APT_NW 8
#endif
__host__ __device__ constexpr int apt_stage(int S) { return (5 * TMA_CH + 2) * S; }
__host__ __device__ constexpr size_t apt_smem_bytes(int S) {
  return (size_t)(2 * apt_stage(S) + 8) * sizeof(double) + 8 * sizeof(uint64_t);
}

template <int S>
__global__ void __launch_bounds__(APT_NW * 32 + 32, 2) k_apply_tma(OpDev op, ApplyGramCall c,
                                                                   DevState* st, TStore T,
                                                                   double* partials,
                                                                   unsigned* ticket) {
  extern __shared__ __align__(128) double smem[];
  double* zero = smem + 2 * apt_stage(S);
  uint64_t* bars = reinterpret_cast<uint64_t*>(zero + 8);   // full[2], empty[2]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  if (threadIdx.x < 8) zero[threadIdx.x] = 0.0;
  if (threadIdx.x == 0) {
    mbar_init(bars + 0, 1);
    mbar_init(bars + 1, 1);
    mbar_init(bars + 2, APT_NW);
    mbar_init(bars + 3, APT_NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  __syncthreads();
  const int64_t ntiles = (c.n + TMA_CH - 1) / TMA_CH;
  const int64_t G = gridDim.x;
  const int64_t kend = (ntiles - blockIdx.x + G - 1) / G;
  const int n = (int)c.n;
  constexpr unsigned RB = TMA_CH * S * 8;
  auto tile_of = [&](int64_t k) {
    const int64_t it = blockIdx.x + k * G;
    return c.reverse ? ntiles - 1 - it : it;
  };
  // stage layout: centre (CH + 2 rows), ym, yp, zm, zp (CH rows each)
  auto ptr = [&](int stg, int r) { return smem + stg * apt_stage(S) + (r == 0 ? 0 : (TMA_CH + 2) * S + (r - 1) * TMA_CH * S); };
  if (warp == APT_NW) {
    const bool has_y = op.ny > 1;
    for (int64_t k = 0; k < kend; ++k) {
      const int stg = (int)(k & 1);
      if (k >= 2) mbar_wait(bars + 2 + stg, (unsigned)(((k - 2) >> 1) & 1));
      if (lane == 0) {
        const int64_t c0 = tile_of(k) * TMA_CH;
        if (k + 3 < kend) {   // L2 prefetch of the tile three iterations ahead
          const int64_t p0 = tile_of(k + 3) * TMA_CH;
          prefetch_l2(c.v + p0 * S, RB);
          prefetch_l2(c.v + (p0 + op.nxy) * S, RB);
        }
        mbar_arrive_tx(bars + stg, RB * (has_y ? 4 : 2) + (TMA_CH + 2) * S * 8);
        tma_load_1d(ptr(stg, 0), c.v + (c0 - 1) * S, (TMA_CH + 2) * S * 8, bars + stg);
        if (has_y) {
          tma_load_1d(ptr(stg, 1), c.v + (c0 - op.nx) * S, RB, bars + stg);
          tma_load_1d(ptr(stg, 2), c.v + (c0 + op.nx) * S, RB, bars + stg);
        }
        tma_load_1d(ptr(stg, 3), c.v + (c0 - op.nxy) * S, RB, bars + stg);
        tma_load_1d(ptr(stg, 4), c.v + (c0 + op.nxy) * S, RB, bars + stg);
      }
      __syncwarp();
    }
  } else {
    // operand reads in the production layout (lane (g, t) = point perm(g),
    // columns {2t, 2t+1}; 16-byte shared loads without bank conflicts), the
    // stencil per column pair, A V stored as 512 contiguous bytes per warp,
    // then V and W0 transposed by a DMMA with a permuted identity (exact)
    // into the Gram fragment layout (column g of points t and 4 + (t+1)%4)
    const int col = min(2 * t, S - 2);
    const double e0 = (g == 2 * t && 2 * t < S) ? 1.0 : 0.0;          // k-step h = 0
    const double e1 = (g == 2 * t + 1 && 2 * t + 1 < S) ? 1.0 : 0.0;  // k-step h = 1
    const int pg = (g & 1) ? 4 + (((g >> 1) + 1) & 3) : (g >> 1);
    for (int64_t k = 0; k < kend; ++k) {
      const int stg = (int)(k & 1);
      mbar_wait(bars + stg, (unsigned)((k >> 1) & 1));
      const int c0 = (int)(tile_of(k) * TMA_CH);
      const double* C = ptr(stg, 0);
      const double* YM = ptr(stg, 1);
      const double* YP = ptr(stg, 2);
      const double* ZM = ptr(stg, 3);
      const double* ZP = ptr(stg, 4);
#pragma unroll
      for (int j = 0; j < TMA_CH / 8 / APT_NW; ++j) {
        const int r0 = (warp + j * APT_NW) * 8;
        const int r = r0 + pg;
        const int p = c0 + r;
        bool mx0, mx1, my0, my1;
        xy_mask(op, min(p, n - 1), mx0, mx1, my0, my1);
        auto ld2 = [&](const double* row) { return *reinterpret_cast<const double2*>(row + col); };
        const double2 v = ld2(C + (r + 1) * S);
        const double2 z0 = ld2(ZM + r * S), z1 = ld2(ZP + r * S);
        const double2 y0 = ld2(my0 ? YM + r * S : zero), y1 = ld2(my1 ? YP + r * S : zero);
        const double2 x0 = ld2(mx0 ? C + r * S : zero), x1 = ld2(mx1 ? C + (r + 2) * S : zero);
        double2 w = make_double2(0.0, 0.0);
        if (p < n) {
          const int pc = min(p, n - 1);
          w.x = stencil_val(op, pc, v.x, z0.x, y0.x, x0.x, x1.x, y1.x, z1.x);
          w.y = stencil_val(op, pc, v.y, z0.y, y0.y, x0.y, x1.y, y1.y, z1.y);
          if (c.wout && 2 * t < S)
            *reinterpret_cast<double2*>(c.wout + (int64_t)p * S + 2 * t) = w;
        }
        double vt0 = 0.0, vt1 = 0.0, wt0 = 0.0, wt1 = 0.0;
        dmma(vt0, vt1, e0, v.x);
        dmma(vt0, vt1, e1, v.y);
        dmma(wt0, wt1, e0, w.x);
        dmma(wt0, wt1, e1, w.y);
        dmma(acc[0][0], acc[0][1], vt0, wt0);   // V^T W0, points t
        dmma(acc[0][0], acc[0][1], vt1, wt1);   //         points 4 + (t+1)%4
        dmma(acc[1][0], acc[1][1], wt0, wt0);   // W0^T W0
        dmma(acc[1][0], acc[1][1], wt1, wt1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_empty(bars + 2 + stg);
    }
  }
  __syncthreads();
  finish_reduction<16, APT_NW + 1>(acc, smem, partials, ticket, c.post, st, T);
}

int launch_apply_tma(cudaStream_t st, int s, const OpDev& op, const ApplyGramCall& c,
                     DevState* dst, const TStore& T, GramScratch& g) {
  ApplyGramCall cc = c;
  cc.post = POST_STEP8;
  const int threads = APT_NW * 32 + 32;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#define L(S)                                                                               \
  {                                                                                        \
    static int per_dev[64] = {0};   /* attribute + occupancy are per device */             \
    int& per = per_dev[dev & 63];                                                          \
    const size_t sm = apt_smem_bytes(S);                                                   \
    if (!per) {                                                                            \
      KRY_CUDA(cudaFuncSetAttribute(k_apply_tma<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                    (int)sm));                                             \
      int nb = 1;                                                                          \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_apply_tma<S>, threads, sm);    \
      per = std::max(1, nb);                                                               \
    }                                                                                      \
    const int64_t ntiles = (c.n + TMA_CH - 1) / TMA_CH;                                     \
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)per * sms));  \
    if (c.grid_cap > 0) grid = std::min(grid, c.grid_cap);                                 \
    k_apply_tma<S><<<grid, threads, sm, st>>>(op, cc, dst, T, g.partials, g.ticket + 1 * KRY_TICKET_STRIDE);   \
  }
  switch (s) {
    case 2: L(2); break;
    case 4: L(4); break;
    case 6: L(6); break;
    case 8: L(8); break;
    default: return fail(KRY_ERR_ARGUMENT, "apply_tma: unsupported block width");
  }
#undef L
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}
