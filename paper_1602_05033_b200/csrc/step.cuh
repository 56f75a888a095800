// Fused single-pass block-Lanczos step for stencil operators (sm_100a, fp64).
// Included by lanczos.cu (shares coef_solve / run_post with the two-kernel
// path).  One launch per step of the reference's lanczos_step
// (basis.py:223-252): the combination that produces V_{m+1} from the
// coefficients of the previous coefficient solve, and the Gram blocks of the
// next solve (MGS twice + QR on the Gram algebra, POST_FUSED).
//
// Work decomposition.  The n points are cut into `nch` chunks of `ch`
// consecutive points; CTAs take work tickets from a global counter.  Ticket t
// produces chunk t (V_{m+1} rows, published with a release flag) and then
// consumes chunk t - lag: W0 = A V_{m+1} on its rows needs V_{m+1} on the
// +-1, +-nx, +-nx*ny neighbours, all of which lie in chunks whose tickets
// are < t (lag = ceil(nx*ny / ch) + 1).  A ticket only ever waits for lower
// tickets, which were taken by CTAs that are already running, so the scheme
// is deadlock free whatever else shares the GPU (no co-residency needed).
// The consumed rows are re-read from L2 right after they were written: HBM
// sees V_{m-1} and V_m read once and V_{m+1} written once per step.
//
// Register layouts (no shared-memory staging; DMMA m8n8k4 f64 fragments come
// straight from the loads).  g = lane / 4, t = lane % 4.
//  * production of an 8-point group: lane (g, t) holds point perm(g) =
//    g/2 + 4 (g%2), columns {2t, 2t+1} (S > 4) or {t} (S <= 4).  Then
//    V_{m+1}^T = [Mo; Mc; Mw]^T [V_{m-1} V_m AV_m]^T is a DMMA with the
//    coefficient matrix as the A operand and the loaded values as the B
//    operand (k = source column); the accumulator lands as lane (g, t) =
//    column g of points t and t + 4, i.e. two 256-byte coalesced stores.
//  * consumption of an 8-point group: lane (g, t) holds column g of points
//    t and t + 4 of V_m, V_{m+1} and W0; every Gram X^T Y is a DMMA with
//    k = point, A and B both taken from the lane's own registers.
// The per-chunk Gram partials are summed in a fixed order (chunks within
// groups of 32, then groups), so the result does not depend on which CTA
// took which ticket: pass 2 regenerates pass 1 bit for bit.

#define STEP_TP 128
#define STEP_NBLK 5
#define STEP_PART (STEP_NBLK * 64)
#define STEP_GROUP 32
#ifndef KRY_STEP_MINB
#define KRY_STEP_MINB 4
#endif

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
#define LD_NEW(p) __ldcg(p)
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Element offsets of the six stencil neighbours of point i.  Missing z
// neighbours fall into the zero halo planes that bracket every ring block;
// a missing x / y neighbour is redirected to the last point of the lower
// halo plane (also zero), so the stencil needs no per-value masking and the
// arithmetic is exactly that of the masked form (x + 0 = x).  A point past
// the end (tail group) reads the first upper-halo point for itself and all
// its neighbours: every value is zero.
struct NbOff {
  int i;                         // the point actually addressed
  int z0, y0, x0, x1, y1, z1;    // neighbour offsets (elements)
};
template <bool TAIL>
__device__ __forceinline__ NbOff nb_off(const OpDev& op, int i, int n, int ld) {
  NbOff o;
  const bool out = TAIL && i >= n;
  if (TAIL) i = out ? n : i;
  const unsigned r = fdiv((unsigned)i, op.fx);
  const int x = i - (int)r * op.nx;
  const unsigned zq = fdiv(r, op.fy);
  const int y = (int)r - (int)zq * op.ny;
  const int zero = -(i + 1) * ld;
  o.i = i;
  o.z0 = -op.nxy * ld;
  o.z1 = op.nxy * ld;
  o.y0 = y > 0 ? -op.nx * ld : zero;
  o.y1 = y < op.ny - 1 ? op.nx * ld : zero;
  o.x0 = x > 0 ? -ld : zero;
  o.x1 = x < op.nx - 1 ? ld : zero;
  if (TAIL && out) o.z0 = o.z1 = o.y0 = o.y1 = o.x0 = o.x1 = 0;
  return o;
}

// One stencil value (same arithmetic as stencil_fast / stage_warp_coop:
// constant coefficients folded per axis in FMA form; variable coefficients
// accumulated -x, +x, -y, +y, -z, +z).  The coefficient arrays carry a zero
// plane on both sides, so their unmasked loads stay in bounds.
__device__ __forceinline__ double stencil_val(const OpDev& op, int i, double v, double nz0,
                                              double ny0, double nx0, double nx1, double ny1,
                                              double nz1) {
  if (!op.variable)
    return fma(op.cd, v, fma(op.cz, nz0 + nz1, fma(op.cy, ny0 + ny1, op.cx * (nx0 + nx1))));
  double t = __ldg(op.d + i) * v;
  t = fma(__ldg(op.ex + i - 1), nx0, t);
  t = fma(__ldg(op.ex + i), nx1, t);
  t = fma(__ldg(op.ey + i - op.nx), ny0, t);
  t = fma(__ldg(op.ey + i), ny1, t);
  t = fma(__ldg(op.ez + i - op.nxy), nz0, t);
  return fma(__ldg(op.ez + i), nz1, t);
}

__host__ __device__ constexpr int step_pair(int S) { return S > 4 ? 1 : 0; }

// ---------------------------------------------------------------- production
// NG 8-point groups of V_{m+1} (all loads of the NG groups are issued before
// any is used).  aM[b][h]: A fragment of block b (o, c, w), k-step h.
// c.vo == c.vc at step 1 (its coefficient block Mo is zero).
template <int S, bool TAIL, int NG>
__device__ __forceinline__ void produce_groups(const OpDev& op, const StepCall& c, int pb0,
                                               int gstride, const double (&aM)[3][2]) {
  constexpr bool PAIR = step_pair(S);
  constexpr int NV = PAIR ? 2 : 1;       // values per lane per block
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ld = (int)c.ld;
  const int n = (int)c.n;
  const int col = PAIR ? min(2 * t, S - 2) : min(t, S - 1);
  double xv[NG][8][NV];   // [group][old, cur, z0, y0, x0, x1, y1, z1][value]
  int ii[NG];
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const NbOff o = nb_off<TAIL>(op, pb0 + q * gstride + (g >> 1) + 4 * (g & 1), n, ld);
    ii[q] = o.i;
    const int e = o.i * ld + col;
    const int offs[8] = {0, 0, o.z0, o.y0, o.x0, o.x1, o.y1, o.z1};
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double* src = (v == 0 ? c.vo : c.vc) + e + offs[v];
      if constexpr (PAIR) {
        const double2 d = __ldg(reinterpret_cast<const double2*>(src));
        xv[q][v][0] = d.x;
        xv[q][v][NV - 1] = d.y;
      } else {
        xv[q][v][0] = __ldg(src);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    double w[NV];
#pragma unroll
    for (int h = 0; h < NV; ++h)
      w[h] = stencil_val(op, ii[q], xv[q][1][h], xv[q][2][h], xv[q][3][h], xv[q][4][h],
                         xv[q][5][h], xv[q][6][h], xv[q][7][h]);
    // two independent accumulation chains (old + cur, A V), summed at the end
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
    for (int h = 0; h < NV; ++h) {
      dmma(d0, d1, aM[0][h], xv[q][0][h]);
      dmma(e0, e1, aM[2][h], w[h]);
    }
#pragma unroll
    for (int h = 0; h < NV; ++h) dmma(d0, d1, aM[1][h], xv[q][1][h]);
    d0 += e0;
    d1 += e1;
    // accumulator: lane (g, t) = column g of points pb + t (d0), pb + t + 4 (d1)
    if (g < S) {
      const int pb = pb0 + q * gstride;
      const int q0 = pb + t, q1 = pb + t + 4;
      if (!TAIL || q0 < n) {
        c.vn[q0 * ld + g] = d0;
        if (c.vn2) __stcs(c.vn2 + (int64_t)q0 * c.ldn2 + g, d0);
      }
      if (!TAIL || q1 < n) {
        c.vn[q1 * ld + g] = d1;
        if (c.vn2) __stcs(c.vn2 + (int64_t)q1 * c.ldn2 + g, d1);
      }
    }
  }
}

// this warp's groups of chunk u (the warps of a CTA interleave by group)
template <int S>
__device__ __forceinline__ void step_produce(const OpDev& op, const StepCall& c, int64_t u,
                                             const double (&aM)[3][2]) {
  const int warp = threadIdx.x >> 5;
  constexpr int GS = STEP_TP / 4;          // points between a warp's groups
  const int p0 = (int)(u * c.ch);
  const int pend = min(p0 + c.ch, (int)c.n);
  int pb = p0 + warp * 8;
  for (; pb + GS + 8 <= pend; pb += 2 * GS) produce_groups<S, false, 2>(op, c, pb, GS, aM);
  for (; pb < pend; pb += GS) {
    if (pb + 8 <= (int)c.n)
      produce_groups<S, false, 1>(op, c, pb, GS, aM);
    else
      produce_groups<S, true, 1>(op, c, pb, GS, aM);
  }
}

// ---------------------------------------------------------------- consumption
// NG 8-point groups of the Gram blocks (V_{m+1} = c.vn was written by this
// launch: its loads go through L2 only).  Lanes with g >= S duplicate column
// S-1; the Gram rows / columns they produce are never read.
template <int S, bool TAIL, int NG>
__device__ __forceinline__ void consume_groups(const OpDev& op, const StepCall& c, int pb0,
                                               int gstride, double (&acc)[STEP_NBLK][2]) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ld = (int)c.ld;
  const int n = (int)c.n;
  const int col = min(g, S - 1);
  double xv[NG][2][8];    // [group][k][old, cur, z0, y0, x0, x1, y1, z1]
  int ii[NG][2];
#pragma unroll
  for (int q = 0; q < NG; ++q)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const NbOff o = nb_off<TAIL>(op, pb0 + q * gstride + t + 4 * k, n, ld);
      ii[q][k] = o.i;
      const int e = o.i * ld + col;
      const double* pc = c.vn + e;
      xv[q][k][0] = __ldg(c.vc + e);
      xv[q][k][1] = LD_NEW(pc);
      xv[q][k][2] = LD_NEW(pc + o.z0);
      xv[q][k][3] = LD_NEW(pc + o.y0);
      xv[q][k][4] = LD_NEW(pc + o.x0);
      xv[q][k][5] = LD_NEW(pc + o.x1);
      xv[q][k][6] = LD_NEW(pc + o.y1);
      xv[q][k][7] = LD_NEW(pc + o.z1);
    }
#pragma unroll
  for (int q = 0; q < NG; ++q)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double* x = xv[q][k];
      const double w = stencil_val(op, ii[q][k], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
      dmma(acc[0][0], acc[0][1], x[0], x[1]);   // V_m^T V_{m+1}
      dmma(acc[1][0], acc[1][1], x[0], w);      // V_m^T W0
      dmma(acc[2][0], acc[2][1], x[1], x[1]);   // V_{m+1}^T V_{m+1}
      dmma(acc[3][0], acc[3][1], x[1], w);      // V_{m+1}^T W0
      dmma(acc[4][0], acc[4][1], w, w);         // W0^T W0
    }
}

template <int S>
__device__ __forceinline__ void step_consume(const OpDev& op, const StepCall& c, int64_t u,
                                             double (&acc)[STEP_NBLK][2]) {
  const int warp = threadIdx.x >> 5;
  constexpr int GS = STEP_TP / 4;
  const int p0 = (int)(u * c.ch);
  const int pend = min(p0 + c.ch, (int)c.n);
  int pb = p0 + warp * 8;
  for (; pb + GS + 8 <= pend; pb += 2 * GS) consume_groups<S, false, 2>(op, c, pb, GS, acc);
  for (; pb < pend; pb += GS) {
    if (pb + 8 <= (int)c.n)
      consume_groups<S, false, 1>(op, c, pb, GS, acc);
    else
      consume_groups<S, true, 1>(op, c, pb, GS, acc);
  }
}

// ---------------------------------------------------------------- apply kernel, register fragments
// The coefficient-solve input of the two-kernel path, [V^T W0 | W0^T W0]
// with W0 = A V, computed like the fused kernel's consumption: lane (g, t)
// holds column g of points t and t + 4 of an 8-point group (8-byte loads,
// 256 contiguous bytes per instruction), the stencil uses the zero-halo
// redirection, both Grams are DMMAs straight from the registers, and W0 is
// stored for the combine kernel.  No shared-memory staging (the staged
// kernel spent ~30 % of its LSU wavefronts on the smem tile).
template <int S, bool TAIL>
__device__ __forceinline__ void apply_gl_group(const OpDev& op, const ApplyGramCall& c, int pb,
                                               double (&acc)[2][2]) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n = (int)c.n;
  const int col = min(g, S - 1);
  double v[2], w[2];
  int ip[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const NbOff o = nb_off<TAIL>(op, pb + t + 4 * k, n, S);
    ip[k] = pb + t + 4 * k;
    const double* pc = c.v + o.i * S + col;
    v[k] = __ldg(pc);
    const double n0 = __ldg(pc + o.z0), n1 = __ldg(pc + o.y0), n2 = __ldg(pc + o.x0);
    const double n3 = __ldg(pc + o.x1), n4 = __ldg(pc + o.y1), n5 = __ldg(pc + o.z1);
    w[k] = stencil_val(op, o.i, v[k], n0, n1, n2, n3, n4, n5);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (c.wout && g < S && (!TAIL || ip[k] < n)) c.wout[(int64_t)ip[k] * S + g] = w[k];
    dmma(acc[0][0], acc[0][1], v[k], w[k]);   // V^T W0
    dmma(acc[1][0], acc[1][1], w[k], w[k]);   // W0^T W0
  }
}

template <int S>
__global__ void __launch_bounds__(128, 8) k_apply_gl(OpDev op, ApplyGramCall c, DevState* st,
                                                     TStore T, double* partials,
                                                     unsigned* ticket) {
  __shared__ __align__(16) double sX[4 * 128 + 14 * 64 + 256];
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const int warp = threadIdx.x >> 5;
  const int64_t ntiles = (c.n + TP - 1) / TP;
  const int n = (int)c.n;
  const TileOrder ord(ntiles);
  for (int64_t k = 0; ord.valid(k); ++k) {
    const int64_t it = ord.at(k);
    const int64_t tile = c.reverse ? (ntiles - 1 - it) : it;
    if (threadIdx.x == 0 && ord.valid(k + 1)) {
      const int64_t nx_ = ord.at(k + 1);
      const int64_t nt = c.reverse ? (ntiles - 1 - nx_) : nx_;
      prefetch_rows(c.v, c.ldv, nt * TP, c.n);
    }
    // this warp's 32 points = four 8-point groups
    const int p0 = (int)(tile * TP) + warp * 32;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int pb = p0 + 8 * q;
      if (pb >= n) break;
      if (pb + 8 <= n)
        apply_gl_group<S, false>(op, c, pb, acc);
      else
        apply_gl_group<S, true>(op, c, pb, acc);
    }
  }
  finish_reduction<16>(acc, sX, partials, ticket, c.post, st, T);
}

// apply kernel variant for a single-GPU stencil step with even s:
// 0 = shared-memory staged (k_apply_gram), 1 = register fragments
// (k_apply_gl, KRY_APPLY_GL=1), 2 = TMA-staged (k_apply_tma).  Default: the
// TMA-staged kernel for constant-coefficient stencils (c4: whole solve
// 0.888 -> 0.853 s); variable coefficients keep the staged kernel (their
// per-point coefficient loads go through L1 either way).
// KRY_APPLY_KERNEL=staged|gl|tma overrides.
int apply_mode(const OpDev& op, int s) {
  if (op.kind != KRY_OP_STENCIL || op.halo_lo || op.halo_hi) return 0;
  if (s != 2 && s != 4 && s != 6 && s != 8) return 0;
  if (const char* k = getenv("KRY_APPLY_KERNEL")) {
    if (k[0] == 't') return 2;
    if (k[0] == 'g') return 1;
    return 0;
  }
  return op.variable ? 0 : 2;
}

int launch_apply_gl(cudaStream_t st, int s, const OpDev& op, const ApplyGramCall& c,
                    DevState* dst, const TStore& T, GramScratch& g) {
  ApplyGramCall cc = c;
  cc.post = POST_STEP8;
#define L(S)                                                                      \
  k_apply_gl<S><<<resident_grid(k_apply_gl<S>, c.n), TP, 0, st>>>(op, cc, dst, T, \
                                                                  g.partials, g.ticket + 1 * KRY_TICKET_STRIDE)
  switch (s) {
    case 2: L(2); break;
    case 4: L(4); break;
    case 6: L(6); break;
    case 8: L(8); break;
    default: return fail(KRY_ERR_ARGUMENT, "apply_gl: unsupported block width");
  }
#undef L
  count_launch();
  KRY_CUDA(cudaGetLastError());
  return KRY_OK;
}

// this warp waits until every chunk holding a stencil neighbour row of chunk
// u is complete (c.fpl releases per chunk and launch)
__device__ __forceinline__ void step_wait(const OpDev& op, const StepCall& c, int64_t u,
                                          const unsigned* flags) {
  const int lane = threadIdx.x & 31;
  if (lane < 14) {
    const int k = lane >> 1;
    const int64_t first = u * c.ch;
    const int64_t last = min(first + c.ch, c.n) - 1;
    const int64_t mag = (k == 0 || k == 6) ? op.nxy : (k == 1 || k == 5) ? op.nx : (k == 3 ? 0 : 1);
    int64_t row = ((lane & 1) ? last : first) + (k < 3 ? -mag : mag);
    row = row < 0 ? 0 : (row >= c.n ? c.n - 1 : row);
    const unsigned* f = flags + row / c.ch;
    const unsigned want = c.fpl * c.epoch;
    while ((int)(ld_acquire_u32(f) - want) < 0) __nanosleep(32);
  }
  __syncwarp();
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int S>
__global__ void __launch_bounds__(STEP_TP, KRY_STEP_MINB) k_step(OpDev op, StepCall c, DevState* st,
                                                                 TStore T, StepScratch sc) {
  constexpr bool PAIR = step_pair(S);
  __shared__ __align__(16) double sbuf[4 * STEP_PART];   // warp partials / post scratch
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  // A fragments of [Mo; Mc; Mw]^T: lane (g, t) holds M_b[k][g] for the
  // source column k of k-step h (k = 2t + h paired, k = t single)
  double aM[3][2];
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = PAIR ? 2 * t + h : t;
      aM[b][h] = (k < S && g < S && (PAIR || h == 0)) ? st->M[b * 64 + k * 8 + g] : 0.0;
    }
  double acc[STEP_NBLK][2];
#pragma unroll
  for (int b = 0; b < STEP_NBLK; ++b) acc[b][0] = acc[b][1] = 0.0;
  // static round robin: CTA b takes tickets b, b + G, ...; ticket tk produces
  // chunk tk and consumes chunk tk - lag (lag = c.lag grid strides: the
  // consumed chunk is this CTA's own chunk of c.lag iterations ago).  The
  // warps of a CTA work independently (per-warp completion counts).
  const int64_t G = gridDim.x;
  const int64_t lag = (int64_t)c.lag * G;
  const int64_t chunk_bytes = (int64_t)c.ch * c.ld * 8;
  for (int64_t tk = blockIdx.x; tk - lag < c.nch; tk += G) {
    if (tk < c.nch) {
      const int64_t u = c.reverse ? c.nch - 1 - tk : tk;
      // L2 prefetch of the next ticket's centre rows (V_{m-1}, V_m)
      if (threadIdx.x == 0 && tk + G < c.nch) {
        const int64_t un = c.reverse ? c.nch - 1 - (tk + G) : tk + G;
        const int64_t bytes = min(chunk_bytes, (c.n - un * c.ch) * c.ld * 8) & ~15ll;
        if (bytes > 0) {
          prefetch_l2(c.vc + un * c.ch * c.ld, (uint32_t)bytes);
          prefetch_l2(c.vo + un * c.ch * c.ld, (uint32_t)bytes);
        }
      }
      step_produce<S>(op, c, u, aM);
      __syncwarp();
      if (lane == 0) red_release_add(sc.flags + u, 1u);
    }
    if (tk >= lag) {
      const int64_t u = c.reverse ? c.nch - 1 - (tk - lag) : tk - lag;
      step_wait(op, c, u, sc.flags);
      step_consume<S>(op, c, u, acc);
    }
  }
  // fixed-order grid reduction (by CTA index) + carried blocks + the
  // coefficient solve of the next step on the last CTA
  finish_reduction<STEP_NBLK * 8>(acc, sbuf, sc.part, sc.gcnt, POST_FUSED, st, T);
}

void step_geometry(const OpDev& op, int64_t n, int* ch, int* nch, int* lag) {
  const int c = 128;
  *ch = c;
  *nch = (int)((n + c - 1) / c);
  const int64_t reach = (int64_t)std::max(op.nxy, op.nx);
  *lag = (int)((reach + c - 1) / c) + 1;
}

bool step_supported(const OpDev& op, int s, int64_t ld) {
  if (op.kind != KRY_OP_STENCIL || op.halo_lo || op.halo_hi) return false;
  if (s < 1 || s > 8 || s == 5 || s == 7) return false;
  if (s > 4 && (ld % 2) != 0) return false;
  return true;
}

template <class Kern>
static int step_grid(Kern kernel, int nch) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache_dev[64];   // per device
  int per = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto& cache = cache_dev[dev & 63];
    auto it = cache.find((const void*)kernel);
    if (it == cache.end()) {
      int sms = 148, nb = 1;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, STEP_TP, 0);
      per = std::max(1, nb) * sms;
      cache[(const void*)kernel] = per;
    } else {
      per = it->second;
    }
  }
  return std::max(1, std::min(std::min(per, nch), KRY_MAX_GRID));
}

#include "step_tma.cuh"

template <class Kern>
static int step_grid_smem(Kern kernel, int nch, int threads, size_t smem) {
  int dev = 0, sms = 148, nb = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem);
  return std::max(1, std::min(std::min(std::max(1, nb) * sms, nch), KRY_MAX_GRID));
}

// Cooperative launch: every CTA is co-resident (the static ticket order
// spins on flags of other CTAs), and the per-CTA partials are reduced in CTA
// order, so the result is independent of timing (pass 2 == pass 1 bitwise).
int launch_step(cudaStream_t st, int s, const OpDev& op, StepCall c, DevState* dst,
                const TStore& T, StepScratch& sc, float* prof_ms, cudaEvent_t* ev) {
  c.epoch = ++sc.epoch;
  const void* fn = nullptr;
  int grid = 1, threads = STEP_TP;
  size_t smem = 0;
  // even widths: TMA-staged kernel (16-byte aligned bulk copies of whole
  // point rows); odd widths: register-gather kernel
#define L(S)                                \
  grid = step_grid(k_step<S>, c.nch);       \
  fn = (const void*)k_step<S>;              \
  c.fpl = STEP_TP / 32
#define LT(S)                                                                            \
  {                                                                                      \
    static bool attr_dev[64] = {false};   /* per device */                               \
    int adev = 0;                                                                        \
    cudaGetDevice(&adev);                                                                \
    bool& attr = attr_dev[adev & 63];                                                    \
    smem = tma_smem_bytes(S);                                                            \
    if (!attr) {                                                                         \
      KRY_CUDA(cudaFuncSetAttribute(k_step_tma<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                    (int)smem));                                         \
      attr = true;                                                                       \
    }                                                                                    \
    grid = step_grid_smem(k_step_tma<S>, c.nch, TMA_TP + 64, smem);                      \
    fn = (const void*)k_step_tma<S>;                                                     \
    threads = TMA_TP + 64;                                                               \
    c.fpl = 1;                                                                           \
  }
  const char* reg = getenv("KRY_STEP_REGISTER");
  const bool tma = !(reg && reg[0] == '1');
  switch (s) {
    case 1: L(1); break;
    case 2: if (tma) LT(2) else { L(2); } break;
    case 3: L(3); break;
    case 4: if (tma) LT(4) else { L(4); } break;
    case 6: if (tma) LT(6) else { L(6); } break;
    case 8: if (tma) LT(8) else { L(8); } break;
    default: return fail(KRY_ERR_ARGUMENT, "fused step: unsupported block width");
  }
#undef L
#undef LT
  if (grid > sc.nch_cap) return fail(KRY_ERR_STATE, "fused step scratch too small");
  // lag in grid strides: the consumed chunk is the CTA's own chunk of
  // c.lag iterations ago, at least `lag` chunks behind the production front
  // (TMA kernel: four more strides: the consumption copies are issued two
  // iterations ahead and a chunk is released two iterations after it is
  // produced)
  c.lag = std::max(1, (c.lag + grid - 1) / grid) + (smem ? 4 : 0);
  void* args[] = {(void*)&op, (void*)&c, (void*)&dst, (void*)&T, (void*)&sc};
  if (prof_ms && ev) cudaEventRecord(ev[0], st);
  KRY_CUDA(cudaLaunchCooperativeKernel(fn, grid, threads, args, smem, st));
  if (prof_ms && ev) cudaEventRecord(ev[1], st);
  count_launch();
  return KRY_OK;
}
