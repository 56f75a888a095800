// Internal declarations of libkrymat_b200 (not part of the C-ABI).
//
// Data layout in HBM
//   * block vectors: n x s row-major ("point major"): the s values of one grid
//     point are contiguous; consecutive points are `ld` doubles apart (ld = s
//     everywhere: the pass-1 window and the pass-2 chunk slots share the
//     ring layout, a block is written once).
//   * s x s blocks: fixed 8 x 8 row-major slots (s <= 8), zero padded.
//   * projected matrix T_m: per-step slots of the raw MGS sums, symmetrised
//     diagonal blocks, coupling blocks tau (R factors) and the lazy CholQR2
//     corrections S_i (true basis block = stored block * S_i).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include "../../include/krymat_b200.h"

#define KRY_SMAX 8
#define KRY_SS 64
#define KRY_MAX_GRID (148 * 16)
// grid-reduction counters: [0] top level, [1 + group] per group of 32 CTAs
#define KRY_TICKET_STRIDE (2 + KRY_MAX_GRID / 32)
#define KRY_TICKET_SITES 3

namespace kry {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

// Device allocations go through the stream-ordered pool on the legacy stream
// (ordered with every blocking stream of a context): repeated solves and
// finalisations reuse cached memory, and a free never synchronises the
// device (plain cudaFree did, which made finalisation times erratic).
template <class T>
inline int dalloc(T** p, size_t count) {
  cudaError_t e = cudaMallocAsync((void**)p, count * sizeof(T) + 16, (cudaStream_t)0);
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(KRY_ERR_CUDA, std::string("cudaMallocAsync failed: ") + cudaGetErrorString(e) +
                                  " (" + std::to_string(count * sizeof(T)) + " bytes)");
  }
  return KRY_OK;
}
template <class T>
inline void dfree(T* p) {
  if (p) cudaFreeAsync((void*)p, (cudaStream_t)0);
}
// keep freed pool memory cached in the process (once per device)
void keep_pool_memory(int device);
extern thread_local std::string g_last_error;

#define KRY_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess)                                                    \
      return ::kry::fail(KRY_ERR_CUDA, std::string("CUDA error: ") +          \
                                           cudaGetErrorString(_e) + " at " +  \
                                           __FILE__ + ":" +                   \
                                           std::to_string(__LINE__));         \
  } while (0)

#define KRY_CHECK(call)                                                       \
  do {                                                                        \
    int _rc = (call);                                                         \
    if (_rc != KRY_OK) return _rc;                                            \
  } while (0)

void count_launch(int k = 1);

#ifdef __CUDACC__
// Programmatic dependent launch: the kernels of an append form a chain of
// short dependent launches on one stream (5 per scalar row, ~10^4 per c4
// solve).  Each kernel lets its successor be scheduled at once
// (launch_dependents) and waits for its predecessor's completion and memory
// flush before touching any data (griddepcontrol.wait), so the launch
// latency of kernel i+1 overlaps the execution of kernel i.  Both are no-ops
// for a launch without the attribute (the finalisation's plain launches).
__device__ __forceinline__ void pdl_sync() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
inline bool& pdl_scope_flag() {
  static thread_local bool on = true;
  return on;
}
struct PdlScope {   // restricts pdl_launch to plain launches inside a scope
  bool prev;
  explicit PdlScope(bool on) : prev(pdl_scope_flag()) { pdl_scope_flag() = on; }
  ~PdlScope() { pdl_scope_flag() = prev; }
};
inline bool pdl_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KRY_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1 && pdl_scope_flag();
}
template <class... KArgs, class... Args>
inline void pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  if (!pdl_on()) {
    kern<<<grid, block, smem, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#ifndef KRY_SECULAR_W8
#define KRY_SECULAR_W8 0
#endif
// poles of the big appends (K > 2048) cached in registers: 1 = 256 threads x
// 24 terms, 2 = 256 x 16 / 512 x 12 (both measured SLOWER on c5: 2.0 / 1.9 s
// against 1.32 s -- one or two CTAs per SM cannot hide the reciprocal chains),
// 0 = streamed from global memory / L1 with 16 small CTAs per SM
#ifndef KRY_SECULAR_BIG
#define KRY_SECULAR_BIG 0
#endif
#endif

// ---------------------------------------------------------------- operator
// division by an invariant 32-bit divisor: q = (umulhi(n, mul) + n) >> shift
// (round-up method, valid for n < 2^31)
struct FastDiv {
  unsigned d, mul, shift;
};
inline FastDiv make_fastdiv(unsigned d) {
  FastDiv f;
  f.d = d;
  unsigned l = 0;
  while ((1ull << l) < d) ++l;
  f.shift = l;
  f.mul = (unsigned)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
  return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ unsigned fdiv(unsigned n, const FastDiv& f) {
  return (__umulhi(n, f.mul) + n) >> f.shift;
}
#endif

struct OpDev {
  int kind;      // KRY_OP_STENCIL / KRY_OP_CSR
  int variable;  // stencil coefficient mode
  int nx, ny;    // grid extents in x, y
  int nzl;       // local z planes owned
  int halo_lo, halo_hi;  // 1 if a neighbour plane exists below / above
  int nxy;
  double cd, cx, cy, cz;
  const double *d, *ex, *ey, *ez;  // per point, offset so index 0 = first owned
  const int64_t* rp;
  const int* ci;
  const double* va;
  FastDiv fx, fy;   // division by nx and ny
};

// ---------------------------------------------------------------- device state
// Small per-context state living in device memory.  Written by the last CTA
// of the reduction kernels, read by the next kernels; the host only reads the
// status words.
struct DevState {
  double Goo[KRY_SS], Goc[KRY_SS], Gcc[KRY_SS], GoW[KRY_SS];
  double GcW[KRY_SS], GWW[KRY_SS];
  double So[KRY_SS], Sc[KRY_SS];
  double R1prev[KRY_SS];
  double M[3 * KRY_SS];      // Mo, Mc, Mw of the next combine
  double gamma[KRY_SS];      // finalised gamma
  double gram[KRY_SS * 3];   // scratch Gram result of generic reductions
  double acc_a[KRY_SS], acc_b[KRY_SS];  // explicit-path MGS sums
  double beta2;
  double scale2, w2;
  double replay_err;
  double nrows;              // rows of the Krylov vectors (all ranks): shift of CholQR3
  int status;
  int flags;                 // KRY_FLAG_*
  int step;                  // completed coefficient solves
  int replay;                // pass-2 regeneration: compare coupling blocks (2: queued without
                             // per-step host checks; a fallback poisons replay_err)
  int finalize_on_zero;
  int s;
  int has_old;
  int pad_;
};

enum {
  KRY_FLAG_EXHAUSTED = 1,
  KRY_FLAG_FALLBACK = 2,
  KRY_FLAG_SHIFTED = 4,     // the last Cholesky QR stage used the CholQR3 shift
};

// post-reduction routines run by the last CTA of a Gram reduction
enum PostMode {
  POST_NONE = 0,        // store to st->gram
  POST_P = 1,           // combine kernel: Goc, GoW, Gcc
  POST_STEP = 2,        // apply kernel: GcW, GWW, then coefficient solve
  POST_INIT = 3,        // C^T C -> R0, M = [0, R0^-1, 0], beta2
  POST_MGS_OLD = 4,     // explicit path: alpha = Vo^T W -> acc_a += ; M[0] = alpha
  POST_MGS_CUR = 5,     // explicit path: beta = Vc^T W -> acc_b += ; M[0] = beta
  POST_CHOL1 = 6,       // explicit path: R1 = chol(W^T W), M[0] = R1^-1
  POST_CHOL2 = 7,       // explicit path: R2 = chol(V^T V), M[0] = R2^-1, finish
  POST_SCALE = 8,       // explicit path: scale2 = trace
  POST_W2 = 9,          // explicit path: w2 = trace, zero test
  POST_FUSED = 10,      // fused step kernel: carried blocks + deferred solve of step j+1
  POST_STEP8 = 11,      // POST_STEP with W0^T W0 at row 8 (register-fragment apply kernel)
  POST_CHOL_MID = 12,   // shifted CholQR3 middle stage: R = chol(V^T V), M[0] = R^-1,
                        // gram[0..63] = R1prev = R * gram[0..63] (accumulated R chain)
  POST_GCC = 13,        // Gcc = V^T V (refresh after an explicit re-orthonormalisation)
};

struct TStore {  // projected-matrix storage (device), slots of 64 doubles
  double* draw;  // raw MGS diag sums
  double* dsym;  // symmetrised diagonal blocks
  double* off;   // off_mgs sums
  double* sub;   // coupling blocks tau (final R factors)
  double* S;     // lazy CholQR2 corrections per block
  double* tau1;  // first-stage coupling tau_{j+1,j} of step j (read by the async check)
  int cap;       // number of slots
};

struct GramScratch {
  double* partials;   // [grid][24*8]
  unsigned* ticket;   // KRY_TICKET_SITES disjoint blocks of KRY_TICKET_STRIDE counters
  int max_grid;
};

// ---------------------------------------------------------------- kernels (host wrappers)
struct CombineCall {
  const double* vo; int64_t ldo;
  const double* vc; int64_t ldc;
  double* vn; int64_t ldn;
  int64_t n;
  int has_old, use_op, write_new, reverse;
  int post = POST_P;   // POST_NONE in multi-GPU mode (all-reduce, then k_post)
  double* vn2 = nullptr;   // optional second copy of V_{m+1} (pass-2 chunk buffer)
  int64_t ldn2 = 0;
  const double* win = nullptr;   // A V_m stored by the apply kernel (n x s, ld s)
  int grid_cap = 0;              // > 0: at most this many CTAs
};
int launch_combine(cudaStream_t st, int s, const OpDev& op, const CombineCall& c,
                   DevState* dst, const TStore& T, GramScratch& g, int grid,
                   float* prof_ms, cudaEvent_t* ev);
struct ApplyGramCall {
  const double* v; int64_t ldv;
  int64_t n;
  int use_op;        // 1: X=[V|AV], Y=AV ; 0: X=[V], Y=V
  int post;          // PostMode
  int reverse;
  double* wout = nullptr;   // also store A V (n x s, ld s) for the combine kernel
  int grid_cap = 0;         // > 0: at most this many CTAs
};
int launch_apply_gram(cudaStream_t st, int s, const OpDev& op,
                      const ApplyGramCall& c, DevState* dst, const TStore& T,
                      GramScratch& g, int grid);
// generic X^T Y with X,Y given blocks (explicit path); result to post routine
int launch_pair_gram(cudaStream_t st, int s, const double* x, int64_t ldx,
                     const double* y, int64_t ldy, int64_t n, int post,
                     DevState* dst, const TStore& T, GramScratch& g, int grid);
// y[i] = A x[i] (block), write
int launch_apply_store(cudaStream_t st, int s, const OpDev& op, const double* x,
                       int64_t ldx, double* y, int64_t ldy, int64_t n);
// w[i] -= x[i] * Mdev (s x s at dst->M[0]) ; or w = w * Mdev when x == nullptr
int launch_update(cudaStream_t st, int s, double* w, int64_t ldw, const double* x,
                  int64_t ldx, const double* mdev, int64_t n, int subtract);
int launch_copy_block(cudaStream_t st, int s, const double* x, int64_t ldx,
                      double* y, int64_t ldy, int64_t n);
// explicit-step bookkeeping kernel (1 CTA): store T slots from acc, etc.
int launch_explicit_finish(cudaStream_t st, DevState* dst, const TStore& T, int mode);
// post routine on st->gram (the all-reduced Gram totals) in one CTA
int launch_post(cudaStream_t st, int post, DevState* dst, const TStore& T);

int gram_grid_for(int64_t n);



// ---------------------------------------------------------------- fused single-pass step
// One kernel per block-Lanczos step (stencil operators): produces
// V_{m+1} = V_{m-1} Mo + V_m Mc + (A V_m) Mw chunk by chunk and, trailing the
// production front by `lag` chunks inside the same launch, consumes it:
// W0 = A V_{m+1} from the just-written (L2-resident) rows and the Gram blocks
// [V_m^T V_{m+1} | V_m^T W0 | V_{m+1}^T V_{m+1} | V_{m+1}^T W0 | W0^T W0] of
// the next coefficient solve, which the last CTA runs (POST_FUSED).  HBM
// traffic per step: read V_{m-1}, V_m, write V_{m+1} (the three-term minimum).
struct StepCall {
  const double* vo;      // V_{m-1} (nullptr at step 1)
  const double* vc;      // V_m
  double* vn;            // V_{m+1}
  int64_t ld;            // point stride of the three ring blocks (= s)
  double* vn2 = nullptr; // optional second copy of V_{m+1} (pass-2 chunk buffer)
  int64_t ldn2 = 0;
  int64_t n = 0;
  int has_old = 0;
  int ch = 0;            // points per chunk (multiple of 32)
  int nch = 0;           // number of chunks
  int lag = 0;           // consumption lag (chunks; grid strides in the kernel)
  int reverse = 0;       // chunk order descending (L2 reuse across steps)
  unsigned epoch = 0;    // launch counter of this context
  unsigned fpl = 1;      // flag increments per chunk and launch (producer warps or CTAs)
};
struct StepScratch {
  double* part = nullptr;     // [grid + grid/32 + 1][320] per-CTA / per-group partials
  unsigned* gcnt = nullptr;   // [grid/32 + 2] completion counters (self-resetting)
  unsigned* flags = nullptr;  // [nch] production epochs
  int nch_cap = 0;            // max grid
  unsigned epoch = 0;
};
// fused-step geometry for an operator of n local points
void step_geometry(const OpDev& op, int64_t n, int* ch, int* nch, int* lag);
bool step_supported(const OpDev& op, int s, int64_t ld);
// apply + Gram with register DMMA fragments (no shared-memory staging): one
// GPU, stencil, even s, V a ring slot with zero halos; stores A V to c.wout
int apply_mode(const OpDev& op, int s);
int launch_apply_gl(cudaStream_t st, int s, const OpDev& op, const ApplyGramCall& c,
                    DevState* dst, const TStore& T, GramScratch& g);
int launch_apply_tma(cudaStream_t st, int s, const OpDev& op, const ApplyGramCall& c,
                     DevState* dst, const TStore& T, GramScratch& g);
int launch_step(cudaStream_t st, int s, const OpDev& op, StepCall c, DevState* dst,
                const TStore& T, StepScratch& sc, float* prof_ms, cudaEvent_t* ev);

}  // namespace kry
