"""Time the host-facing parts of one c4 solve through the public API
(KRY_TIMING=1 adds the library's own stage timers on stderr)."""
import ctypes, sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1602_05033_b200 as kb
from paper_1602_05033_b200 import _lib, solvers
import torch

cfg, op, _ = bench.build_problem(sys.argv[1] if len(sys.argv) > 1 else "c4")
c = cfg["c"]
pinned = torch.from_numpy(np.ascontiguousarray(c)).pin_memory().numpy()
opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
lib = _lib.load()
for r in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p1 = solvers._Pass1(op, pinned, opts)
    t1 = time.perf_counter()
    hist = np.zeros((opts.max_m + 1, 5))
    nh, its, reason = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    rel = ctypes.c_double(np.inf)
    _lib.check(lib.kry_solve_lyap_pass1(p1.ctx.ptr, float(opts.tol), int(opts.max_m), 1,
                                        _lib.as_dptr(hist), ctypes.byref(nh), ctypes.byref(its),
                                        ctypes.byref(rel), ctypes.byref(reason)))
    t2 = time.perf_counter()
    rank, disc = ctypes.c_int(0), ctypes.c_double(0.0)
    _lib.check(lib.kry_finalize_lyap(p1.ctx.ptr, float(opts.trunc_eps), ctypes.byref(rank),
                                     ctypes.byref(disc)))
    t3 = time.perf_counter()
    z = np.empty((op.n, rank.value))
    t4 = time.perf_counter()
    _lib.check(lib.kry_recover(p1.ctx.ptr, _lib.as_dptr(z)))
    t5 = time.perf_counter()
    p1.ctx.close()
    t6 = time.perf_counter()
    print("run %d: ctx+init %.3f pass1 %.3f finalize %.3f alloc %.3f recover %.3f close %.3f total %.3f"
          % (r, t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t6 - t0), flush=True)
    t = time.perf_counter()
    sol = kb.solve_lyapunov(op, pinned, opts)
    print("   api solve %.3f" % (time.perf_counter() - t), flush=True)
