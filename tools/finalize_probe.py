"""Time kry_finalize_lyap repeatedly after one pass 1 (finalisation variance probe)."""
import ctypes, sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1602_05033_b200 as kb
from paper_1602_05033_b200 import _lib, solvers

cfg, op, _ = bench.build_problem(sys.argv[1] if len(sys.argv) > 1 else "c4")
opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
lib = _lib.load()
p1 = solvers._Pass1(op, np.asarray(cfg["c"], dtype=float), opts)
hist = np.zeros((opts.max_m + 1, 5))
nh, its, reason = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
rel = ctypes.c_double(0)
t = time.perf_counter()
_lib.check(lib.kry_solve_lyap_pass1(p1.ctx.ptr, float(opts.tol), int(opts.max_m), 1, _lib.as_dptr(hist),
                                    ctypes.byref(nh), ctypes.byref(its), ctypes.byref(rel), ctypes.byref(reason)))
print("pass1", time.perf_counter() - t, "its", its.value, flush=True)
for r in range(8):
    rank, disc = ctypes.c_int(0), ctypes.c_double(0.0)
    t = time.perf_counter()
    _lib.check(lib.kry_finalize_lyap(p1.ctx.ptr, float(opts.trunc_eps), ctypes.byref(rank), ctypes.byref(disc)))
    print("finalize", r, time.perf_counter() - t, "rank", rank.value, flush=True)
import torch
k = its.value * 8
a = torch.randn(k, k, dtype=torch.float64, device="cuda")
a = a + a.T
for r in range(6):
    torch.cuda.synchronize(); t = time.perf_counter()
    torch.linalg.eigh(a)
    torch.cuda.synchronize(); print("torch eigh", k, time.perf_counter() - t, flush=True)
p1.ctx.close()
