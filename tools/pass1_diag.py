import sys, time, ctypes
sys.path.insert(0, ".")
import numpy as np
import bench, paper_1602_05033_b200 as kb
from paper_1602_05033_b200 import _lib
cfg, op, _ = bench.build_problem(sys.argv[1])
m = int(sys.argv[2])
ctx = op.context(cfg["c"].shape[1], m + 2)
lib = _lib.load()
c = np.ascontiguousarray(cfg["c"])
for rep in range(3):
    g = np.zeros((c.shape[1],) * 2); b2 = ctypes.c_double()
    lib.kry_init_basis(ctx.ptr, _lib.as_dptr(c), _lib.as_dptr(g), ctypes.byref(b2))
    hist = np.zeros((m + 1, 5)); nh, its, why = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(); rel = ctypes.c_double()
    t = time.perf_counter()
    lib.kry_solve_lyap_pass1(ctx.ptr, 1e-30, m, 1, _lib.as_dptr(hist), ctypes.byref(nh), ctypes.byref(its), ctypes.byref(rel), ctypes.byref(why))
    print(sys.argv[1], "rep", rep, "pass1 %.4f s for %d steps" % (time.perf_counter() - t, m), flush=True)
ctx.close()
