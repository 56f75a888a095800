"""Time kry_band_eigh (band divide and conquer) on a golden's T_m."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1602_05033_b200 import _lib
lib = _lib.load()
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", cfg + ".npz"))
d = np.ascontiguousarray(g["t_diag"]); o = np.ascontiguousarray(g["t_off"])
m, s = d.shape[0], d.shape[1]
k = m * s
lam = np.zeros(k); q = np.zeros((k, k), order="F")
for r in range(reps):
    t = time.perf_counter()
    n0 = lib.kry_launch_count()
    _lib.check(lib.kry_band_eigh(0, s, m, _lib.as_dptr(d), _lib.as_dptr(o), _lib.as_dptr(lam), q.ctypes.data_as(_lib.dptr)))
    print(cfg, "k", k, "band eigh wall %.1f ms (incl. %.1f MB copies), launches %d" % ((time.perf_counter() - t) * 1e3, k * k * 8 / 1e6, lib.kry_launch_count() - n0), flush=True)
