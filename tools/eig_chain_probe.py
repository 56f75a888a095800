"""Time the incremental eigen engine alone (kry_partial_eig: all block appends
of a golden's T_m, no recurrence running beside it)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1602_05033_b200 import _lib
lib = _lib.load()
for cfg in sys.argv[1:] or ["c4"]:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
    if cfg == "c5":
        g = np.load(os.path.join(path, "noise", "c5_blocks_csr.npz")); d, o = g["diag_a"], g["sub_a"]
    else:
        g = np.load(os.path.join(path, cfg + ".npz")); d, o = g["t_diag"], g["t_off"]
    d = np.ascontiguousarray(d); o = np.ascontiguousarray(o[:d.shape[0] - 1])
    m, s = d.shape[0], d.shape[1]; k = m * s
    lam = np.zeros(k); f = np.zeros((s, k)); l = np.zeros((s, k))
    for rep in range(3):
        t = time.perf_counter(); n0 = lib.kry_launch_count()
        _lib.check(lib.kry_partial_eig(0, s, m, _lib.as_dptr(d), _lib.as_dptr(o), _lib.as_dptr(lam), _lib.as_dptr(f), _lib.as_dptr(l)))
        dt = time.perf_counter() - t
        print(cfg, "k", k, "eigen chain alone %.1f ms (%.1f us per scalar row, %d launches)" % (dt * 1e3, dt * 1e6 / k, lib.kry_launch_count() - n0), flush=True)
