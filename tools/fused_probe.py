"""GPU probe: fused single-pass step vs the two-kernel path (same process,
KRY_NO_FUSED_STEP read at context creation) on small grids and configs."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1602_05033_b200 as kb
from paper_1602_05033_b200 import problems as P
import bench


def run(op, c, tol, max_m, fused):
    os.environ["KRY_FUSED_STEP"] = "1" if fused else "0"
    t = time.perf_counter()
    sol = kb.solve_lyapunov(op, c, kb.SolveOptions(tol=tol, max_m=max_m, storage="windowed"))
    return sol, time.perf_counter() - t


cases = [("L3D 13^3", lambda: kb.SparseOperator(P.laplacian3d(13)), 2197),
         ("L2D 37^2", lambda: kb.SparseOperator(P.gen_fd2d("laplacian2d", 37)), 1369),
         ("var2D 29^2", lambda: kb.SparseOperator(P.gen_fd2d("varcoef2d", 29)), 841)]
for name, mk, n in cases:
    for s in (1, 2, 3, 4, 6, 8):
        c = np.random.default_rng(s).standard_normal((n, s))
        a, ta = run(mk(), c, 1e-9, 200, True)
        b, tb = run(mk(), c, 1e-9, 200, False)
        h1 = np.array([r[2] for r in a.history]); h2 = np.array([r[2] for r in b.history])
        k = min(len(h1), len(h2))
        x1 = a.z @ a.z.T; x2 = b.z @ b.z.T
        print("%-10s s=%d its %d/%d rank %d/%d hist maxrel %.2e X rel %.2e" % (
            name, s, a.iterations, b.iterations, a.rank, b.rank,
            np.max(np.abs(h1[:k] - h2[:k]) / h2[:k]), np.linalg.norm(x1 - x2) / np.linalg.norm(x2)),
            flush=True)
for cfg_name in sys.argv[1:] or ["c2", "c4"]:
    cfg, op, _ = bench.build_problem(cfg_name)
    for fused in (True, False, True):
        sol, dt = run(op, cfg["c"], cfg["tol"], cfg["max_m"], fused)
        h = np.array([r[2] for r in sol.history])
        print(cfg_name, "fused" if fused else "2-kernel", "its", sol.iterations, "rank", sol.rank,
              "time %.3f basis %.3f res %.3f rec %.3f" % (dt, sol.basis_seconds, sol.residual_seconds,
                                                          sol.recovery_seconds),
              "last rel %.6e" % h[-1], flush=True)
