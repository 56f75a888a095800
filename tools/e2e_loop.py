"""Per-solve wall time of consecutive API solves (bench e2e pattern)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
import paper_1602_05033_b200 as kb

cfg, op, _ = bench.build_problem("c4")
pinned = torch.from_numpy(np.ascontiguousarray(cfg["c"])).pin_memory().numpy()
opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
for r in range(5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    sol = kb.solve_lyapunov(op, pinned, opts)
    dt = time.perf_counter() - t
    print("solve %d %.3f s  basis %.3f res %.3f rec %.3f pinned=%s" % (
        r, dt, sol.basis_seconds, sol.residual_seconds, sol.recovery_seconds,
        torch.cuda.is_available() and sol.z.base is not None), flush=True)
    del sol
