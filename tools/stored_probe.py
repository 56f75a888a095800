"""c4 through the API: storage='stored' (basis kept on the device) vs 'windowed' (two pass)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
import paper_1602_05033_b200 as kb

cfg, op, _ = bench.build_problem("c4")
pinned = torch.from_numpy(np.ascontiguousarray(cfg["c"])).pin_memory().numpy()
z_ref = None
for storage in ("windowed", "stored", "windowed", "stored"):
    opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage=storage)
    torch.cuda.synchronize()
    t = time.perf_counter()
    sol = kb.solve_lyapunov(op, pinned, opts)
    dt = time.perf_counter() - t
    extra = ""
    if z_ref is None:
        z_ref = sol.z.copy()
    else:
        extra = "max|dz| / max|z| = %.2e" % (np.max(np.abs(sol.z - z_ref)) / np.max(np.abs(z_ref)))
    print("%-8s %.3f s  its %d rank %d basis %.3f res %.3f rec %.3f peak %d %s" % (
        storage, dt, sol.iterations, sol.rank, sol.basis_seconds, sol.residual_seconds,
        sol.recovery_seconds, sol.peak_basis_vectors, extra), flush=True)
    del sol
