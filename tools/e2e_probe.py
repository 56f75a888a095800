"""Time the host-facing parts of one c4 solve through the public API."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1602_05033_b200 as kb
import torch

cfg, op, _ = bench.build_problem("c4")
c = cfg["c"]
pinned = torch.from_numpy(np.ascontiguousarray(c)).pin_memory().numpy()
opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
for r in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    sol = kb.solve_lyapunov(op, pinned, opts)
    print("solve", r, time.perf_counter() - t, "basis", sol.basis_seconds, "rec", sol.recovery_seconds, flush=True)
