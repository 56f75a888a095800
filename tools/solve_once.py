"""One device-resident solve of a config (for ncu launch lists)."""
import argparse, sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1602_05033_b200 as kb

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--max-m", type=int, default=0)
args = ap.parse_args()
cfg, op, _ = bench.build_problem(args.config)
opts = kb.SolveOptions(tol=cfg["tol"], max_m=args.max_m or cfg["max_m"], storage="windowed")
t = time.perf_counter()
try:
    sol = kb.solve_lyapunov(op, cfg["c"], opts)
    print("iterations", sol.iterations, "rank", sol.rank, "time", time.perf_counter() - t,
          "basis", sol.basis_seconds, "res", sol.residual_seconds, "rec", sol.recovery_seconds)
except kb.ConvergenceError as e:
    print("no convergence", len(e.history), time.perf_counter() - t)
