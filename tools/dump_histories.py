"""Run configs through the public API on the GPU and save their residual
histories (and, for c5, the fixed-depth factor sketch) under gpurun_out/,
for calibrating the parity floors against the reference goldens.

    python tools/dump_histories.py c3 c5
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1602_05033_b200 as kb  # noqa: E402

OUT = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for name in names:
        cfg, op, opb = bench.build_problem(name)
        opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
        t = time.perf_counter()
        out = {}
        try:
            if cfg["kind"] == "sylvester":
                sol = kb.solve_sylvester_two_sided(op, opb, cfg["c1"], cfg["c2"], opts)
            else:
                sol = kb.solve_lyapunov(op, cfg["c"], opts)
            out["history"] = np.array(sol.history)
            out["iterations"] = sol.iterations
            out["rank"] = sol.rank
        except kb.ConvergenceError as e:
            out["history"] = np.array(e.history)
        out["wall"] = time.perf_counter() - t
        np.savez_compressed(os.path.join(OUT, "hist_%s.npz" % name), **out)
        print(name, len(out["history"]), out["wall"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
