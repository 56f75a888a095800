"""Wall time of one solve of each BASELINE config through the public API
(second of two runs; c5 ends in the expected ConvergenceError)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1602_05033_b200 as kb

for name in sys.argv[1:] or ["c1", "c2", "c3", "c5"]:
    cfg, op, opb = bench.build_problem(name)
    opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
    for rep in range(2):
        t = time.perf_counter()
        try:
            if cfg["kind"] == "sylvester":
                sol = kb.solve_sylvester_two_sided(op, opb, cfg["c1"], cfg["c2"], opts)
            else:
                sol = kb.solve_lyapunov(op, cfg["c"], opts)
            info = "its %d rank %d rel %.3e" % (sol.iterations, sol.rank, sol.final_residual)
        except kb.ConvergenceError as e:
            info = "ConvergenceError after %d checks (last %.3e)" % (len(e.history), e.history[-1][2])
        dt = time.perf_counter() - t
    print("%s %.3f s  %s" % (name, dt, info), flush=True)
