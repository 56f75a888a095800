import sys, time
sys.path.insert(0, ".")
import bench
import paper_1602_05033_b200 as kb
cfg, op, _ = bench.build_problem(sys.argv[1])
opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
for rep in range(3):
    t = time.perf_counter()
    sol = kb.solve_lyapunov(op, cfg["c"], opts)
    print("rep", rep, "time %.3f" % (time.perf_counter() - t), "rec %.3f" % sol.recovery_seconds, file=sys.stderr, flush=True)
