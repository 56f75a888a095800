"""Small solves that exercise every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

* Lyapunov on a constant 3-D stencil, s = 4 (TMA apply, hand-off combine,
  eigen engine, DMMA Cauchy contraction, finalisation, pass-2 regeneration +
  DMMA factor accumulation), windowed and stored;
* Lyapunov on a variable-coefficient 2-D stencil, s = 1 (staged apply) and
  on a general CSR matrix, s = 3;
* an ill-conditioned right-hand side (shifted CholQR3 fallback);
* two-sided Sylvester (pipelined two-context loop) and one-sided Sylvester;
* the slab-sharded path with 2 loopback ranks.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

import paper_1602_05033_b200 as kb  # noqa: E402
from oracle import problems as P  # noqa: E402
from paper_1602_05033_b200.operators import StencilOperator, detect_stencil  # noqa: E402
from paper_1602_05033_b200.parallel import local_rows, run_ranks, slab_partition  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    a = P.laplacian3d(16)
    c = rng.standard_normal((a.shape[0], 4))
    for storage in ("windowed", "stored"):
        sol = kb.solve_lyapunov(kb.SparseOperator(a), c,
                                kb.SolveOptions(tol=1e-8, max_m=80, storage=storage))
        print("lyap 3d s4", storage, sol.iterations, sol.rank, flush=True)
    av = P.varcoef2d(40)
    sol = kb.solve_lyapunov(kb.SparseOperator(av), rng.standard_normal((1600, 1)),
                            kb.SolveOptions(tol=1e-8, max_m=200, storage="windowed"))
    print("lyap varcoef s1", sol.iterations, sol.rank, flush=True)
    b = sp.random(600, 600, density=0.02, random_state=np.random.RandomState(3), format="csr")
    acsr = (b + b.T - sp.diags(np.full(600, 12.0))).tocsr()
    sol = kb.solve_lyapunov(kb.SparseOperator(acsr), rng.standard_normal((600, 3)),
                            kb.SolveOptions(tol=1e-8, max_m=150, storage="windowed"))
    print("lyap csr s3", sol.iterations, sol.rank, flush=True)
    u, _ = np.linalg.qr(rng.standard_normal((300, 3)))
    cill = u @ np.diag([1.0, 1e-5, 1e-10])
    ad = sp.diags(-np.linspace(1.0, 80.0, 300)).tocsr()
    sol = kb.solve_lyapunov(kb.SparseOperator(ad), cill,
                            kb.SolveOptions(tol=1e-8, max_m=100, storage="windowed"))
    print("lyap ill-conditioned C", sol.iterations, sol.rank, flush=True)
    sa, sb_ = P.laplacian2d(30), P.laplacian3d(10)
    sol = kb.solve_sylvester_two_sided(kb.SparseOperator(sa), kb.SparseOperator(sb_),
                                       rng.standard_normal((900, 2)),
                                       rng.standard_normal((1000, 2)),
                                       kb.SolveOptions(tol=1e-8, max_m=200, storage="windowed"))
    print("sylv two-sided", sol.iterations, sol.rank, flush=True)
    bd = P.laplacian1d(30).toarray()
    sol = kb.solve_sylvester_one_sided(kb.SparseOperator(sa), bd, rng.standard_normal((900, 2)),
                                       rng.standard_normal((30, 2)),
                                       kb.SolveOptions(tol=1e-8, max_m=200))
    print("sylv one-sided", sol.iterations, sol.rank, flush=True)
    st = detect_stencil(a)
    grid = (16, 16, 16)

    def rank(r, comm):
        z = slab_partition(16, 2, r)
        op = StencilOperator(grid, st["c_diag"], st["c_x"], st["c_y"], st["c_z"], slab=z,
                             comm=comm)
        return kb.solve_lyapunov(op, local_rows(c, grid, z),
                                 kb.SolveOptions(tol=1e-8, max_m=80, storage="windowed"))

    sols = run_ranks(2, rank)
    print("sharded 2 ranks", sols[0].iterations, sols[0].rank, flush=True)
    print("SANITIZE_RUN_OK")


if __name__ == "__main__":
    main()
