"""Golden fixtures of the one-sided Sylvester solver,
produced by running the REFERENCE package itself (build container only):

    python tests/golden/make_golden_sylv1.py

Problems: A = krymat.problems.gen_fd2d(kind, n) (large sparse side), B the
dense small side 10 * laplacian1d(n) (the reference's fd3d-split pair,
problems.py:78-85) or a shifted variant; C1, C2 seeded standard normal.
Outputs tests/golden/sylv1_<name>.npz: history, iterations, rank, truncation
mass and the factor sketches X @ Omega2, X^T @ Omega1 (X = Z1 Z2^T).
"""

import os
import sys

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import krymat.problems as kp  # noqa: E402
import krymat.solvers as ks  # noqa: E402
from krymat.operators import SparseOperator  # noqa: E402
from oracle import problems as op_  # noqa: E402

CASES = {
    # name: (kind, n, s, seed, tol)
    "exp30": ("fd2d-exp", 30, 2, 11, 1e-8),
    "lap40": ("laplacian2d", 40, 3, 12, 1e-9),
}


def run(name):
    kind, n, s, seed, tol = CASES[name]
    a, bl = kp.gen_fd3d_split(n) if kind == "fd2d-exp" else (kp.gen_fd2d(kind, n),
                                                              10.0 * kp.laplacian1d(n))
    b = bl.toarray()
    rng = np.random.default_rng(seed)
    c1 = rng.standard_normal((a.shape[0], s))
    c2 = rng.standard_normal((b.shape[0], s))
    sol = ks.solve_sylvester_one_sided(
        SparseOperator(a), b, c1, c2, ks.SolveOptions(tol=tol, max_m=300, storage="windowed"))
    om1 = op_.sketch_omega(a.shape[0], 2)
    om2 = op_.sketch_omega(b.shape[0], 2)
    out = dict(
        history=np.array(sol.history), iterations=np.int64(sol.iterations),
        rank=np.int64(sol.rank), discarded=np.float64(sol.truncation_discarded),
        final_residual=np.float64(sol.final_residual),
        peak_basis_vectors=np.int64(sol.peak_basis_vectors),
        sketch_right=sol.z1 @ (sol.z2.T @ om2), sketch_left=sol.z2 @ (sol.z1.T @ om1),
        digest_a=np.array(op_.csr_digest(a)), b=b, c1=c1, c2=c2, tol=np.float64(tol))
    np.savez_compressed(os.path.join(HERE, "sylv1_%s.npz" % name), **out)
    print(name, "iterations", sol.iterations, "rank", sol.rank, "res", sol.final_residual)


if __name__ == "__main__":
    for nm in (sys.argv[1:] or list(CASES)):
        run(nm)
