"""Generate golden fixtures by running the REFERENCE package (krymat) itself.

Run in the build container only (needs /root/reference; it never travels to
the GPU box):

    python tests/golden/make_golden.py small          # seconds
    python tests/golden/make_golden.py c1 c2          # ~1 min
    python tests/golden/make_golden.py c3             # ~45-50 min (max_m=1000)
    python tests/golden/make_golden.py c4             # ~2-2.5 h

Each config run calls the reference's own public solver
(``solve_lyapunov`` / ``solve_sylvester_two_sided``, storage="windowed") on
operators built with the reference's own generators
(``krymat.problems.gen_fd2d`` / ``laplacian1d``; the 3-D Laplacian as the
kron sum of SURVEY.md §8(d), the variable coefficient a=1+x+y by swapping
``krymat.problems._coefficients``).  The residual-check entry point is
wrapped only to record its inputs (T_m, gamma, tau) at the last check.
Outputs (``tests/golden/<name>.npz``): residual history, iteration count,
rank, truncation mass, the final projected blocks, factor sketches
X @ Omega (Omega = oracle.problems.sketch_omega), and CSR digests that pin
oracle/problems.py's builders to the reference's generators.
"""

import os
import sys
import time

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

import krymat  # noqa: E402
import krymat.problems as kp  # noqa: E402
import krymat.solvers as ks  # noqa: E402
from oracle import problems as op_  # noqa: E402


def ref_laplacian3d(n):
    lap = kp.laplacian1d(n)
    eye = sp.identity(n, format="csr")
    a = sp.kron(eye, sp.kron(eye, lap)) + sp.kron(eye, sp.kron(lap, eye))
    a = a + sp.kron(lap, sp.kron(eye, eye))
    return a.tocsr()


def ref_varcoef2d(n):
    saved = kp._coefficients
    f = lambda x, y: 1.0 + x + y  # noqa: E731
    kp._coefficients = lambda kind: (f, f)
    try:
        return kp.gen_fd2d("laplacian2d", n)
    finally:
        kp._coefficients = saved


class Recorder:
    """Wraps a residual entry point and remembers the last call's inputs."""

    def __init__(self, fn):
        self.fn = fn
        self.last = None
        self.calls = 0

    def __call__(self, *args, **kwargs):
        self.calls += 1
        self.last = (args, kwargs)
        return self.fn(*args, **kwargs)


def _blocks(t):
    return np.array(t.diag), (np.array(t.offdiag) if t.offdiag else
                              np.zeros((0, t.block_size, t.block_size)))


def run_lyapunov(name, a, c, tol, max_m, sketch_rows=None):
    rec = Recorder(ks.ctri_lyapunov)
    ks.ctri_lyapunov = rec
    try:
        op = krymat.SparseOperator(a)
        opts = krymat.SolveOptions(tol=tol, max_m=max_m, storage="windowed")
        tic = time.perf_counter()
        err = None
        try:
            sol = krymat.solve_lyapunov(op, c, opts)
        except krymat.ConvergenceError as exc:
            sol, err = None, exc
        wall = time.perf_counter() - tic
    finally:
        ks.ctri_lyapunov = rec.fn
    out = {}
    (t, gamma, tau), kw = rec.last
    out["t_diag"], out["t_off"] = _blocks(t)
    out["gamma"] = np.asarray(gamma)
    out["tau"] = np.asarray(tau)
    out["beta2"] = np.float64(kw["rhs_norm"])
    out["wall_seconds"] = np.float64(wall)
    if sol is None:
        out["history"] = np.array(err.history, dtype=float)
        out["converged"] = np.int64(0)
        out["error"] = np.array(str(err))
        return out
    out["history"] = np.array(sol.history, dtype=float)
    out["converged"] = np.int64(1)
    out["iterations"] = np.int64(sol.iterations)
    out["rank"] = np.int64(sol.rank)
    out["final_residual"] = np.float64(sol.final_residual)
    out["discarded"] = np.float64(sol.truncation_discarded)
    out["peak_basis_vectors"] = np.int64(sol.peak_basis_vectors)
    out["basis_seconds"] = np.float64(sol.basis_seconds)
    out["residual_seconds"] = np.float64(sol.residual_seconds)
    out["recovery_seconds"] = np.float64(sol.recovery_seconds)
    z = sol.z1
    n = z.shape[0]
    omega = op_.sketch_omega(n, 2)
    sk = z @ (z.T @ omega)
    out["x_norm_fro"] = np.float64(np.linalg.norm(z.T @ z))
    if sketch_rows is None:
        out["sketch"] = sk
    else:
        rows = np.sort(np.random.default_rng(7).choice(n, sketch_rows,
                                                        replace=False))
        out["sketch_rows"] = rows
        out["sketch"] = sk[rows]
    return out


def run_sylvester(name, a, b, c1, c2, tol, max_m):
    rec = Recorder(ks.ctri_sylvester)
    ks.ctri_sylvester = rec
    try:
        opa, opb = krymat.SparseOperator(a), krymat.SparseOperator(b)
        opts = krymat.SolveOptions(tol=tol, max_m=max_m, storage="windowed")
        tic = time.perf_counter()
        sol = krymat.solve_sylvester_two_sided(opa, opb, c1, c2, opts)
        wall = time.perf_counter() - tic
    finally:
        ks.ctri_sylvester = rec.fn
    out = {}
    (t, j, g1, g2, tau, iota), kw = rec.last
    out["t_diag"], out["t_off"] = _blocks(t)
    out["j_diag"], out["j_off"] = _blocks(j)
    out["gamma1"], out["gamma2"] = np.asarray(g1), np.asarray(g2)
    out["tau"], out["iota"] = np.asarray(tau), np.asarray(iota)
    out["rhs_norm"] = np.float64(kw["rhs_norm"])
    out["wall_seconds"] = np.float64(wall)
    out["history"] = np.array(sol.history, dtype=float)
    out["converged"] = np.int64(1)
    out["iterations"] = np.int64(sol.iterations)
    out["rank"] = np.int64(sol.rank)
    out["final_residual"] = np.float64(sol.final_residual)
    out["discarded"] = np.float64(sol.truncation_discarded)
    out["peak_basis_vectors"] = np.int64(sol.peak_basis_vectors)
    out["basis_seconds"] = np.float64(sol.basis_seconds)
    out["residual_seconds"] = np.float64(sol.residual_seconds)
    out["recovery_seconds"] = np.float64(sol.recovery_seconds)
    z1, z2 = sol.z1, sol.z2
    om1 = op_.sketch_omega(z1.shape[0], 2)
    om2 = op_.sketch_omega(z2.shape[0], 2)
    out["sketch_right"] = z1 @ (z2.T @ om2)   # X @ Omega2  (n1 x 2)
    out["sketch_left"] = z2 @ (z1.T @ om1)    # X^T @ Omega1 (n2 x 2)
    return out


def config(name):
    cfg = op_.build_config(name, with_matrix=False)
    if name == "c1":
        a = kp.gen_fd2d("laplacian2d", 100)
    elif name == "c2":
        a = ref_laplacian3d(50)
    elif name == "c3":
        a = ref_varcoef2d(300)
        b = ref_laplacian3d(40)
    elif name == "c4":
        a = ref_laplacian3d(200)
    elif name == "c5":
        a = kp.gen_fd2d("laplacian2d", 2000)
    digests = {"digest_a": np.array(op_.csr_digest(a))}
    if name == "c3":
        digests["digest_b"] = np.array(op_.csr_digest(b))
        out = run_sylvester(name, a, b, cfg["c1"], cfg["c2"], cfg["tol"],
                            cfg["max_m"])
    else:
        rows = 4096 if name in ("c4", "c5") else None
        out = run_lyapunov(name, a, cfg["c"], cfg["tol"], cfg["max_m"],
                           sketch_rows=rows)
    out.update(digests)
    out["tol"] = np.float64(cfg["tol"])
    out["max_m"] = np.int64(cfg["max_m"])
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print("%s: wrote %s (history rows %d, wall %.1f s)"
          % (name, path, len(out["history"]), out["wall_seconds"]), flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        if arg == "small":
            from make_golden_small import main as small_main  # noqa: E402
            small_main()
        else:
            config(arg)
