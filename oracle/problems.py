"""Problem builders for the five BASELINE configs (test / bench infrastructure).

ORACLE-SIDE CODE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  It builds the
seeded synthetic inputs of SURVEY.md §8(d) in the reference's own conventions:

* Dirichlet grids with ``n`` interior points per direction, ``h = 1/(n+1)``,
  x varying fastest, then y, then z;
* variable coefficients sampled at cell faces (midpoints), as the reference's
  five-point generator does (reference ``pkg/src/krymat/problems.py:28-67``);
* 1-D Laplacian ``tridiag(1, -2, 1)/h^2`` (``problems.py:70-75``);
* the 3-D Laplacian as ``kron(I,I,L) + kron(I,L,I) + kron(L,I,I)`` (SURVEY §8(d)
  c2; the reference has no 3-D generator, so this sum order is a convention
  the golden fixtures pin, see tests/golden/make_golden.py).

Everything returned is a scipy CSR matrix with the exact double values the
reference would produce, so a device stencil operator detected from it
(``paper_1602_05033_b200.operators``) reproduces the CSR products bit for bit.
"""

import numpy as np
import scipy.sparse as sp


def fd2d_face_matrix(n, a_fun, b_fun):
    """Five-point operator for (a u_x)_x + (b u_y)_y on the unit square.

    Restates reference ``problems.py:28-67``: coefficients at the faces
    x +- h/2 (a) and y +- h/2 (b), each divided by h^2; the diagonal is minus
    the sum east+west+north+south (in that order); east couplings are cut at
    the x boundary.  Returns CSR of order n^2.
    """
    h = 1.0 / (n + 1)
    grid = np.arange(1, n + 1) * h
    # first index = x; flatten in Fortran order so x varies fastest
    xx, yy = np.meshgrid(grid, grid, indexing="ij")
    east = a_fun(xx + 0.5 * h, yy) / h**2
    west = a_fun(xx - 0.5 * h, yy) / h**2
    north = b_fun(xx, yy + 0.5 * h) / h**2
    south = b_fun(xx, yy - 0.5 * h) / h**2

    def fl(v):
        return v.reshape(-1, order="F")

    size = n * n
    diag = -fl(east + west + north + south)
    e = fl(east)[: size - 1].copy()
    e[n - 1:: n] = 0.0
    keep = e != 0.0
    ie = np.arange(size - 1)[keep]
    nn = fl(north)[: size - n]
    inn = np.arange(size - n)
    rows = np.concatenate([np.arange(size), ie, ie + 1, inn, inn + n])
    cols = np.concatenate([np.arange(size), ie + 1, ie, inn + n, inn])
    vals = np.concatenate([diag, e[keep], e[keep], nn, nn])
    return sp.coo_matrix((vals, (rows, cols)), shape=(size, size)).tocsr()


def laplacian2d(n):
    one = lambda x, y: np.ones_like(x)  # noqa: E731
    return fd2d_face_matrix(n, one, one)


def varcoef2d(n):
    """a(x, y) = b(x, y) = 1 + x + y at the faces (config 3, operator A)."""
    f = lambda x, y: 1.0 + x + y  # noqa: E731
    return fd2d_face_matrix(n, f, f)


def laplacian1d(n):
    """Reference ``problems.py:70-75``: tridiag(1, -2, 1) / h^2, CSR."""
    h = 1.0 / (n + 1)
    main = np.full(n, -2.0 / h**2)
    off = np.full(n - 1, 1.0 / h**2)
    return sp.diags([off, main, off], (-1, 0, 1)).tocsr()


def laplacian3d(n):
    """Negated 3-D 7-point Laplacian, x fastest."""
    lap = laplacian1d(n)
    eye = sp.identity(n, format="csr")
    a = sp.kron(eye, sp.kron(eye, lap)) + sp.kron(eye, sp.kron(lap, eye))
    a = a + sp.kron(lap, sp.kron(eye, eye))
    return a.tocsr()


CONFIGS = ("c1", "c2", "c3", "c4", "c5")


def build_config(name, with_matrix=True):
    """Return a dict with the operator(s), right-hand side(s) and options.

    Keys: ``kind`` ("lyapunov" | "sylvester"), ``a`` (CSR or None when
    with_matrix=False), ``grid_a`` (grid shape, x first), ``c`` / ``c1``,
    ``c2``, ``b``, ``grid_b``, ``tol``, ``max_m``.
    """
    if name == "c1":
        out = dict(kind="lyapunov", grid_a=(100, 100), tol=1e-6, max_m=500)
        out["a"] = laplacian2d(100) if with_matrix else None
        out["c"] = np.random.default_rng(0).standard_normal((10000, 1))
        return out
    if name == "c2":
        out = dict(kind="lyapunov", grid_a=(50, 50, 50), tol=1e-8, max_m=500)
        out["a"] = laplacian3d(50) if with_matrix else None
        raw = np.random.default_rng(1).standard_normal((125000, 4))
        out["c"] = np.linalg.qr(raw)[0]
        return out
    if name == "c3":
        out = dict(kind="sylvester", grid_a=(300, 300), grid_b=(40, 40, 40),
                   tol=1e-8, max_m=1000)
        out["a"] = varcoef2d(300) if with_matrix else None
        out["b"] = laplacian3d(40) if with_matrix else None
        rng = np.random.default_rng(2)
        out["c1"] = rng.standard_normal((90000, 2))
        out["c2"] = rng.standard_normal((64000, 2))
        return out
    if name == "c4":
        out = dict(kind="lyapunov", grid_a=(200, 200, 200), tol=1e-8, max_m=600)
        out["a"] = laplacian3d(200) if with_matrix else None
        out["c"] = np.random.default_rng(3).standard_normal((8_000_000, 8))
        return out
    if name == "c5":
        out = dict(kind="lyapunov", grid_a=(2000, 2000), tol=1e-10, max_m=1500)
        out["a"] = laplacian2d(2000) if with_matrix else None
        out["c"] = np.random.default_rng(4).standard_normal((4_000_000, 4))
        return out
    raise ValueError("unknown config %r" % name)


def csr_digest(a):
    """Order-sensitive digest of a CSR matrix (indptr, indices, data bits)."""
    import hashlib

    a = sp.csr_matrix(a)
    a.sort_indices()
    h = hashlib.sha256()
    for arr in (a.indptr.astype(np.int64), a.indices.astype(np.int64),
                a.data.astype(np.float64)):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def sketch_omega(n, p, seed=99):
    """Seeded Gaussian probe block used for factor sketches X @ Omega."""
    return np.random.default_rng(seed).standard_normal((n, p))
