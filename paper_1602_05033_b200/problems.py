"""Deterministic generators for the benchmark operators and the BASELINE
workloads (the package-side counterpart of the reference's
``pkg/src/krymat/problems.py``; bench.py and the tools use this module, the
oracle keeps its own independent restatement for the checks).

Conventions (reference ``problems.py:1-7``): zero Dirichlet conditions, ``n``
interior points per direction, ``h = 1/(n+1)``, x varying fastest, then y,
then z; variable coefficients evaluated at the cell faces so the matrices
are exactly symmetric and negative definite.

Operators come in two forms with the same double values:

* ``gen_fd2d`` / ``laplacian1d`` / ``laplacian3d``: scipy CSR, exactly the
  matrices the reference builds (``problems.py:28-75``; the 3-D Laplacian as
  ``kron(I,I,L) + kron(I,L,I) + kron(L,I,I)``);
* ``stencil_operator``: the device stencil description of a constant
  Laplacian, without materialising the CSR (8M-point grids), with the
  diagonal constant summed in the same order as the CSR construction.

``workload(name)`` returns the seeded inputs of the five BASELINE configs
(SURVEY.md §8(d)); tests/test_workloads.py pins the CSR digests to the
reference's own generators (tests/golden/*.npz).
"""

import numpy as np
import scipy.sparse as sp

FD2D_KINDS = ("fd2d-exp", "fd2d-trig", "laplacian2d", "varcoef2d")


def _coefficients(kind):
    """Face coefficient functions a(x, y), b(x, y) (reference problems.py:18-25;
    ``varcoef2d`` is config 3's a = b = 1 + x + y)."""
    if kind == "fd2d-exp":
        return (lambda x, y: np.exp(-x * y)), (lambda x, y: np.exp(x * y))
    if kind == "fd2d-trig":
        return (lambda x, y: np.sin(x * y)), (lambda x, y: np.cos(x * y))
    if kind == "laplacian2d":
        return (lambda x, y: np.ones_like(x)), (lambda x, y: np.ones_like(x))
    if kind == "varcoef2d":
        return (lambda x, y: 1.0 + x + y), (lambda x, y: 1.0 + x + y)
    raise ValueError("unknown 2-D problem kind %r" % kind)


def gen_fd2d(kind, n):
    """Five-point operator for (a u_x)_x + (b u_y)_y on the unit square, CSR of
    order n^2 (reference problems.py:28-67): face values / h^2, diagonal =
    -(east + west + north + south) in that order, east couplings cut at the
    x boundary, entries assembled as COO (diag, east pairs, north pairs)."""
    a_fun, b_fun = _coefficients(kind)
    h = 1.0 / (n + 1)
    pts = np.arange(1, n + 1) * h
    x, y = np.meshgrid(pts, pts, indexing="ij")
    east = a_fun(x + 0.5 * h, y) / h**2
    west = a_fun(x - 0.5 * h, y) / h**2
    north = b_fun(x, y + 0.5 * h) / h**2
    south = b_fun(x, y - 0.5 * h) / h**2
    col = lambda v: v.reshape(-1, order="F")  # noqa: E731  (x fastest)
    size = n * n
    main = -col(east + west + north + south)
    ev = col(east)[: size - 1].copy()
    ev[n - 1:: n] = 0.0
    ke = np.flatnonzero(ev != 0.0)
    nv = col(north)[: size - n]
    kn = np.arange(size - n)
    r = np.concatenate([np.arange(size), ke, ke + 1, kn, kn + n])
    c = np.concatenate([np.arange(size), ke + 1, ke, kn + n, kn])
    v = np.concatenate([main, ev[ke], ev[ke], nv, nv])
    return sp.coo_matrix((v, (r, c)), shape=(size, size)).tocsr()


def laplacian1d(n):
    """tridiag(1, -2, 1) / h^2 (reference problems.py:70-75)."""
    h = 1.0 / (n + 1)
    return sp.diags([np.full(n - 1, 1.0 / h**2), np.full(n, -2.0 / h**2),
                     np.full(n - 1, 1.0 / h**2)], (-1, 0, 1)).tocsr()


def laplacian3d(n):
    """Negated 3-D 7-point Laplacian kron(I,I,L) + kron(I,L,I) + kron(L,I,I)."""
    lap = laplacian1d(n)
    eye = sp.identity(n, format="csr")
    out = sp.kron(eye, sp.kron(eye, lap)) + sp.kron(eye, sp.kron(lap, eye))
    return (out + sp.kron(lap, sp.kron(eye, eye))).tocsr()


def laplacian_constants(dims, n):
    """(diagonal, off-diagonal) doubles of the constant Laplacians, summed in
    the CSR construction order: 3-D diag = ((d + d) + d) with d = -2/h^2 (the
    kron sum); 2-D diag = -(((c + c) + c) + c) with c = 1/h^2 (face sum)."""
    h = 1.0 / (n + 1)
    if dims == 3:
        d = -2.0 / h**2
        return (d + d) + d, 1.0 / h**2
    c = 1.0 / h**2
    return -(((c + c) + c) + c), c


def stencil_operator(grid, slab=None, comm=None):
    """Device stencil operator of the constant Laplacian on ``grid`` (x first;
    2 or 3 entries), optionally restricted to the z-slab [z0, z1) of a
    sharded run.  A 2-D grid is presented as (nx, 1, ny) so the slab axis is y."""
    from .operators import StencilOperator

    grid = tuple(grid)
    if len(grid) == 3:
        cd, co = laplacian_constants(3, grid[0])
        return StencilOperator(grid, cd, co, co, co, slab=slab, comm=comm)
    cd, co = laplacian_constants(2, grid[0])
    return StencilOperator((grid[0], 1, grid[1]), cd, co, 0.0, co, slab=slab, comm=comm)


def gen_fd3d_split(n):
    """(A, B) of the 3-D operator (e^{-xy} u_x)_x + (e^{xy} u_y)_y + 10 u_zz
    split as a Sylvester pair: A the 2-D part (n^2), B = 10 laplacian1d(n)
    (reference problems.py:78-85)."""
    return gen_fd2d("fd2d-exp", n), (10.0 * laplacian1d(n)).tocsr()


def gen_operator(kind, n):
    """Matrix (or pair) of a named problem kind (reference problems.py:101-109)."""
    if kind in ("fd2d-exp", "fd2d-trig", "laplacian2d"):
        return gen_fd2d(kind, n)
    if kind == "laplacian1d":
        return laplacian1d(n)
    if kind == "fd3d-split":
        return gen_fd3d_split(n)
    raise ValueError("unknown problem kind %r" % kind)


def gen_rhs(n, s, seed, normalize=True):
    """Right-hand side block, entries uniform in (0, 1) from PCG64(seed),
    scaled to unit Frobenius norm (reference problems.py:88-98)."""
    c = np.random.default_rng(seed).random((n, s))
    if normalize:
        c /= np.linalg.norm(c)
    return c


WORKLOADS = ("c1", "c2", "c3", "c4", "c5")

DESCRIPTIONS = {
    "c1": "Lyapunov L2D 100^2 (n=10,000), s=1, tol 1e-6",
    "c2": "Lyapunov L3D 50^3 (n=125,000), s=4 QR'd C, tol 1e-8",
    "c3": "Sylvester var-coef 2D 300^2 x L3D 40^3, s=2, tol 1e-8",
    "c4": "Lyapunov L3D 200^3 (n=8,000,000), s=8, tol 1e-8, maxit 600",
    "c5": "Lyapunov L2D 2000^2 (n=4,000,000), s=4, tol 1e-10, 1500 its",
}


def workload(name, with_matrix=True):
    """Seeded inputs of a BASELINE config.

    Returns a dict: ``kind`` ("lyapunov" | "sylvester"), ``grid_a`` (x first),
    ``a`` (CSR, or None with ``with_matrix=False``), ``c`` (Lyapunov) or
    ``c1``/``b``/``grid_b``/``c2`` (Sylvester), ``tol``, ``max_m``.
    """
    if name == "c1":
        out = dict(kind="lyapunov", grid_a=(100, 100), tol=1e-6, max_m=500)
        out["a"] = gen_fd2d("laplacian2d", 100) if with_matrix else None
        out["c"] = np.random.default_rng(0).standard_normal((10000, 1))
    elif name == "c2":
        out = dict(kind="lyapunov", grid_a=(50, 50, 50), tol=1e-8, max_m=500)
        out["a"] = laplacian3d(50) if with_matrix else None
        out["c"] = np.linalg.qr(np.random.default_rng(1).standard_normal((125000, 4)))[0]
    elif name == "c3":
        out = dict(kind="sylvester", grid_a=(300, 300), grid_b=(40, 40, 40),
                   tol=1e-8, max_m=1000)
        out["a"] = gen_fd2d("varcoef2d", 300) if with_matrix else None
        out["b"] = laplacian3d(40) if with_matrix else None
        rng = np.random.default_rng(2)
        out["c1"] = rng.standard_normal((90000, 2))
        out["c2"] = rng.standard_normal((64000, 2))
    elif name == "c4":
        out = dict(kind="lyapunov", grid_a=(200, 200, 200), tol=1e-8, max_m=600)
        out["a"] = laplacian3d(200) if with_matrix else None
        out["c"] = np.random.default_rng(3).standard_normal((8_000_000, 8))
    elif name == "c5":
        out = dict(kind="lyapunov", grid_a=(2000, 2000), tol=1e-10, max_m=1500)
        out["a"] = gen_fd2d("laplacian2d", 2000) if with_matrix else None
        out["c"] = np.random.default_rng(4).standard_normal((4_000_000, 4))
    else:
        raise ValueError("unknown workload %r" % name)
    return out


def sketch_omega(n, p, seed=99):
    """Seeded Gaussian probe block for factor sketches X @ Omega."""
    return np.random.default_rng(seed).standard_normal((n, p))
