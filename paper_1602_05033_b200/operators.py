"""Operators on the device (reference ``operators.py``).

``SparseOperator(a)`` keeps the reference contract (exact symmetry check with
the same message, ``n``, ``definite``, ``apply``) but its products run on the
GPU.  At construction the CSR matrix is inspected: when its pattern is the
3/5/7-point stencil of a Dirichlet grid (x fastest), the operator is stored
as a stencil (constant coefficients: 4 doubles; variable: 4 doubles per
point) instead of CSR, which is what makes the fused SpMM HBM-efficient.
Row sums are accumulated on the device in CSR column order without FMA
contraction, so ``apply`` equals scipy's ``csr_matvecs`` (reference
``operators.py:101``) bit for bit.
"""

import ctypes

import numpy as np
import scipy.sparse as sp

from . import _lib
from .errors import AsymmetricMatrixError, DimensionMismatchError


def validate_symmetric(a):
    """Return ``a`` as CSR after checking exact symmetry (reference
    ``operators.py:24-42``: same error classes and message)."""
    a = sp.csr_matrix(a)
    if a.shape[0] != a.shape[1]:
        raise DimensionMismatchError("matrix is %dx%d, not square" % a.shape)
    diff = (a - a.T).tocoo()
    bad = diff.data != 0.0
    if bad.any():
        i = int(diff.row[bad][0])
        j = int(diff.col[bad][0])
        raise AsymmetricMatrixError(
            "matrix is not symmetric: entry (%d, %d) = %.17g but (%d, %d) = %.17g"
            % (i, j, a[i, j], j, i, a[j, i]))
    return a


class LinearOperator:
    """Symmetric operator interface (reference ``operators.py:65-79``)."""

    n = 0
    definite = False

    def apply(self, v):
        raise NotImplementedError

    @property
    def can_solve(self):
        return False

    def solve(self, v):
        raise NotImplementedError("operator has no inverse-apply capability")


def require_device(op):
    """The device solvers need an operator that lives on the GPU
    (SparseOperator / StencilOperator).  A host-only LinearOperator (the
    reference's plug-in protocol, operators.py:65-79, whose ``apply`` is
    Python code) cannot feed the device recurrence: it is rejected with a
    typed error instead of failing later on a missing attribute."""
    if not callable(getattr(op, "context", None)):
        raise TypeError(
            "%s is not a device operator: the B200 solvers need a SparseOperator "
            "(or StencilOperator) whose products run on the GPU; wrap the matrix "
            "with paper_1602_05033_b200.SparseOperator(a)" % type(op).__name__)
    return op


def _grid_from_offsets(n, pos):
    """(nx, nxy) such that the positive offsets are a subset of {1, nx, nxy}."""
    p = [int(v) for v in pos]
    if len(p) == 0:
        return n, n
    if len(p) == 1:
        return (n, n) if p[0] == 1 else (p[0], n)
    if len(p) == 2:
        return (p[1], n) if p[0] == 1 else (p[0], p[1])
    if len(p) == 3 and p[0] == 1:
        return p[1], p[2]
    return None


def detect_stencil(a):
    """Recognise a Dirichlet-grid 3/5/7-point pattern in a CSR matrix.

    Returns a dict (grid, constant / per-point coefficients) or None.
    Coefficients: diag[i] = A[i,i], cx[i] = A[i,i+1], cy[i] = A[i,i+nx],
    cz[i] = A[i,i+nx*ny] (zero where the grid has no such neighbour).
    """
    n = a.shape[0]
    if n == 0 or not a.has_canonical_format:
        return None
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.indptr))
    off = a.indices.astype(np.int64) - rows
    upper = off > 0
    dims = _grid_from_offsets(n, np.unique(off[upper]))
    if dims is None:
        return None
    nx, nxy = dims
    if nx < 1 or nxy % nx or n % nxy:
        return None
    ny, nz = nxy // nx, n // nxy
    r_up, o_up, v_up = rows[upper], off[upper], a.data[upper]
    x, y, z = r_up % nx, (r_up // nx) % ny, r_up // nxy
    is_x = o_up == 1
    is_y = (o_up == nx) & (nx < n) & ~is_x
    is_z = (o_up == nxy) & (nxy < n) & ~is_x & ~is_y
    if not np.all(is_x | is_y | is_z):
        return None
    inside = (is_x & (x < nx - 1)) | (is_y & (y < ny - 1)) | (is_z & (z < nz - 1))
    # a link that leaves the grid must be absent or an explicit zero
    if not np.all(inside | (v_up == 0.0)):
        return None
    diag = np.zeros(n)
    dmask = off == 0
    diag[rows[dmask]] = a.data[dmask]
    arrays = {}
    for name, sel in (("cx", is_x), ("cy", is_y), ("cz", is_z)):
        arr = np.zeros(n)
        m = sel & inside
        arr[r_up[m]] = v_up[m]
        arrays[name] = arr
    idx = np.arange(n)
    masks = {"cx": idx % nx < nx - 1, "cy": (idx // nx) % ny < ny - 1,
             "cz": idx // nxy < nz - 1}
    constant = bool(np.all(diag == diag[0]))
    const = {}
    for name in ("cx", "cy", "cz"):
        v = arrays[name][masks[name]]
        if v.size == 0:
            const[name] = 0.0
            continue
        if not np.all(v == v[0]) or v[0] == 0.0:
            constant = False
        const[name] = float(v[0])
    return dict(grid=(nx, ny, nz), constant=constant, c_diag=float(diag[0]),
                c_x=const["cx"], c_y=const["cy"], c_z=const["cz"], diag=diag,
                cx=arrays["cx"], cy=arrays["cy"], cz=arrays["cz"])


class _DeviceOperator(LinearOperator):
    """Common device plumbing: builds the C operator description."""

    device = 0

    def _desc(self):
        raise NotImplementedError

    def context(self, s, max_m):
        """A fresh device context for a solve with block width s."""
        _lib.require_device()
        lib = _lib.load()
        desc = self._desc()
        ctx = ctypes.c_void_p()
        _lib.check(lib.kry_ctx_create(ctypes.byref(ctx), int(self.device), ctypes.byref(desc),
                                      int(s), int(max_m)))
        context = Context(ctx, self, s, max_m)
        comm = getattr(self, "comm", None)
        if comm is not None and comm.nranks > 1:
            comm.attach(context)
        return context

    def apply(self, v):
        v = np.asarray(v, dtype=float)
        if v.shape[0] != self.n:
            raise DimensionMismatchError(
                "operator is order %d, block has %d rows" % (self.n, v.shape[0]))
        squeeze = v.ndim == 1
        vb = np.ascontiguousarray(v.reshape(self.n, -1))
        out = np.empty_like(vb)
        ctx = self.context(1, 1)
        try:
            _lib.check(_lib.load().kry_apply(ctx.ptr, _lib.as_dptr(vb), _lib.as_dptr(out),
                                             int(vb.shape[1])))
        finally:
            ctx.close()
        return out[:, 0] if squeeze else out.reshape(v.shape)


class StencilOperator(_DeviceOperator):
    """Dirichlet-grid stencil operator (x fastest), constant or per point."""

    def __init__(self, grid, c_diag=None, c_x=0.0, c_y=0.0, c_z=0.0, diag=None, cx=None,
                 cy=None, cz=None, definite=True, slab=None, comm=None):
        g = tuple(int(v) for v in grid) + (1,) * (3 - len(grid))
        self.grid = g
        self.n_global = g[0] * g[1] * g[2]
        self.definite = definite
        # slab sharding (parallel.py): this rank owns planes [z0, z1) of the
        # slowest axis; n is then the local row count
        self.comm = comm
        self.slab = tuple(slab) if slab is not None else (0, g[2])
        self.n = g[0] * g[1] * (self.slab[1] - self.slab[0])
        self.variable = diag is not None
        if self.variable:
            self._arrays = [np.ascontiguousarray(x, dtype=float) for x in (diag, cx, cy, cz)]
            for arr in self._arrays:
                if arr.shape != (self.n_global,):
                    raise DimensionMismatchError("coefficient array has the wrong length")
        else:
            self._arrays = None
        self.c = (float(c_diag), float(c_x), float(c_y), float(c_z)) if c_diag is not None \
            else (0.0, 0.0, 0.0, 0.0)

    def _desc(self):
        d = _lib.OperatorDesc()
        d.kind = _lib.KRY_OP_STENCIL
        d.variable = 1 if self.variable else 0
        d.n = self.n_global
        d.nx, d.ny, d.nz = self.grid
        d.c_diag, d.c_x, d.c_y, d.c_z = self.c
        if self.variable:
            d.diag, d.cx, d.cy, d.cz = (_lib.as_dptr(x) for x in self._arrays)
        d.z_begin, d.z_end = self.slab
        return d


class SparseOperator(_DeviceOperator):
    """Operator backed by a sparse symmetric matrix (reference
    ``operators.py:82-113``), executed on the GPU.  Inverse-applies (extended
    Krylov) are out of the B200 scope."""

    def __init__(self, a, definite=True):
        self.matrix = validate_symmetric(a)
        self.matrix.sort_indices()
        self.n = self.matrix.shape[0]
        self.definite = definite
        st = detect_stencil(self.matrix)
        self.stencil = None
        if st is not None:
            if st["constant"]:
                self.stencil = StencilOperator(st["grid"], st["c_diag"], st["c_x"], st["c_y"],
                                               st["c_z"], definite=definite)
            else:
                self.stencil = StencilOperator(st["grid"], diag=st["diag"], cx=st["cx"],
                                               cy=st["cy"], cz=st["cz"], definite=definite)
        else:
            self._indptr = np.ascontiguousarray(self.matrix.indptr, dtype=np.int64)
            self._indices = np.ascontiguousarray(self.matrix.indices, dtype=np.int32)
            self._data = np.ascontiguousarray(self.matrix.data, dtype=np.float64)

    @property
    def kind(self):
        if self.stencil is None:
            return "csr"
        return "stencil-variable" if self.stencil.variable else "stencil-constant"

    def _desc(self):
        if self.stencil is not None:
            return self.stencil._desc()
        d = _lib.OperatorDesc()
        d.kind = _lib.KRY_OP_CSR
        d.n = self.n
        d.nnz = int(self._data.size)
        d.indptr = self._indptr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        d.indices = self._indices.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        d.values = _lib.as_dptr(self._data)
        d.nx, d.ny, d.nz = self.n, 1, 1
        return d

    @property
    def can_solve(self):
        return False


class Context:
    """Owns one kry_ctx (device state of one Krylov basis)."""

    def __init__(self, ptr, op, s, max_m):
        self.ptr = ptr
        self.op = op
        self.s = s
        self.max_m = max_m

    def close(self):
        if self.ptr is not None and self.ptr.value:
            _lib.load().kry_ctx_destroy(self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def block_apply(op, v):
    """Apply an operator to a block of vectors (reference ``operators.py:166``)."""
    return op.apply(v)
