"""Step-level block Krylov API (reference ``basis.py``), backed by the device.

``init_basis`` / ``lanczos_step`` / ``BasisWindow`` / ``ProjectionState``
keep the reference contracts (standard space) so code written against
``krymat.basis`` runs unchanged; each step is one C-ABI call
(``kry_lanczos_step``: fused apply-Gram, MGS-twice/Cholesky-QR coefficient
solve, combine) and the eigen data of T_m are updated on the device, so
``ctri_lyapunov(state.projected_matrix(), ...)`` and ``state.check_lyapunov``
need no host work.  Basis blocks are copied to the host only when asked for
(``window.last_two()``) or, in ``stored`` mode, after every step (the
reference keeps every block in memory in that mode).
"""

import ctypes

import numpy as np

from . import _lib
from .errors import DeflationUnsupportedError, DimensionMismatchError
from .kernels import BlockTridiagonal
from .operators import require_device

#: Relative size of a residual block treated as zero (reference basis.py:30).
ZERO_BLOCK_TOL = 1e-13


class BasisWindow:
    """Three-block window over the device basis (reference basis.py:33-83)."""

    def __init__(self, mode, ctx, s, n):
        if mode not in ("windowed", "stored"):
            raise ValueError("storage mode must be 'windowed' or 'stored'")
        self.mode = mode
        self.extended = False
        self._ctx = ctx
        self._s = s
        self._n = n
        self.stored = [] if mode == "stored" else None
        self.second_halves = None
        self.generated = 0
        self.peak_vectors = 0

    def _pushed(self, exhausted):
        if not exhausted:
            self.generated += 1
            if self.stored is not None:
                _, cur = self.last_two()
                self.stored.append(cur)
        if self.stored is not None:
            held = max(self.generated - 1, 1) * self._s
        else:
            held = min(self.generated, 3) * self._s
        self.peak_vectors = max(self.peak_vectors, held)

    def last_two(self):
        """The two most recent (orthonormal) blocks, oldest first."""
        older = np.empty((self._n, self._s))
        cur = np.empty((self._n, self._s))
        have = ctypes.c_int(0)
        _lib.check(_lib.load().kry_get_window(self._ctx.ptr, _lib.as_dptr(older),
                                              _lib.as_dptr(cur), ctypes.byref(have)))
        return (older if have.value else None), cur

    def basis_blocks(self, m):
        if self.stored is None:
            raise DimensionMismatchError("basis blocks were not stored")
        return self.stored[:m]


class ProjectionState:
    """Projection coefficients held on the device (reference basis.py:86-161)."""

    def __init__(self, ctx, s, gamma, rhs, beta2):
        self.space = "standard"
        self.s = s
        self.ell = s
        self.gamma = gamma
        self.rhs = rhs
        self.beta2 = beta2
        self.m = 1
        self.exhausted = False
        self._ctx = ctx
        self._cache = None

    @property
    def n_t_blocks(self):
        return self.m - 1

    def _fetch(self):
        if self._cache is not None and self._cache[0] == self.m:
            return self._cache[1]
        k = self.n_t_blocks
        s = self.s
        m = ctypes.c_int(0)
        raw = np.zeros((max(k, 1), s, s))
        sym = np.zeros_like(raw)
        off = np.zeros_like(raw)
        sub = np.zeros_like(raw)
        if k:
            _lib.check(_lib.load().kry_get_projection(self._ctx.ptr, ctypes.byref(m),
                                                      _lib.as_dptr(raw), _lib.as_dptr(sym),
                                                      _lib.as_dptr(off), _lib.as_dptr(sub)))
        blocks = dict(diag_raw=list(raw[:k]), diag_sym=list(sym[:k]),
                      off_mgs=[None] + list(off[1:k]) if k else [], sub=list(sub[:k]))
        self._cache = (self.m, blocks)
        return blocks

    @property
    def diag_raw(self):
        return self._fetch()["diag_raw"]

    @property
    def off_mgs(self):
        return self._fetch()["off_mgs"]

    @property
    def sub(self):
        return self._fetch()["sub"]

    def projected_matrix(self):
        k = self.n_t_blocks
        if k < 1:
            raise DimensionMismatchError("no completed projection blocks yet")
        b = self._fetch()
        return BlockTridiagonal(self.s, list(b["diag_sym"]), list(b["sub"][:k - 1]))

    def coupling_block(self):
        return self._fetch()["sub"][self.n_t_blocks - 1]

    def coupling_upper(self):
        return self.coupling_block()

    def check_lyapunov(self, rhs_norm=None):
        """cTri residual of the current projection from the device eigen data."""
        res, rel = ctypes.c_double(), ctypes.c_double()
        b2 = float(rhs_norm) if rhs_norm is not None else self.beta2
        _lib.check(_lib.load().kry_check_lyap(self._ctx.ptr, b2, ctypes.byref(res),
                                              ctypes.byref(rel)))
        return res.value, rel.value


def init_basis(op, c, space="standard", storage="stored", fact=None, max_m=1000):
    """First block V1 = QR(C) on the device (reference basis.py:192-220).
    ``max_m`` bounds the number of steps the device context can hold."""
    if space != "standard":
        raise NotImplementedError("extended Krylov spaces are outside the B200 hot path")
    require_device(op)
    c = np.ascontiguousarray(np.asarray(c, dtype=float))
    if c.ndim != 2 or c.shape[0] != op.n:
        raise DimensionMismatchError(
            "right-hand side block of shape %s does not match operator order %d"
            % (c.shape, op.n))
    s = c.shape[1]
    ctx = op.context(s, max_m + 2)
    gamma = np.zeros((s, s))
    beta2 = ctypes.c_double()
    _lib.check(_lib.load().kry_init_basis(ctx.ptr, _lib.as_dptr(c), _lib.as_dptr(gamma),
                                          ctypes.byref(beta2)))
    window = BasisWindow(storage, ctx, s, op.n)
    state = ProjectionState(ctx, s, gamma, c, beta2.value)
    window._pushed(False)
    return window, state


def lanczos_step(op, window, state, on_zero_residual="raise"):
    """One block-Lanczos step with MGS performed twice and QR (reference
    basis.py:223-252); ``on_zero_residual="finalize"`` appends a zero coupling
    block and marks the state exhausted instead of raising."""
    if state.exhausted:
        raise DeflationUnsupportedError("the Krylov space is already invariant")
    ex = ctypes.c_int(0)
    _lib.check(_lib.load().kry_lanczos_step(state._ctx.ptr,
                                            1 if on_zero_residual == "finalize" else 0,
                                            ctypes.byref(ex)))
    state.m += 1
    state._cache = None
    if ex.value:
        state.exhausted = True
    window._pushed(bool(ex.value))
    return window, state


def two_pass_recover(op, state, qy, window=None):
    """Second Lanczos pass (reference solvers.py:130-169): regenerate the
    basis on the device and accumulate Z = sum_i V_i qy_i."""
    qy = np.ascontiguousarray(np.asarray(qy, dtype=float))
    m = state.n_t_blocks
    if qy.shape[0] != m * state.s:
        raise DimensionMismatchError("qy has %d rows, expected %d" % (qy.shape[0], m * state.s))
    t = qy.shape[1]
    lib = _lib.load()
    _lib.check(lib.kry_set_qy(state._ctx.ptr, m, t, _lib.as_dptr(qy)))
    z = np.empty((op.n, t))
    if t:
        _lib.check(lib.kry_recover(state._ctx.ptr, _lib.as_dptr(z)))
    return z
