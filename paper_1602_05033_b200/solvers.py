"""Outer Galerkin drivers (reference ``solvers.py``), executed on the GPU.

Same signatures, options, result record and exceptions as the reference:
``solve_lyapunov(op, c, options)`` (``solvers.py:200-285``) and
``solve_sylvester_two_sided(op_a, op_b, c1, c2, options)`` (``:288-383``).
The host keeps only bookkeeping; every n-sized and k^2-sized operation is a
C-ABI call into libkrymat_b200.so (pass-1 loop with the cheap residual every
``check_period`` iterations, finalisation, pass-2 regeneration of the basis).

Storage: ``storage="stored"`` (the reference default) keeps every basis block
of pass 1 in device memory while it fits and assembles Z = V qy directly
(``_assemble_stored``, ``solvers.py:125-127``); ``"windowed"`` (and stored
runs that outgrow the device) regenerate the basis in a second pass, which
is bitwise deterministic (replay check), so both give the same factor.
``peak_basis_vectors`` follows the reference's accounting for the requested
mode (``basis.py:63-71``).
"""

import ctypes
from concurrent.futures import ThreadPoolExecutor
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .operators import require_device as _require_device
from .errors import (ConvergenceError, DimensionMismatchError, IndefiniteMatrixError,
                     KrymatError)

#: Largest operator order for which ``verify`` recomputes the true residual.
VERIFY_LIMIT = 20000
#: Tolerance of the pass-2 replay check (coupling blocks, relative).
REPLAY_TOL = 1e-8
#: Default truncation tail mass (reference ``kernels.py:25``).
TRUNC_EPS = 1e-12

HISTORY_COLUMNS = (
    "m",
    "space_dim",
    "relative_residual",
    "cum_basis_secs",
    "cum_residual_secs",
)


@dataclass
class SolveOptions:
    """Knobs of the outer iteration (reference ``solvers.py:49-73``)."""

    tol: float = 1e-6
    max_m: int = 500
    check_period: int = 1
    space: str = "standard"
    storage: str = "stored"
    trunc_eps: float = TRUNC_EPS
    verify: bool = False

    def __post_init__(self):
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")
        if self.check_period < 1:
            raise ValueError("check_period must be >= 1")
        if self.space not in ("standard", "extended"):
            raise ValueError("space must be 'standard' or 'extended'")
        if self.storage not in ("stored", "windowed"):
            raise ValueError("storage must be 'stored' or 'windowed'")


@dataclass
class LowRankSolution:
    """Low-rank factors with convergence history (reference ``solvers.py:76-101``)."""

    z1: np.ndarray
    z2: np.ndarray = None
    rank: int = 0
    iterations: int = 0
    space_dim: int = 0
    final_residual: float = np.inf
    history: list = field(default_factory=list)
    basis_seconds: float = 0.0
    residual_seconds: float = 0.0
    recovery_seconds: float = 0.0
    peak_basis_vectors: int = 0
    truncation_discarded: float = 0.0
    verified_residual: float = None

    @property
    def z(self):
        return self.z1


def _rows(hist, nh):
    out = []
    for r in hist[:nh]:
        out.append((int(r[0]), int(r[1]), float(r[2]), float(r[3]), float(r[4])))
    return out


def _peak(storage, steps, exhausted, s):
    pushed = 1 + steps - (1 if exhausted else 0)
    if storage == "stored":
        return max(pushed - 1, 1) * s
    return min(pushed, 3) * s


def _check_space(opts):
    if opts.space != "standard":
        raise NotImplementedError(
            "extended Krylov spaces need sparse inverse-applies, which are outside the "
            "B200 hot path (SURVEY.md §8(f) f4); use space='standard'")


def _as_rhs(op, c):
    c = np.atleast_2d(np.asarray(c, dtype=float))
    if c.ndim != 2 or c.shape[0] != op.n:
        raise DimensionMismatchError(
            "right-hand side block of shape %s does not match operator order %d"
            % (c.shape, op.n))
    if c.shape[1] > 8:
        raise DimensionMismatchError("block width %d exceeds the device limit 8" % c.shape[1])
    return np.ascontiguousarray(c)


def _nonconvergence(opts, reason, m, rel, history, both=False):
    if reason == 2:
        what = "both Krylov spaces became invariant" if both else \
            "the Krylov space became invariant"
        raise ConvergenceError(
            "%s at m=%d without meeting the tolerance (residual %.3e)" % (what, m, rel),
            history)
    raise ConvergenceError(
        "no convergence to %.1e within %d iterations (last residual %s)"
        % (opts.tol, opts.max_m, "%.3e" % rel if history else "never checked"),
        history)


# Factors of 1e9+ entries are returned in page-locked host memory from
# torch's caching host allocator: the device-to-host copy then runs at full
# PCIe rate straight into the result (no staging copy, no page faults), and a
# released result's pages are reused by the next solve instead of being
# pinned again.  Small factors (and hosts without CUDA) use plain numpy.
PINNED_MIN_BYTES = 256 << 20


def host_factor(n, rank):
    """Uninitialised C-order n x rank float64 array for a device factor."""
    if n * rank * 8 >= PINNED_MIN_BYTES:
        try:
            import torch
            if torch.cuda.is_available():
                t = torch.empty((n, rank), dtype=torch.float64, pin_memory=True)
                return t.numpy()
        except Exception:  # pragma: no cover - plain host memory below
            pass
    return np.empty((n, rank))


class _Pass1:
    """Runs init + pass 1 on one context; keeps the state for finalisation."""

    def __init__(self, op, c, opts, store=False):
        self.op = _require_device(op)
        self.c = c
        self.s = c.shape[1]
        self.ctx = op.context(self.s, opts.max_m + 2)
        # storage="stored": keep the basis on the device while it fits (the
        # factor is then assembled without regenerating the basis)
        _lib.check(_lib.load().kry_set_storage(self.ctx.ptr, 1 if store else 0))
        self.gamma = np.zeros((self.s, self.s))
        beta2 = ctypes.c_double()
        _lib.check(_lib.load().kry_init_basis(self.ctx.ptr, _lib.as_dptr(c),
                                              _lib.as_dptr(self.gamma), ctypes.byref(beta2)))
        self.beta2 = beta2.value

    def info(self):
        m, ex = ctypes.c_int(), ctypes.c_int()
        _lib.load().kry_ctx_info(self.ctx.ptr, None, None, ctypes.byref(m), ctypes.byref(ex))
        return m.value, bool(ex.value)

    def recover(self, rank):
        z = host_factor(self.op.n, rank)
        if rank > 0:
            _lib.check(_lib.load().kry_recover(self.ctx.ptr, _lib.as_dptr(z)))
        return z


def solve_lyapunov(op, c, options=None):
    """Galerkin projection solver for A X + X A + C C^T = 0 on the GPU.

    Grows the standard block Krylov space of A and C until the relative
    residual ||R_m||_F / ||C||_F^2 (cheap projected evaluation) drops below
    ``options.tol``, then returns X ~ Z Z^T (reference ``solvers.py:200-285``).
    Raises ConvergenceError (history attached) if ``max_m`` does not suffice.
    """
    opts = options if options is not None else SolveOptions()
    _check_space(opts)
    _require_device(op)
    c = _as_rhs(op, c)
    lib = _lib.load()
    tic = time.perf_counter()
    p1 = _Pass1(op, c, opts, store=opts.storage == "stored")
    t_init = time.perf_counter() - tic
    try:
        hist = np.zeros((opts.max_m + 1, 5))
        nh, its, reason = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
        rel = ctypes.c_double(np.inf)
        rc = lib.kry_solve_lyap_pass1(p1.ctx.ptr, float(opts.tol), int(opts.max_m),
                                      int(opts.check_period), _lib.as_dptr(hist),
                                      ctypes.byref(nh), ctypes.byref(its), ctypes.byref(rel),
                                      ctypes.byref(reason))
        hist[:nh.value, 3] += t_init
        history = _rows(hist, nh.value)
        if rc == _lib.KRY_ERR_CONVERGENCE:
            m, _ = p1.info()
            _nonconvergence(opts, reason.value, m, rel.value, history)
        _lib.check(rc, history)
        t_basis = history[-1][3] if history else t_init
        t_res = history[-1][4] if history else 0.0
        tic = time.perf_counter()
        rank, disc = ctypes.c_int(0), ctypes.c_double(0.0)
        _lib.check(lib.kry_finalize_lyap(p1.ctx.ptr, float(opts.trunc_eps), ctypes.byref(rank),
                                         ctypes.byref(disc)))
        z = p1.recover(rank.value)
        t_rec = time.perf_counter() - tic
        m, ex = p1.info()
        verified = None
        if opts.verify and op.n <= VERIFY_LIMIT:
            verified = true_lyapunov_residual(op, z, c) / p1.beta2
        return LowRankSolution(
            z1=z,
            rank=rank.value,
            iterations=its.value,
            space_dim=its.value * p1.s,
            final_residual=rel.value,
            history=history,
            basis_seconds=t_basis,
            residual_seconds=t_res,
            recovery_seconds=t_rec,
            # steps of the reference run = converged iterations (the device may
            # have computed one or two discarded blocks beyond)
            peak_basis_vectors=_peak(opts.storage, min(m, its.value), ex, p1.s),
            truncation_discarded=disc.value,
            verified_residual=verified,
        )
    finally:
        p1.ctx.close()


def solve_sylvester_two_sided(op_a, op_b, c1, c2, options=None):
    """Galerkin solver for A X + X B + C1 C2^T = 0 with both sides large
    (reference ``solvers.py:288-383``): two bases grown in lock step (one
    device context and CUDA stream each), residual from both projections."""
    opts = options if options is not None else SolveOptions()
    _check_space(opts)
    c1 = np.atleast_2d(np.asarray(c1, dtype=float))
    c2 = np.atleast_2d(np.asarray(c2, dtype=float))
    if c1.shape[1] != c2.shape[1]:
        raise DimensionMismatchError("C1 and C2 must have the same number of columns")
    _require_device(op_a)
    _require_device(op_b)
    c1 = _as_rhs(op_a, c1)
    c2 = _as_rhs(op_b, c2)
    lib = _lib.load()
    tic = time.perf_counter()
    pa = _Pass1(op_a, c1, opts)
    try:
        pb = _Pass1(op_b, c2, opts)
    except Exception:
        pa.ctx.close()
        raise
    t_init = time.perf_counter() - tic
    try:
        hist = np.zeros((opts.max_m + 1, 5))
        nh, its, reason = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
        rel = ctypes.c_double(np.inf)
        rc = lib.kry_solve_sylv_pass1(pa.ctx.ptr, pb.ctx.ptr, float(opts.tol), int(opts.max_m),
                                      int(opts.check_period), _lib.as_dptr(hist),
                                      ctypes.byref(nh), ctypes.byref(its), ctypes.byref(rel),
                                      ctypes.byref(reason))
        hist[:nh.value, 3] += t_init
        history = _rows(hist, nh.value)
        if rc == _lib.KRY_ERR_CONVERGENCE:
            m, _ = pa.info()
            _nonconvergence(opts, reason.value, m, rel.value, history, both=True)
        _lib.check(rc, history)
        t_basis = history[-1][3] if history else t_init
        t_res = history[-1][4] if history else 0.0
        tic = time.perf_counter()
        rank, disc = ctypes.c_int(0), ctypes.c_double(0.0)
        _lib.check(lib.kry_finalize_sylv(pa.ctx.ptr, pb.ctx.ptr, float(opts.trunc_eps),
                                         ctypes.byref(rank), ctypes.byref(disc)))
        # the two second passes are independent (own contexts and streams):
        # two host threads (the C-ABI calls release the GIL), so the latency-
        # bound steps of the two sides interleave on the GPU
        with ThreadPoolExecutor(max_workers=2) as pool:
            f2 = pool.submit(pb.recover, rank.value)
            z1 = pa.recover(rank.value)
            z2 = f2.result()
        t_rec = time.perf_counter() - tic
        ma, exa = pa.info()
        mb, exb = pb.info()
        rhs_norm = float(np.sqrt(pa.beta2) * np.sqrt(pb.beta2))
        verified = None
        if opts.verify and max(op_a.n, op_b.n) <= VERIFY_LIMIT:
            verified = true_sylvester_residual(op_a, z1, z2, c1, c2, op_b.apply) / rhs_norm
        return LowRankSolution(
            z1=z1,
            z2=z2,
            rank=rank.value,
            iterations=its.value,
            space_dim=its.value * pa.s,
            final_residual=rel.value,
            history=history,
            basis_seconds=t_basis,
            residual_seconds=t_res,
            recovery_seconds=t_rec,
            peak_basis_vectors=_peak(opts.storage, ma, exa, pa.s)
            + _peak(opts.storage, mb, exb, pb.s),
            truncation_discarded=disc.value,
            verified_residual=verified,
        )
    finally:
        pa.ctx.close()
        pb.ctx.close()


def solve_sylvester_one_sided(op_a, b, c1, c2, options=None):
    """Galerkin solver for A X + X B + C1 C2^T = 0 with B small and dense
    (reference ``solvers.py:386-481``): B is eigendecomposed once on the
    device, only A is projected (its block Krylov space of C1 grows on the
    device), the residual is ``residual_one_sided`` (``residual.py:87-104``)
    evaluated on the incrementally updated eigen data of T_m, and the right
    factor is recovered in the eigenbasis of B."""
    opts = options if options is not None else SolveOptions()
    _check_space(opts)
    b = np.asarray(b, dtype=float)
    c1 = np.atleast_2d(np.asarray(c1, dtype=float))
    c2 = np.atleast_2d(np.asarray(c2, dtype=float))
    if b.ndim != 2 or b.shape[0] != b.shape[1] or not np.array_equal(b, b.T):
        raise DimensionMismatchError("small coefficient matrix B must be symmetric")
    if c1.shape[1] != c2.shape[1]:
        raise DimensionMismatchError("C1 and C2 must have the same number of columns")
    if c2.shape[0] != b.shape[0]:
        raise DimensionMismatchError("C2 does not conform with B")
    _require_device(op_a)
    c1 = _as_rhs(op_a, c1)
    c2 = np.ascontiguousarray(c2)
    b = np.ascontiguousarray(b)
    n2, s = b.shape[0], c1.shape[1]
    lib = _lib.load()
    tic = time.perf_counter()
    ctx = op_a.context(s, opts.max_m + 2)
    try:
        ups = np.zeros(n2)
        _lib.check(lib.kry_sylv1_setup(ctx.ptr, n2, _lib.as_dptr(b), _lib.as_dptr(c2),
                                       _lib.as_dptr(ups)))
        if ups[-1] >= 0.0:
            raise IndefiniteMatrixError("B must be negative definite")
        gamma = np.zeros((s, s))
        beta2 = ctypes.c_double()
        _lib.check(lib.kry_init_basis(ctx.ptr, _lib.as_dptr(c1), _lib.as_dptr(gamma),
                                      ctypes.byref(beta2)))
        t_basis = time.perf_counter() - tic
        t_res = 0.0
        rhs_norm = float(np.sqrt(beta2.value) * np.linalg.norm(c2))
        history, converged_at, rel_v = [], None, None
        ex = ctypes.c_int(0)
        res, rel = ctypes.c_double(), ctypes.c_double()
        for it in range(1, opts.max_m + 1):
            tic = time.perf_counter()
            _lib.check(lib.kry_lanczos_step(ctx.ptr, 1, ctypes.byref(ex)))
            t_basis += time.perf_counter() - tic
            if it % opts.check_period == 0 or ex.value:
                tic = time.perf_counter()
                _lib.check(lib.kry_check_sylv1(ctx.ptr, rhs_norm, ctypes.byref(res),
                                               ctypes.byref(rel)))
                t_res += time.perf_counter() - tic
                rel_v = rel.value
                history.append((it, it * s, rel_v, t_basis, t_res))
                if rel_v <= opts.tol:
                    converged_at = it
                    break
                if ex.value:
                    raise ConvergenceError(
                        "the Krylov space became invariant at m=%d without meeting the "
                        "tolerance (residual %.3e)" % (it, rel_v), history)
        if converged_at is None:
            raise ConvergenceError(
                "no convergence to %.1e within %d iterations (last residual %s)"
                % (opts.tol, opts.max_m, "%.3e" % rel_v if rel_v is not None else "never checked"),
                history)
        tic = time.perf_counter()
        rank, disc = ctypes.c_int(0), ctypes.c_double(0.0)
        _lib.check(lib.kry_finalize_sylv1(ctx.ptr, float(opts.trunc_eps), ctypes.byref(rank),
                                          ctypes.byref(disc), None, 0))
        z2 = np.zeros((n2, rank.value))
        if rank.value > 0:
            _lib.check(lib.kry_finalize_sylv1(ctx.ptr, float(opts.trunc_eps), ctypes.byref(rank),
                                              ctypes.byref(disc), _lib.as_dptr(z2), z2.size))
        z1 = host_factor(op_a.n, rank.value)
        if rank.value > 0:
            _lib.check(lib.kry_recover(ctx.ptr, _lib.as_dptr(z1)))
        t_rec = time.perf_counter() - tic
        m, exh = ctypes.c_int(), ctypes.c_int()
        lib.kry_ctx_info(ctx.ptr, None, None, ctypes.byref(m), ctypes.byref(exh))
        verified = None
        if opts.verify and op_a.n <= VERIFY_LIMIT:
            verified = true_sylvester_residual(op_a, z1, z2, c1, c2, lambda v: b @ v) / rhs_norm
        return LowRankSolution(
            z1=z1,
            z2=z2,
            rank=rank.value,
            iterations=converged_at,
            space_dim=converged_at * s,
            final_residual=rel_v,
            history=history,
            basis_seconds=t_basis,
            residual_seconds=t_res,
            recovery_seconds=t_rec,
            peak_basis_vectors=_peak(opts.storage, min(m.value, converged_at), bool(exh.value), s),
            truncation_discarded=disc.value,
            verified_residual=verified,
        )
    finally:
        ctx.close()


def true_lyapunov_residual(op, z, c):
    """||A Z Z^T + Z Z^T A + C C^T||_F from small Gram matrices, on the device
    (reference ``solvers.py:104-115``)."""
    _require_device(op)
    z = np.ascontiguousarray(np.atleast_2d(np.asarray(z, dtype=float)))
    c = np.ascontiguousarray(np.atleast_2d(np.asarray(c, dtype=float)))
    ctx = op.context(c.shape[1], 1)
    try:
        res = ctypes.c_double()
        _lib.check(_lib.load().kry_true_lyap_residual(ctx.ptr, _lib.as_dptr(z), z.shape[1],
                                                      _lib.as_dptr(c), ctypes.byref(res)))
        return res.value
    finally:
        ctx.close()


def true_sylvester_residual(op_a, z1, z2, c1, c2, apply_b):
    """||A Z1 Z2^T + Z1 Z2^T B + C1 C2^T||_F via small Gram matrices
    (reference ``solvers.py:118-122``; the Gram products are tiny)."""
    az1 = op_a.apply(z1)
    bz2 = apply_b(z2)
    u = np.hstack([az1, z1, c1])
    w = np.hstack([z2, bz2, c2])
    val = np.sum((u.T @ u) * (w.T @ w))
    return float(np.sqrt(max(val, 0.0)))
