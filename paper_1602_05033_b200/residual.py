"""Residual norms from projected data alone (reference ``residual.py``), on
the GPU: the eigen data of the block-tridiagonal matrix come from the
incremental bordered eigen engine (csrc/eigen.cu) and the residual from the
fused Cauchy contraction  sqrt(2) ||((u u^T) o C) w||_F, C_ij = 1/(lam_i+lam_j).
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .kernels import BlockTridiagonal, _pack_blocks


@dataclass
class ResidualValue:
    """Absolute residual norm and its normalised value (reference
    ``residual.py:28-37``)."""

    res: float
    relative: float


def _sq(a, s):
    a = np.atleast_2d(np.asarray(a, dtype=float))
    out = np.zeros((s, s))
    out[: a.shape[0], : a.shape[1]] = a[:s, :s]
    return np.ascontiguousarray(out)


def ctri_lyapunov(t, gamma, tau_next, rhs_norm=None, device=0):
    """sqrt(2) ||Y Em tau^T||_F without forming Y (reference
    ``residual.py:40-59``).  ``gamma``: coefficient of C in the first block;
    ``tau_next``: coupling block to the next basis block; ``rhs_norm``
    overrides beta^2 = ||gamma||_F^2."""
    if not isinstance(t, BlockTridiagonal):
        raise TypeError("t must be a BlockTridiagonal")
    _lib.require_device()
    s, m = t.block_size, t.n_blocks
    gamma = np.atleast_2d(np.asarray(gamma, dtype=float))
    diag, sub = _pack_blocks(t)
    res = ctypes.c_double()
    _lib.check(_lib.load().kry_ctri_lyap_blocks(
        int(device), s, m, _lib.as_dptr(diag), _lib.as_dptr(sub), _lib.as_dptr(_sq(gamma, s)),
        _lib.as_dptr(_sq(tau_next, s)), ctypes.byref(res)))
    beta2 = float(rhs_norm) if rhs_norm is not None else float(np.sum(gamma * gamma))
    return ResidualValue(res.value, res.value / beta2)


def ctri_sylvester(t, j, gamma1, gamma2, tau_next, iota_next, rhs_norm=None, device=0):
    """Two-sided Sylvester residual (reference ``residual.py:62-84``)."""
    if t.block_size != j.block_size:
        raise ValueError("both projections must use the same block size")
    _lib.require_device()
    s = t.block_size
    g1 = np.atleast_2d(np.asarray(gamma1, dtype=float))
    g2 = np.atleast_2d(np.asarray(gamma2, dtype=float))
    d1, s1 = _pack_blocks(t)
    d2, s2 = _pack_blocks(j)
    res = ctypes.c_double()
    _lib.check(_lib.load().kry_ctri_sylv_blocks(
        int(device), s, t.n_blocks, _lib.as_dptr(d1), _lib.as_dptr(s1), j.n_blocks,
        _lib.as_dptr(d2), _lib.as_dptr(s2), _lib.as_dptr(_sq(g1, s)), _lib.as_dptr(_sq(g2, s)),
        _lib.as_dptr(_sq(tau_next, s)), _lib.as_dptr(_sq(iota_next, s)), ctypes.byref(res)))
    if rhs_norm is None:
        rhs_norm = np.linalg.norm(g1) * np.linalg.norm(g2)
    return ResidualValue(res.value, res.value / float(rhs_norm))
