"""Projected-matrix containers and device eigen entry points (reference
``kernels.py``).

``BlockTridiagonal`` / ``PartialSpectral`` / ``TruncatedFactor`` and the
module constants keep the reference's contracts.  ``partial_eig_blocktridiag``
runs on the GPU (csrc/eigen.cu): instead of a band reduction followed by a
tridiagonal solver (reference ``kernels.py:184-306``) the eigenvalues and the
first / last ``block_size`` eigenvector rows are built by bordered
(arrowhead) updates with Gu-Eisenstat recomputation, one scalar row at a
time.  General (non-triangular) coupling blocks are first rotated to upper
triangular form by block-diagonal Householder transforms (same spectrum; the
last rows are mapped back), so any symmetric block-tridiagonal input works.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatchError, IndefiniteMatrixError

#: Relative threshold for rank deficiency of a triangular factor.
RANK_TOL = 1e-12
#: Default tail mass allowed when truncating a low-rank factorisation.
TRUNC_EPS = 1e-12
#: Guard for eigenvalue-sum denominators, relative to the spectral radius.
DENOM_TOL = 1e-14


def guarded_denominators(left, right, tol=DENOM_TOL):
    """Pairwise sums left_i + right_j with the reference's singularity guard
    (``kernels.py:31-45``).  Host bookkeeping helper; the device kernels apply
    the same guard inside the residual contraction."""
    left = np.asarray(left, dtype=float)
    right = np.asarray(right, dtype=float)
    denom = left[:, None] + right[None, :]
    scale = max(np.max(np.abs(left)), np.max(np.abs(right)))
    if np.min(np.abs(denom)) < tol * scale:
        raise IndefiniteMatrixError(
            "eigenvalue-sum denominator is numerically singular; "
            "coefficient matrices must be definite (of one sign)")
    return denom


@dataclass
class BlockTridiagonal:
    """Symmetric block tridiagonal matrix stored as its lower block bands
    (reference ``kernels.py:48-108``)."""

    block_size: int
    diag: list
    offdiag: list

    def __post_init__(self):
        ell = self.block_size
        if len(self.offdiag) != max(len(self.diag) - 1, 0):
            raise DimensionMismatchError(
                "expected %d off-diagonal blocks, got %d"
                % (len(self.diag) - 1, len(self.offdiag)))
        for blk in list(self.diag) + list(self.offdiag):
            if np.shape(blk) != (ell, ell):
                raise DimensionMismatchError(
                    "block of shape %s does not match block size %d" % (np.shape(blk), ell))

    @property
    def n_blocks(self):
        return len(self.diag)

    @property
    def dim(self):
        return self.block_size * len(self.diag)

    def to_dense(self):
        ell, k = self.block_size, self.dim
        a = np.zeros((k, k))
        for i, blk in enumerate(self.diag):
            a[i * ell:(i + 1) * ell, i * ell:(i + 1) * ell] = blk
        for i, blk in enumerate(self.offdiag):
            a[(i + 1) * ell:(i + 2) * ell, i * ell:(i + 1) * ell] = blk
            a[i * ell:(i + 1) * ell, (i + 1) * ell:(i + 2) * ell] = np.asarray(blk).T
        return a

    @classmethod
    def from_dense(cls, a, block_size):
        a = np.asarray(a, dtype=float)
        k = a.shape[0]
        if a.shape != (k, k) or k % block_size:
            raise DimensionMismatchError(
                "cannot split %s into blocks of size %d" % (a.shape, block_size))
        m, ell = k // block_size, block_size
        diag = [a[i * ell:(i + 1) * ell, i * ell:(i + 1) * ell].copy() for i in range(m)]
        off = [a[(i + 1) * ell:(i + 2) * ell, i * ell:(i + 1) * ell].copy()
               for i in range(m - 1)]
        return cls(ell, diag, off)


@dataclass
class PartialSpectral:
    """Eigenvalues plus first / last ``block_size`` eigenvector rows."""

    eigenvalues: np.ndarray
    first_rows: np.ndarray
    last_rows: np.ndarray


@dataclass
class TruncatedFactor:
    """Tall factor of a truncated low-rank factorisation and the discarded
    Frobenius tail mass."""

    factor: np.ndarray
    discarded_mass: float

    @property
    def rank(self):
        return self.factor.shape[1]


def _pack_blocks(t):
    s, m = t.block_size, t.n_blocks
    diag = np.ascontiguousarray(np.array([np.asarray(b, dtype=float) for b in t.diag])
                                .reshape(m, s, s))
    sub = np.zeros((max(m - 1, 1), s, s))
    for i, b in enumerate(t.offdiag):
        sub[i] = np.asarray(b, dtype=float)
    return diag, np.ascontiguousarray(sub)


def partial_eig_blocktridiag(t, device=0):
    """Eigenvalues (ascending) with the first and last ``block_size`` rows of
    the eigenvector matrix (reference ``kernels.py:296-306``), on the GPU.
    Eigenvector signs are arbitrary (the residual formulas are invariant)."""
    _lib.require_device()
    s, m = t.block_size, t.n_blocks
    k = s * m
    diag, sub = _pack_blocks(t)
    lam = np.empty(k)
    first = np.empty((s, k))
    last = np.empty((s, k))
    _lib.check(_lib.load().kry_partial_eig(int(device), s, m, _lib.as_dptr(diag),
                                           _lib.as_dptr(sub), _lib.as_dptr(lam),
                                           _lib.as_dptr(first), _lib.as_dptr(last)))
    return PartialSpectral(lam, first, last)
