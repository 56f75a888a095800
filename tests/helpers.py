"""Test-input generators (seeded), written for this repo.

``lanczos_tridiagonal`` builds the projected matrix of a full
re-orthogonalisation block Lanczos run on a random negative spectrum: the
distribution of T_m the solvers see (the reference tests draw theirs the
same way, reference pkg/tests/conftest.py:58-97).
"""

import numpy as np

from oracle.krymat_oracle import BlockTri


def lanczos_tridiagonal(rng, s, m, extra=60, general=False, lo=0.1, hi=1e3):
    n = s * m + extra
    spec = -np.exp(rng.uniform(np.log(lo), np.log(hi), n))
    q0, _ = np.linalg.qr(rng.standard_normal((n, s)))
    basis, diag, off = [q0], [], []
    for j in range(m):
        w = spec[:, None] * basis[-1]
        if j:
            w = w - basis[-2] @ off[-1].T
        d = basis[-1].T @ w
        diag.append(0.5 * (d + d.T))
        w = w - basis[-1] @ d
        for b in basis:
            w = w - b @ (b.T @ w)
        q, r = np.linalg.qr(w)
        sg = np.where(np.diag(r) < 0, -1.0, 1.0)
        basis.append(q * sg)
        off.append(r * sg[:, None])
    tau = off.pop()
    if general:
        rots = [np.linalg.qr(rng.standard_normal((s, s)))[0] for _ in range(m)]
        diag = [rots[i].T @ diag[i] @ rots[i] for i in range(m)]
        off = [rots[i + 1].T @ off[i] @ rots[i] for i in range(m - 1)]
        tau = tau @ rots[-1]
    return BlockTri(s, diag, off), tau


def to_device_tri(t):
    import paper_1602_05033_b200 as kb
    return kb.BlockTridiagonal(t.ell, [np.array(d) for d in t.diag],
                               [np.array(b) for b in t.off])


class ReorderedOperator:
    """Oracle operator with a different (exact-arithmetic-equal) summation
    order: (U v + D v) + L v.  Running the oracle with it measures the
    reference algorithm's own roundoff floor (SURVEY.md §8(c) protocol)."""

    def __init__(self, a):
        import scipy.sparse as sp
        a = sp.csr_matrix(a)
        self.n = a.shape[0]
        self.lo = sp.tril(a, -1).tocsr()
        self.up = sp.triu(a, 1).tocsr()
        self.d = sp.diags(a.diagonal()).tocsr()

    def apply(self, v):
        return (self.up @ v + self.d @ v) + self.lo @ v


def noise_floor(h_ref, h_perturbed):
    """max |delta| over the common prefix of two residual histories."""
    k = min(len(h_ref), len(h_perturbed))
    a, b = np.asarray(h_ref[:k]), np.asarray(h_perturbed[:k])
    return float(np.max(np.abs(a - b))) if k else 0.0
