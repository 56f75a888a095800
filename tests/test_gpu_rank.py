"""Rank resolution of new basis blocks (reference economy_qr + rank_deficient,
kernels.py:134-160, called by _qr_new_block, basis.py:183-189).

The reference factors every new block with Householder QR and raises
DeflationUnsupportedError only when min |R_ii| < 1e-12 ||R||_F.  The device
uses Cholesky QR; blocks too ill-conditioned for it (kappa beyond ~1e7) take
the shifted CholQR3 fallback, so the device must proceed exactly where the
reference proceeds (kappa up to ~1e12) and raise where it raises.

Cases: an ill-conditioned right-hand side C (the initial QR, basis.py:207)
and an operator whose first Lanczos residual block W = [eta q3, q4] has
condition number 1/eta (lanczos_step, basis.py:223-252).
"""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1602_05033_b200 as kb
from oracle import krymat_oracle as ko
from tests.helpers import ReorderedOperator, noise_floor

pytestmark = pytest.mark.gpu


def ill_rhs(n, s, kappa, seed):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((n, s)))
    sv = np.geomspace(1.0, 1.0 / kappa, s)
    v, _ = np.linalg.qr(rng.standard_normal((s, s)))
    return u @ np.diag(sv) @ v


def coupled_operator(n, eta, seed):
    """A = Q M Q^T negative definite with A q1 = d1 q1 + b q2 + eta q3 and
    A q2 = b q1 + d2 q2 + q4: the first residual block of V1 = [q1, q2] is
    [eta q3, q4] (condition number 1/eta)."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    m = np.diag(-np.linspace(10.0, 60.0, n))
    m[0, 1] = m[1, 0] = 0.3
    m[0, 2] = m[2, 0] = eta
    m[1, 3] = m[3, 1] = 1.0
    for i in range(2, n - 1):   # a generic chain so the later blocks are regular
        m[i, i + 1] = m[i + 1, i] = 0.5 * rng.uniform()
    a = q @ m @ q.T
    a = 0.5 * (a + a.T)
    assert np.linalg.eigvalsh(a).max() < 0
    return sp.csr_matrix(a), q[:, :2].copy()


def _both(a, c, tol=1e-10, max_m=25):
    opts = dict(tol=tol, max_m=max_m, storage="windowed")
    ref = err_ref = None
    try:
        ref = ko.solve_lyapunov(ko.SparseOperator(a), c, ko.SolveOptions(**opts))
        # the reference against itself (SURVEY.md section 8(c) protocol):
        # with a reordered SpMM, and with C moved by a backward error of the
        # size its own Householder QR commits (||E|| = 4 u ||C||; any
        # backward-stable QR, the device's shifted CholQR3 included, differs
        # from it by such an E).  Ill-conditioned blocks amplify exactly
        # this, so the history bar is 1e-9 rel + 2x the largest deviation.
        hr = [r[2] for r in ref.history]
        floors = []
        per = ko.solve_lyapunov(ReorderedOperator(a), c, ko.SolveOptions(**opts))
        floors.append(noise_floor(hr, [r[2] for r in per.history]))
        for seed in (1, 2):
            e = np.random.default_rng(seed).standard_normal(c.shape)
            ce = c + e * (4 * 2.220446049250313e-16 * np.linalg.norm(c) / np.linalg.norm(e))
            per = ko.solve_lyapunov(ko.SparseOperator(a), ce, ko.SolveOptions(**opts))
            floors.append(noise_floor(hr, [r[2] for r in per.history]))
        ref.floor = max(floors)
    except (ko.DeflationError, ko.NoConvergence) as e:
        err_ref = e
    sol = err = None
    try:
        sol = kb.solve_lyapunov(kb.SparseOperator(a), c, kb.SolveOptions(**opts))
    except (kb.DeflationUnsupportedError, kb.ConvergenceError) as e:
        err = e
    return ref, err_ref, sol, err


def _same(ref, sol):
    assert sol.iterations == ref.iterations
    h = np.array([r[2] for r in sol.history])
    hr = np.array([r[2] for r in ref.history])
    floor = max(2.0 * ref.floor, 1e-15)
    assert np.all(np.abs(h - hr) <= 1e-9 * hr + floor), (np.max(np.abs(h - hr) / hr), floor)
    x, xr = sol.z @ sol.z.T, ref.z @ ref.z.T
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


@pytest.mark.parametrize("kappa", [1e4, 1e8, 1e10, 1e11])
def test_ill_conditioned_rhs_proceeds_like_householder(kappa):
    a = sp.diags(-np.linspace(1.0, 80.0, 300)).tocsr() + sp.diags(
        [np.full(299, 0.2), np.full(299, 0.2)], [-1, 1])
    c = ill_rhs(300, 3, kappa, 5)
    ref, err_ref, sol, err = _both(sp.csr_matrix(a), c, tol=1e-8, max_m=100)
    assert err_ref is None and err is None, (err_ref, err)
    _same(ref, sol)


@pytest.mark.parametrize("kappa", [1e14, 1e16])
def test_numerically_rank_deficient_rhs_raises_like_reference(kappa):
    a = sp.diags(-np.linspace(1.0, 80.0, 300)).tocsr()
    c = ill_rhs(300, 3, kappa, 6)
    ref, err_ref, sol, err = _both(a, c)
    assert isinstance(err_ref, ko.DeflationError)
    assert isinstance(err, kb.DeflationUnsupportedError)


@pytest.mark.parametrize("eta", [1e-8, 1e-10])
def test_ill_conditioned_lanczos_block_proceeds(eta):
    a, c = coupled_operator(40, eta, 7)
    # the reference proceeds through the ill-conditioned block
    w = a @ c
    w = w - c @ (c.T @ w)
    r = np.linalg.qr(w)[1]
    assert np.min(np.abs(np.diag(r))) >= 1e-12 * np.linalg.norm(r)
    ref, err_ref, sol, err = _both(a, c, tol=1e-9, max_m=18)
    assert err_ref is None and err is None, (err_ref, err)
    _same(ref, sol)


def test_rank_deficient_lanczos_block_raises():
    a, c = coupled_operator(40, 1e-15, 8)
    ref, err_ref, sol, err = _both(a, c, tol=1e-9, max_m=18)
    assert isinstance(err_ref, ko.DeflationError)
    assert isinstance(err, kb.DeflationUnsupportedError)
