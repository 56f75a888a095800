"""Edge cases of the pass-1 loop and the alternative kernel paths.

* converged-then-rank-deficient: the reference stops at its converged
  iteration m* and never computes step m*+1 (solvers.py:224-240); the device
  loop runs the next steps ahead of the check, so a rank-deficient block past
  m* must not turn a converged solve into DeflationUnsupportedError.
  n = 21, s = 2 on a 1-D Laplacian: block 11 has one dimension left, the
  reference raises at step 10 (measured with the oracle).
* the opt-in fused single-pass step (KRY_FUSED_STEP=1) and the register-
  fragment apply kernel (KRY_APPLY_KERNEL=gl) against the oracle.
"""

import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1602_05033_b200 as kb
from oracle import krymat_oracle as ko
from oracle import problems as P


def lap1d(n):
    h2 = float((n + 1) ** 2)
    return sp.diags([np.full(n - 1, h2), np.full(n, -2.0 * h2), np.full(n - 1, h2)],
                    [-1, 0, 1]).tocsr()


def test_host_only_operator_is_a_type_error():
    class HostOp(kb.LinearOperator):
        n = 10
        definite = True

        def apply(self, v):
            return -v

    with pytest.raises(TypeError, match="not a device operator"):
        kb.solve_lyapunov(HostOp(), np.ones((10, 1)))
    with pytest.raises(TypeError, match="not a device operator"):
        kb.solve_sylvester_two_sided(HostOp(), HostOp(), np.ones((10, 1)), np.ones((10, 1)))


def _oracle_history(a, c, m):
    try:
        ko.solve_lyapunov(ko.SparseOperator(a), c,
                          ko.SolveOptions(tol=1e-300, max_m=m, storage="windowed"))
    except ko.NoConvergence as e:
        return np.array([r[2] for r in e.history])
    raise AssertionError("oracle converged at tol 1e-300")


@pytest.mark.gpu
@pytest.mark.parametrize("mstar", [7, 8, 9])
def test_converged_before_rank_deficient_block(mstar):
    a = lap1d(21)
    c = np.random.default_rng(11).standard_normal((21, 2))
    with pytest.raises(ko.DeflationError):
        ko.solve_lyapunov(ko.SparseOperator(a), c,
                          ko.SolveOptions(tol=1e-300, max_m=40, storage="windowed"))
    h = _oracle_history(a, c, 9)
    tol = h[mstar - 1] * (1.0 + 1e-7)
    assert tol < h[mstar - 2]
    opts = dict(tol=tol, max_m=40, storage="windowed")
    ref = ko.solve_lyapunov(ko.SparseOperator(a), c, ko.SolveOptions(**opts))
    sol = kb.solve_lyapunov(kb.SparseOperator(a), c, kb.SolveOptions(**opts))
    assert sol.iterations == ref.iterations == mstar
    x, xr = sol.z @ sol.z.T, ref.z @ ref.z.T
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


@pytest.mark.gpu
def test_rank_deficient_block_still_raises_when_not_converged():
    a = lap1d(21)
    c = np.random.default_rng(11).standard_normal((21, 2))
    with pytest.raises(kb.DeflationUnsupportedError):
        kb.solve_lyapunov(kb.SparseOperator(a), c,
                          kb.SolveOptions(tol=1e-300, max_m=40, storage="windowed"))


@pytest.mark.gpu
def test_phase_seconds_are_device_times():
    a = P.laplacian2d(60)
    c = np.random.default_rng(2).standard_normal((3600, 2))
    sol = kb.solve_lyapunov(kb.SparseOperator(a), c,
                            kb.SolveOptions(tol=1e-8, max_m=200, storage="windowed"))
    hb = np.array([r[3] for r in sol.history])
    hr = np.array([r[4] for r in sol.history])
    assert np.all(np.diff(hb) >= 0) and np.all(np.diff(hr) >= 0)
    assert hb[-1] > 0 and hr[-1] > 0
    assert sol.basis_seconds == hb[-1] and sol.residual_seconds == hr[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"KRY_FUSED_STEP": "1"}, {"KRY_APPLY_KERNEL": "gl"},
                                 {"KRY_APPLY_KERNEL": "staged"}])
@pytest.mark.parametrize("s", [2, 4])
def test_alternative_step_kernels_match_oracle(env, s, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    a = P.laplacian3d(24)
    c = np.random.default_rng(40 + s).standard_normal((a.shape[0], s))
    opts = dict(tol=1e-9, max_m=200, storage="windowed")
    ref = ko.solve_lyapunov(ko.SparseOperator(a), c, ko.SolveOptions(**opts))
    sol = kb.solve_lyapunov(kb.SparseOperator(a), c, kb.SolveOptions(**opts))
    assert sol.iterations == ref.iterations
    assert sol.rank == ref.rank
    h = np.array([r[2] for r in sol.history])
    hr = np.array([r[2] for r in ref.history])
    assert np.all(np.abs(h - hr) <= 1e-9 * hr + 1e-15), np.max(np.abs(h - hr) / hr)
    za, zb = sol.z, ref.z
    x, xr = za @ za.T, zb @ zb.T
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"KRY_FINALIZE_DENSE": "1"}, {"KRY_T_JACOBI": "1"}])
def test_finalisation_dense_fallbacks_match_oracle(env, monkeypatch):
    # the routes taken when the reduced solution is not of low rank (dense
    # block Jacobi eigh / SVD of Ytilde) and the A/B route of eigh(T_m) on
    # the dense Jacobi kernel instead of the band divide and conquer
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    a = P.laplacian3d(16)
    c = np.random.default_rng(77).standard_normal((a.shape[0], 2))
    opts = dict(tol=1e-9, max_m=200, storage="windowed")
    ref = ko.solve_lyapunov(ko.SparseOperator(a), c, ko.SolveOptions(**opts))
    sol = kb.solve_lyapunov(kb.SparseOperator(a), c, kb.SolveOptions(**opts))
    assert sol.iterations == ref.iterations and sol.rank == ref.rank
    x, xr = sol.z @ sol.z.T, ref.z @ ref.z.T
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
    # two-sided Sylvester: dense Jacobi SVD of Ytilde
    b = P.laplacian2d(20)
    c1 = np.random.default_rng(78).standard_normal((a.shape[0], 2))
    c2 = np.random.default_rng(79).standard_normal((b.shape[0], 2))
    rs = ko.solve_sylvester(ko.SparseOperator(a), ko.SparseOperator(b), c1, c2,
                                      ko.SolveOptions(**opts))
    ss = kb.solve_sylvester_two_sided(kb.SparseOperator(a), kb.SparseOperator(b), c1, c2,
                                      kb.SolveOptions(**opts))
    assert ss.iterations == rs.iterations and ss.rank == rs.rank
    x, xr = ss.z1 @ ss.z2.T, rs.z1 @ rs.z2.T
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", ["1", "3", "7"])
def test_pass2_small_chunks_match_oracle(chunk, monkeypatch):
    # pass 2 folds the regenerated blocks into Z chunk by chunk (two chunk
    # buffers, accumulation on the second stream); tiny chunks exercise the
    # buffer hand-over that the full-size config 4 only reaches at G = 64
    monkeypatch.setenv("KRY_PASS2_CHUNK", chunk)
    a = P.laplacian3d(14)
    c = np.random.default_rng(91).standard_normal((a.shape[0], 4))
    opts = dict(tol=1e-9, max_m=200, storage="windowed")
    ref = ko.solve_lyapunov(ko.SparseOperator(a), c, ko.SolveOptions(**opts))
    sol = kb.solve_lyapunov(kb.SparseOperator(a), c, kb.SolveOptions(**opts))
    assert sol.iterations == ref.iterations and sol.rank == ref.rank
    x, xr = sol.z @ sol.z.T, ref.z @ ref.z.T
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
