"""The finalisation's dense eigensolver / SVD (csrc/dense.cu, block one-sided
Jacobi on DMMA) against numpy's LAPACK: the calls the reference makes at
solvers.py:256 / :350-351 (eigh of T_m), kernels.py:316 (eigh of Ytilde) and
kernels.py:337 (svd of Ytilde)."""

import ctypes

import numpy as np
import pytest

from paper_1602_05033_b200 import _lib

pytestmark = pytest.mark.gpu


def _eigh(a, semidefinite=0):
    lib = _lib.load()
    k = a.shape[0]
    q = np.asfortranarray(a, dtype=float).copy(order="F")
    w = np.zeros(k)
    sw = ctypes.c_int(0)
    _lib.check(lib.kry_dense_eigh(0, k, q.ctypes.data_as(_lib.dptr), _lib.as_dptr(w),
                                  ctypes.byref(sw), semidefinite))
    return w, q, sw.value


def _svd(a):
    lib = _lib.load()
    m, n = a.shape
    af = np.asfortranarray(a, dtype=float)
    u = np.zeros((m, n), order="F")
    vt = np.zeros((n, n), order="F")
    sig = np.zeros(n)
    sw = ctypes.c_int(0)
    _lib.check(lib.kry_dense_svd(0, m, n, af.ctypes.data_as(_lib.dptr),
                                 u.ctypes.data_as(_lib.dptr), _lib.as_dptr(sig),
                                 vt.ctypes.data_as(_lib.dptr), ctypes.byref(sw)))
    return u, sig, vt, sw.value


def _check_eigh(a, tol=1e-13):
    w, q, sweeps = _eigh(a)
    k = a.shape[0]
    ref = np.linalg.eigvalsh(a)
    na = np.abs(ref).max()
    assert np.all(np.diff(w) >= 0)
    assert np.max(np.abs(w - ref)) <= tol * na
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= tol * np.sqrt(k)
    assert np.linalg.norm(a @ q - q * w) <= 10 * tol * na * np.sqrt(k)
    return sweeps


@pytest.mark.parametrize("k", [1, 2, 7, 16, 33, 100, 257, 600])
def test_eigh_random_symmetric(k):
    rng = np.random.default_rng(k)
    a = rng.standard_normal((k, k))
    a = a + a.T
    _check_eigh(a)


def test_eigh_negative_definite_band_with_clusters():
    # block-tridiagonal, negative definite, with repeated (ghost-like) eigenvalues
    rng = np.random.default_rng(3)
    s, m = 4, 60
    k = s * m
    t = np.zeros((k, k))
    for i in range(m):
        d = rng.standard_normal((s, s))
        t[i * s:(i + 1) * s, i * s:(i + 1) * s] = -(d @ d.T) - 4 * np.eye(s)
        if i + 1 < m:
            r = np.triu(rng.standard_normal((s, s)))
            t[(i + 1) * s:(i + 2) * s, i * s:(i + 1) * s] = r
            t[i * s:(i + 1) * s, (i + 1) * s:(i + 2) * s] = r.T
    t -= (np.linalg.eigvalsh(t).max() + 1.0) * np.eye(k)
    _check_eigh(t)
    # two decoupled copies: every eigenvalue is exactly double
    z = np.zeros_like(t)
    _check_eigh(np.block([[t, z], [z, t]]))


def test_eigh_low_rank_psd_small_eigenvalues_absolute_accuracy():
    # Ytilde-like: PSD, numerically low rank, spectrum decaying to roundoff
    rng = np.random.default_rng(5)
    k = 400
    q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    lam = np.concatenate([np.logspace(1, -15, 60), np.zeros(k - 60)])
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    w, v, _ = _eigh(a, semidefinite=1)
    ref = np.linalg.eigvalsh(a)
    assert np.max(np.abs(w - ref)) <= 1e-14 * lam.max()
    top = v[:, ::-1][:, :40]
    assert np.linalg.norm(a @ top - top * w[::-1][:40]) <= 1e-13 * lam.max()


@pytest.mark.parametrize("shape", [(1, 1), (5, 3), (40, 40), (300, 77), (513, 200), (700, 700)])
def test_svd_random(shape):
    rng = np.random.default_rng(shape[0] + shape[1])
    a = rng.standard_normal(shape)
    u, sig, vt, _ = _svd(a)
    ref = np.linalg.svd(a, compute_uv=False)
    n = shape[1]
    assert np.all(np.diff(sig) <= 0)
    assert np.max(np.abs(sig - ref)) <= 1e-13 * ref[0]
    assert np.linalg.norm(u.T @ u - np.eye(n)) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(vt @ vt.T - np.eye(n)) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm((u * sig) @ vt - a) <= 1e-12 * ref[0] * np.sqrt(n)


def test_svd_graded_low_rank_relative_accuracy():
    # Cauchy-like Ytilde of a Sylvester solve: singular values down to 1e-20
    lam = -np.logspace(0, 4, 300)
    ups = -np.logspace(0.3, 3.5, 260)
    rng = np.random.default_rng(7)
    u0 = rng.standard_normal((300, 2))
    v0 = rng.standard_normal((260, 2))
    y = -(u0 @ v0.T) / (lam[:, None] + ups[None, :])
    u, sig, vt, _ = _svd(y)
    ref = np.linalg.svd(y, compute_uv=False)
    assert np.max(np.abs(sig - ref)) <= 1e-14 * ref[0]
    assert np.linalg.norm((u * sig) @ vt - y) <= 1e-13 * ref[0]


def _band_eigh(diag, sub):
    lib = _lib.load()
    m, s = diag.shape[0], diag.shape[1]
    k = m * s
    lam = np.zeros(k)
    q = np.zeros((k, k), order="F")
    d = np.ascontiguousarray(diag, dtype=float)
    o = np.ascontiguousarray(sub if len(sub) else np.zeros((1, s, s)), dtype=float)
    _lib.check(lib.kry_band_eigh(0, s, m, _lib.as_dptr(d), _lib.as_dptr(o), _lib.as_dptr(lam),
                                 q.ctypes.data_as(_lib.dptr)))
    return lam, q


def _band_dense(diag, sub):
    m, s = diag.shape[0], diag.shape[1]
    t = np.zeros((m * s, m * s))
    for i in range(m):
        t[i * s:(i + 1) * s, i * s:(i + 1) * s] = diag[i]
        if i + 1 < m:
            t[(i + 1) * s:(i + 2) * s, i * s:(i + 1) * s] = sub[i]
            t[i * s:(i + 1) * s, (i + 1) * s:(i + 2) * s] = sub[i].T
    return t


def _check_band(diag, sub, tol=2e-13):
    lam, q = _band_eigh(diag, sub)
    t = _band_dense(diag, sub)
    k = t.shape[0]
    ref = np.linalg.eigvalsh(t)
    nt = np.abs(ref).max()
    assert np.all(np.diff(lam) >= 0)
    assert np.max(np.abs(lam - ref)) <= tol * nt
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= tol * np.sqrt(k) * 4
    assert np.linalg.norm(t @ q - q * lam) <= tol * nt * np.sqrt(k) * 4


@pytest.mark.parametrize("s,m", [(1, 1), (1, 5), (1, 33), (1, 200), (2, 3), (2, 17), (2, 150),
                                 (3, 40), (4, 9), (4, 97), (5, 30), (7, 21), (8, 4), (8, 5),
                                 (8, 60)])
def test_band_eigh_random_negative_definite(s, m):
    rng = np.random.default_rng(100 * s + m)
    diag = np.zeros((m, s, s))
    sub = np.zeros((max(m - 1, 0), s, s))
    for i in range(m):
        d = rng.standard_normal((s, s))
        diag[i] = -(d @ d.T) - 3.0 * s * np.eye(s)
    for i in range(m - 1):
        sub[i] = np.triu(rng.standard_normal((s, s)))
    _check_band(diag, sub)


def test_band_eigh_full_subdiagonal_blocks_and_decoupled_halves():
    rng = np.random.default_rng(11)
    s, m = 4, 40
    diag = np.array([-(lambda d: d @ d.T)(rng.standard_normal((s, s))) - 10 * np.eye(s)
                     for _ in range(m)])
    sub = rng.standard_normal((m - 1, s, s))
    _check_band(diag, sub)
    # exactly decoupled in the middle and repeated blocks: massive deflation
    diag2 = np.tile(diag[:1], (m, 1, 1))
    sub2 = np.tile(sub[:1], (m - 1, 1, 1))
    sub2[m // 2] = 0.0
    _check_band(diag2, sub2)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c4"])
def test_band_eigh_on_reference_projections(cfg):
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", cfg + ".npz"))
    _check_band(g["t_diag"], g["t_off"], tol=5e-13)


def test_band_eigh_large_order_deflation_path(monkeypatch):
    # orders beyond ~10^4 keep the deflation's work arrays in global memory
    monkeypatch.setenv("KRY_DC_NOSMEM", "1")
    rng = np.random.default_rng(21)
    s, m = 4, 120
    diag = np.array([-(lambda d: d @ d.T)(rng.standard_normal((s, s))) - 10 * np.eye(s)
                     for _ in range(m)])
    sub = np.array([np.triu(rng.standard_normal((s, s))) for _ in range(m - 1)])
    _check_band(diag, sub)


def test_svd_wide_matrix_has_zero_trailing_singular_values():
    rng = np.random.default_rng(12)
    a = rng.standard_normal((40, 70))
    u, sig, vt, _ = _svd(a)
    ref = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(sig[:40] - ref)) <= 1e-13 * ref[0]
    assert np.all(np.abs(sig[40:]) <= 1e-12 * ref[0])
    assert np.linalg.norm((u * sig) @ vt - a) <= 1e-12 * ref[0] * np.sqrt(70)
    assert np.linalg.norm(vt @ vt.T - np.eye(70)) <= 1e-12 * np.sqrt(70)
