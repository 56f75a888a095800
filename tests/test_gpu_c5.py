"""Config 5 (2-D Laplacian 2000^2, n = 4e6, s = 4, tol 1e-10, 1500 iterations,
T_m up to k = 6000) against the REFERENCE.

A full reference solve is infeasible (~1.4 days, dominated by its O(k^2 s)
band reduction per check), so the golden is built from the reference's own
init_basis + lanczos_step for all 1500 iterations (tests/golden/
make_golden_blocks.py, ~50 min single thread): its projected blocks at every
m (tests/golden/noise/c5_blocks_csr.npz), the paper's residual formula
evaluated on them at every m with a dense eigensolver (c5_noise.npz
"surrogate", pinned to the reference's ctri_lyapunov at sampled m by
tests/test_oracle.py), the calibrated noise floor of an ensemble of runs of
the same reference algorithm (reordered SpMM sums, Cholesky-QR), and the
reference's fixed-depth factor at m = 1500 (its finalisation + its own
two_pass_recover, seeded sketch on 4096 rows).  The reference raises
ConvergenceError at 1500; so must the device, with the same history.

Also the eigen engine alone at k = 6000 on the reference's T_1500 and on
glued-Wilkinson clusters (reference tests/test_kernels.py:235-252).
"""

import ctypes
import os

import numpy as np
import pytest

import paper_1602_05033_b200 as kb
from oracle import krymat_oracle as ko
from paper_1602_05033_b200 import _lib

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(rel):
    path = os.path.join(GOLD, rel)
    if not os.path.exists(path):
        pytest.skip("golden %s not generated" % rel)
    return np.load(path)


def _dense(diag, sub, m):
    s = diag.shape[1]
    t = np.zeros((m * s, m * s))
    for i in range(m):
        t[i * s:(i + 1) * s, i * s:(i + 1) * s] = diag[i]
        if i + 1 < m:
            t[(i + 1) * s:(i + 2) * s, i * s:(i + 1) * s] = sub[i]
            t[i * s:(i + 1) * s, (i + 1) * s:(i + 2) * s] = sub[i].T
    return t


def _spectral_invariants(sp_, t, s, tol):
    """Cluster-proof checks of partial eigen data: the first / last rows of
    an orthogonal Q are orthonormal and reproduce the corner blocks of
    T = Q diag(lam) Q^T, whatever rotation a cluster's eigenvectors take."""
    lam, f, l_ = sp_.eigenvalues, sp_.first_rows, sp_.last_rows
    nt = np.linalg.norm(t, 2) if t.shape[0] <= 2000 else np.abs(lam).max()
    eye = np.eye(s)
    assert np.linalg.norm(f @ f.T - eye) <= tol
    assert np.linalg.norm(l_ @ l_.T - eye) <= tol
    assert np.linalg.norm((f * lam) @ f.T - t[:s, :s]) <= tol * nt
    assert np.linalg.norm((l_ * lam) @ l_.T - t[-s:, -s:]) <= tol * nt
    assert np.linalg.norm((f * lam) @ l_.T - t[:s, -s:]) <= tol * nt


def glued_wilkinson(w=10, blocks=4, glue=1e-14):
    d1 = np.abs(np.arange(-w, w + 1)).astype(float)
    e1 = np.ones(2 * w)
    d = np.tile(d1, blocks)
    e = np.concatenate(sum(([e1, np.array([glue])] for _ in range(blocks - 1)), []) + [e1])
    return d, e


@pytest.mark.parametrize("glue", [1e-14, 1e-10, 0.0])
def test_eigen_engine_glued_wilkinson_clusters(glue):
    d, e = glued_wilkinson(glue=glue)
    k = d.size
    t = kb.BlockTridiagonal(1, [np.array([[v]]) for v in d], [np.array([[v]]) for v in e])
    f = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    sp_ = kb.partial_eig_blocktridiag(t)
    ref = np.linalg.eigvalsh(f)
    assert np.allclose(sp_.eigenvalues, ref, atol=1e-12 * np.linalg.norm(f))
    _spectral_invariants(sp_, f, 1, 1e-12 * np.sqrt(k))
    # the cheap residual on the (shifted, definite) clustered matrix
    shift = -12.0
    ts = kb.BlockTridiagonal(1, [np.array([[v + shift]]) for v in d],
                             [np.array([[v]]) for v in e])
    ot = ko.BlockTri(1, [np.array([[v + shift]]) for v in d], [np.array([[v]]) for v in e])
    gamma, tau = np.array([[1.3]]), np.array([[0.7]])
    got = kb.ctri_lyapunov(ts, gamma, tau)
    want, _ = ko.ctri_lyapunov(ot, gamma, tau)
    # glued blocks decouple the first rows from the last ones: the residual
    # is then at roundoff level, so the bar has an absolute part relative
    # to the residual's natural scale |gamma|^2 |tau| / min |lambda|
    lam = np.linalg.eigvalsh(np.diag(d + shift) + np.diag(e, 1) + np.diag(e, -1))
    scale = 1.3 ** 2 * 0.7 / np.abs(lam).min()
    assert abs(got.res - want) <= 1e-11 * want + 1e-14 * scale


def test_eigen_engine_k6000_on_reference_projection():
    # the reference's own T_1500 of config 5 (k = 6000, s = 4)
    b = _load("noise/c5_blocks_csr.npz")
    diag, sub = b["diag_a"], b["sub_a"]
    m = diag.shape[0]
    t = kb.BlockTridiagonal(4, list(diag), list(sub[:m - 1]))
    sp_ = kb.partial_eig_blocktridiag(t)
    dense = _dense(diag, sub, m)
    import torch
    ref = torch.linalg.eigvalsh(torch.from_numpy(dense).cuda()).cpu().numpy()
    scale = np.abs(ref).max()
    assert np.all(np.diff(sp_.eigenvalues) >= 0)
    assert np.max(np.abs(sp_.eigenvalues - ref)) <= 1e-12 * scale
    _spectral_invariants(sp_, dense, 4, 1e-11)


def _c5_history():
    import bench
    cfg, op, _ = bench.build_problem("c5")
    opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
    with pytest.raises(kb.ConvergenceError) as ei:
        kb.solve_lyapunov(op, cfg["c"], opts)
    assert "no convergence to 1.0e-10 within 1500 iterations" in str(ei.value)
    return np.array([r[2] for r in ei.value.history])


def test_config5_full_history_matches_reference():
    noise = _load("c5_noise.npz")
    sur, env = noise["surrogate"], noise["env"]
    h = _c5_history()
    assert len(h) == 1500 == len(sur)
    n = min(len(h), len(env))
    floor = 2.0 * np.maximum.accumulate(env[:n])
    dev = np.abs(h[:n] - sur[:n])
    assert np.all(dev <= 1e-9 * sur[:n] + floor + 2e-16), np.max(dev / (1e-9 * sur[:n] + floor))
    assert np.all(dev[:60] <= 1e-9 * sur[:60] + 2e-16)


def test_config5_fixed_depth_factor_matches_reference():
    # the reference's finalisation + two_pass_recover at m = 1500 (the
    # recipe of reference tests/test_acceptance.py:190-215) against the
    # device's kry_finalize_lyap + kry_recover on its own T_1500
    import bench
    from oracle import problems as P
    from paper_1602_05033_b200.solvers import _Pass1
    g = _load("noise/c5_blocks_csr.npz")
    if "sketch" not in g:
        pytest.skip("c5 fixed-depth factor not generated yet")
    cfg, op, _ = bench.build_problem("c5")
    opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
    lib = _lib.load()
    p1 = _Pass1(op, np.ascontiguousarray(cfg["c"]), opts)
    try:
        hist = np.zeros((opts.max_m + 1, 5))
        nh, its, reason = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
        rel = ctypes.c_double(0.0)
        rc = lib.kry_solve_lyap_pass1(p1.ctx.ptr, opts.tol, opts.max_m, 1, _lib.as_dptr(hist),
                                      ctypes.byref(nh), ctypes.byref(its), ctypes.byref(rel),
                                      ctypes.byref(reason))
        assert rc == _lib.KRY_ERR_CONVERGENCE and reason.value == 1
        rank, disc = ctypes.c_int(0), ctypes.c_double(0.0)
        _lib.check(lib.kry_finalize_lyap(p1.ctx.ptr, 1e-12, ctypes.byref(rank), ctypes.byref(disc)))
        assert rank.value == int(g["rank"])
        assert abs(disc.value - float(g["discarded"])) <= 1e-2 * float(g["discarded"])
        z = p1.recover(rank.value)
    finally:
        p1.ctx.close()
    rows = g["sketch_rows"]
    om = P.sketch_omega(z.shape[0], 2)
    sk = (z @ (z.T @ om))[rows]
    assert np.linalg.norm(sk - g["sketch"]) <= 1e-8 * np.linalg.norm(g["sketch"])
