"""GPU: the step-level API (reference basis.py / two_pass_recover) through the
C-ABI, mirroring the reference's basis tests (pkg/tests/test_basis.py) with
the device kernels swapped in."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1602_05033_b200 as kb
from oracle import krymat_oracle as ko
from oracle import problems as P

pytestmark = pytest.mark.gpu


def _diag_op(vals):
    return kb.SparseOperator(sp.diags(vals).tocsr())


def _full_basis(window, m):
    return np.concatenate(window.basis_blocks(m), axis=1)


def test_canonical_vector():
    c = np.zeros((5, 1))
    c[0] = 1.0
    window, state = kb.init_basis(_diag_op([-1.0, -2, -3, -4, -5]), c)
    assert np.allclose(window.basis_blocks(1)[0], c)
    assert np.allclose(state.gamma, [[1.0]])


def test_hand_computed_first_diagonal_block():
    op = _diag_op([-1.0, -2.0])
    window, state = kb.init_basis(op, np.array([[1.0], [1.0]]) / np.sqrt(2.0))
    kb.lanczos_step(op, window, state, on_zero_residual="finalize")
    assert np.allclose(state.projected_matrix().diag[0], [[-1.5]])


def test_invariant_subspace_breakdown():
    op = _diag_op([-1.0] * 4)
    c = np.zeros((4, 1))
    c[0] = 1.0
    window, state = kb.init_basis(op, c)
    with pytest.raises(kb.DeflationUnsupportedError):
        kb.lanczos_step(op, window, state)


def test_projection_identity_stored_mode():
    a = P.laplacian1d(200)
    op = kb.SparseOperator(a)
    c = np.random.default_rng(4).standard_normal((200, 2))
    window, state = kb.init_basis(op, c, storage="stored")
    for _ in range(10):
        kb.lanczos_step(op, window, state)
    m = state.n_t_blocks
    v = _full_basis(window, m)
    assert np.linalg.norm(v.T @ v - np.eye(v.shape[1])) <= 1e-10
    t = state.projected_matrix().to_dense()
    proj = v.T @ (a @ v)
    assert np.linalg.norm(proj - t) <= 1e-10 * np.linalg.norm(proj)
    assert np.linalg.eigvalsh(t)[-1] < 0.0
    coupling = window.stored[m].T @ (a @ window.stored[m - 1])
    assert np.allclose(coupling, state.coupling_block(), atol=1e-10 * np.abs(a).max())


def test_windowed_peak_storage_and_reference_blocks():
    a = P.laplacian1d(100)
    op = kb.SparseOperator(a)
    c = np.random.default_rng(5).standard_normal((100, 3))
    window, state = kb.init_basis(op, c, storage="windowed")
    bs = ko.Basis(ko.SparseOperator(a), c)
    for _ in range(8):
        kb.lanczos_step(op, window, state)
        bs.step(finalize=False)
    assert window.peak_vectors == 3 * 3
    for j in range(8):
        ref = 0.5 * (bs.diag_raw[j] + bs.diag_raw[j].T)
        assert np.allclose(state.projected_matrix().diag[j], ref, rtol=1e-12, atol=1e-9)
        assert np.allclose(state.sub[j], bs.sub[j], rtol=1e-12, atol=1e-9)
    res, rel = state.check_lyapunov()
    ref_res, _ = ko.ctri_lyapunov(bs.projection(), bs.gamma, bs.coupling())
    assert abs(res - ref_res) <= 1e-10 * ref_res


def test_determinism():
    op = kb.SparseOperator(P.laplacian1d(50))
    c = np.random.default_rng(6).standard_normal((50, 2))
    runs = []
    for _ in range(2):
        window, state = kb.init_basis(op, c.copy(), storage="stored")
        for _ in range(6):
            kb.lanczos_step(op, window, state)
        runs.append(np.concatenate(window.stored, axis=1))
    assert np.array_equal(runs[0], runs[1])


@pytest.mark.parametrize("s", [1, 3])
def test_two_pass_equals_stored(s):
    a = P.laplacian2d(20)
    op = kb.SparseOperator(a)
    c = np.random.default_rng(10 + s).random((400, s))
    m = 20
    window, state = kb.init_basis(op, c, storage="stored")
    for _ in range(m):
        kb.lanczos_step(op, window, state)
    lam, q = np.linalg.eigh(state.projected_matrix().to_dense())
    u = q[:s, :].T @ state.gamma
    yt = -(u @ u.T) / (lam[:, None] + lam[None, :])
    fac, _ = ko.truncated_spd(0.5 * (yt + yt.T))
    qy = q @ fac
    z_stored = _full_basis(window, m) @ qy
    z_two = kb.two_pass_recover(op, state, qy, window)
    assert np.linalg.norm(z_two - z_stored) <= 1e-12 * np.linalg.norm(z_stored)


def test_global_orthogonality_moderate_run():
    op = kb.SparseOperator(P.laplacian2d(16))
    c = np.random.default_rng(10).standard_normal((256, 2))
    window, state = kb.init_basis(op, c, storage="stored")
    for _ in range(40):
        kb.lanczos_step(op, window, state)
    v = _full_basis(window, 40)
    assert np.linalg.norm(v.T @ v - np.eye(80)) <= 1e-8
