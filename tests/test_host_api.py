"""CPU: the host side of the drop-in API (no device calls): option
validation, result record, error-class mapping of the C-ABI status codes,
the exact symmetry check and its message, stencil detection from CSR, and
the host factor allocation.  Mirrors the reference tests of the same
behaviour (reference pkg/tests/test_solvers.py, test_cli.py:53-61)."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1602_05033_b200 as kb
from paper_1602_05033_b200 import _lib, problems as P, solvers


# ------------------------------------------------------------------ options / record
def test_solve_options_defaults_match_reference():
    o = kb.SolveOptions()
    assert (o.tol, o.max_m, o.check_period, o.space, o.storage) == (1e-6, 500, 1, "standard",
                                                                    "stored")
    assert o.trunc_eps == kb.TRUNC_EPS == 1e-12
    assert o.verify is False


@pytest.mark.parametrize("kw", [dict(tol=0.0), dict(tol=-1.0), dict(check_period=0),
                                dict(space="rational"), dict(storage="disk")])
def test_solve_options_reject_bad_values(kw):
    with pytest.raises(ValueError):
        kb.SolveOptions(**kw)


def test_history_columns_and_solution_record():
    assert kb.HISTORY_COLUMNS == ("m", "space_dim", "relative_residual", "cum_basis_secs",
                                  "cum_residual_secs")
    z = np.arange(6.0).reshape(3, 2)
    sol = kb.LowRankSolution(z1=z, rank=2)
    assert sol.z is z or np.array_equal(sol.z, z)   # Lyapunov: z2 defaults to z1
    assert sol.final_residual == np.inf and sol.history == []


# ------------------------------------------------------------------ status -> exception
@pytest.mark.parametrize("code,exc", [
    (_lib.KRY_ERR_DIMENSION, kb.DimensionMismatchError),
    (_lib.KRY_ERR_ASYMMETRIC, kb.AsymmetricMatrixError),
    (_lib.KRY_ERR_DEFLATION, kb.DeflationUnsupportedError),
    (_lib.KRY_ERR_INDEFINITE, kb.IndefiniteMatrixError),
    (_lib.KRY_ERR_FACTORIZATION, kb.FactorizationError),
    (_lib.KRY_ERR_RECURRENCE, kb.RecurrenceMismatchError),
    (_lib.KRY_ERR_CUDA, kb.KrymatError),
    (_lib.KRY_ERR_ARGUMENT, ValueError),
])
def test_status_codes_map_to_reference_exceptions(code, exc):
    with pytest.raises(exc):
        _lib.check(code)
    _lib.check(_lib.KRY_OK)


def test_convergence_error_carries_history():
    rows = [(1, 2, 0.5, 0.0, 0.0)]
    with pytest.raises(kb.ConvergenceError) as err:
        _lib.check(_lib.KRY_ERR_CONVERGENCE, rows)
    assert err.value.history == rows


def test_exception_hierarchy():
    for cls in (kb.DimensionMismatchError, kb.AsymmetricMatrixError,
                kb.DeflationUnsupportedError, kb.IndefiniteMatrixError,
                kb.FactorizationError, kb.RecurrenceMismatchError, kb.ConvergenceError):
        assert issubclass(cls, kb.KrymatError)


# ------------------------------------------------------------------ symmetry check
def test_validate_symmetric_message_names_first_pair():
    a = sp.csr_matrix(np.array([[2.0, 1.0], [0.5, 2.0]]))
    with pytest.raises(kb.AsymmetricMatrixError) as err:
        kb.validate_symmetric(a)
    msg = str(err.value)
    assert "not symmetric" in msg and "(0, 1)" in msg


def test_validate_symmetric_rejects_non_square():
    with pytest.raises(kb.DimensionMismatchError):
        kb.validate_symmetric(sp.csr_matrix(np.ones((2, 3))))


def test_validate_symmetric_accepts_generators():
    for a in (P.laplacian1d(9), P.gen_fd2d("varcoef2d", 7), P.laplacian3d(4)):
        assert kb.validate_symmetric(a).shape == a.shape


# ------------------------------------------------------------------ stencil detection
@pytest.mark.parametrize("name,builder,grid,constant", [
    ("1d", lambda: P.laplacian1d(11), (11, 1, 1), True),
    ("2d", lambda: P.gen_fd2d("laplacian2d", 9), (9, 9, 1), True),
    ("3d", lambda: P.laplacian3d(5), (5, 5, 5), True),
    ("var", lambda: P.gen_fd2d("varcoef2d", 8), (8, 8, 1), False),
])
def test_detect_stencil_recovers_grid_and_coefficients(name, builder, grid, constant):
    a = sp.csr_matrix(builder())
    a.sum_duplicates()
    d = kb.detect_stencil(a)
    assert d is not None and tuple(d["grid"]) == grid and d["constant"] == constant
    n = a.shape[0]
    nx, ny, _ = grid
    # rebuild the matrix from the detected coefficients: identical entries
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [d["diag"]]
    for key, off in (("cx", 1), ("cy", nx), ("cz", nx * ny)):
        arr = d[key]
        i = np.flatnonzero(arr)
        rows += [i, i + off]
        cols += [i + off, i]
        vals += [arr[i], arr[i]]
    b = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    assert (a != b).nnz == 0


def test_detect_stencil_rejects_general_sparsity():
    rng = np.random.default_rng(0)
    m = sp.random(30, 30, density=0.2, random_state=rng)
    assert kb.detect_stencil(sp.csr_matrix(m + m.T + 30 * sp.identity(30))) is None


# ------------------------------------------------------------------ host factor
def test_host_factor_small_is_plain_numpy():
    z = solvers.host_factor(1000, 7)
    assert z.shape == (1000, 7) and z.dtype == np.float64 and z.flags.c_contiguous
