"""ctypes binding of libkrymat_b200.so (the C-ABI in include/krymat_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_1602_05033_b200/csrc``).  There is no fallback: if the
library is missing or no CUDA device is visible, every compute entry point
raises.
"""

import ctypes
import os

import numpy as np

from .errors import (
    AsymmetricMatrixError,
    ConvergenceError,
    DeflationUnsupportedError,
    DimensionMismatchError,
    FactorizationError,
    IndefiniteMatrixError,
    KrymatError,
    RecurrenceMismatchError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libkrymat_b200.so")

KRY_OK = 0
KRY_ERR_DIMENSION = 1
KRY_ERR_ASYMMETRIC = 2
KRY_ERR_DEFLATION = 3
KRY_ERR_INDEFINITE = 4
KRY_ERR_FACTORIZATION = 5
KRY_ERR_RECURRENCE = 6
KRY_ERR_CUDA = 7
KRY_ERR_ARGUMENT = 8
KRY_ERR_NCCL = 9
KRY_ERR_STATE = 10
KRY_ERR_CONVERGENCE = 11

KRY_OP_STENCIL = 0
KRY_OP_CSR = 1

_EXC = {
    KRY_ERR_DIMENSION: DimensionMismatchError,
    KRY_ERR_ASYMMETRIC: AsymmetricMatrixError,
    KRY_ERR_DEFLATION: DeflationUnsupportedError,
    KRY_ERR_INDEFINITE: IndefiniteMatrixError,
    KRY_ERR_FACTORIZATION: FactorizationError,
    KRY_ERR_RECURRENCE: RecurrenceMismatchError,
    KRY_ERR_CUDA: KrymatError,
    KRY_ERR_ARGUMENT: ValueError,
    KRY_ERR_NCCL: KrymatError,
    KRY_ERR_STATE: KrymatError,
    KRY_ERR_CONVERGENCE: ConvergenceError,
}

dptr = ctypes.POINTER(ctypes.c_double)
iptr = ctypes.POINTER(ctypes.c_int)


class OperatorDesc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("variable", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("nx", ctypes.c_int64),
        ("ny", ctypes.c_int64),
        ("nz", ctypes.c_int64),
        ("c_diag", ctypes.c_double),
        ("c_x", ctypes.c_double),
        ("c_y", ctypes.c_double),
        ("c_z", ctypes.c_double),
        ("diag", dptr),
        ("cx", dptr),
        ("cy", dptr),
        ("cz", dptr),
        ("nnz", ctypes.c_int64),
        ("indptr", ctypes.POINTER(ctypes.c_int64)),
        ("indices", ctypes.POINTER(ctypes.c_int32)),
        ("values", dptr),
        ("z_begin", ctypes.c_int64),
        ("z_end", ctypes.c_int64),
    ]


# exported symbol -> (restype, argtypes)
_P = ctypes.c_void_p
SIGNATURES = {
    "kry_version": (ctypes.c_int, []),
    "kry_last_error": (ctypes.c_char_p, []),
    "kry_device_count": (ctypes.c_int, [iptr]),
    "kry_launch_count": (ctypes.c_int64, []),
    "kry_reset_launch_count": (None, []),
    "kry_ctx_create": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int,
                                      ctypes.POINTER(OperatorDesc), ctypes.c_int,
                                      ctypes.c_int]),
    "kry_ctx_destroy": (None, [_P]),
    "kry_ctx_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64), iptr, iptr, iptr]),
    "kry_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "kry_comm_init": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    "kry_fp64_peak": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double)]),
    "kry_profile_check": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_int)]),
    "kry_profile_zacc": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_int)]),
    "kry_loop_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "kry_loop_destroy": (None, [ctypes.c_void_p]),
    "kry_comm_init_loopback": (ctypes.c_int, [_P, ctypes.c_void_p, ctypes.c_int]),
    "kry_apply": (ctypes.c_int, [_P, dptr, dptr, ctypes.c_int]),
    "kry_init_basis": (ctypes.c_int, [_P, dptr, dptr, dptr]),
    "kry_init_basis_device": (ctypes.c_int, [_P, ctypes.c_void_p, dptr, dptr]),
    "kry_lanczos_step": (ctypes.c_int, [_P, ctypes.c_int, iptr]),
    "kry_get_projection": (ctypes.c_int, [_P, iptr, dptr, dptr, dptr, dptr]),
    "kry_get_window": (ctypes.c_int, [_P, dptr, dptr, iptr]),
    "kry_check_lyap": (ctypes.c_int, [_P, ctypes.c_double, dptr, dptr]),
    "kry_check_sylv": (ctypes.c_int, [_P, _P, ctypes.c_double, dptr, dptr]),
    "kry_solve_lyap_pass1": (ctypes.c_int, [_P, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                            dptr, iptr, iptr, dptr, iptr]),
    "kry_solve_sylv_pass1": (ctypes.c_int, [_P, _P, ctypes.c_double, ctypes.c_int,
                                            ctypes.c_int, dptr, iptr, iptr, dptr, iptr]),
    "kry_finalize_lyap": (ctypes.c_int, [_P, ctypes.c_double, iptr, dptr]),
    "kry_finalize_sylv": (ctypes.c_int, [_P, _P, ctypes.c_double, iptr, dptr]),
    "kry_recover": (ctypes.c_int, [_P, dptr]),
    "kry_set_storage": (ctypes.c_int, [_P, ctypes.c_int]),
    "kry_set_qy": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, dptr]),
    "kry_get_factor": (ctypes.c_int, [_P, dptr]),
    "kry_partial_eig": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, dptr, dptr,
                                       dptr, dptr, dptr]),
    "kry_band_eigh": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, dptr, dptr, dptr,
                                     dptr]),
    "kry_dense_eigh": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, dptr, dptr, iptr, ctypes.c_int]),
    "kry_dense_svd": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, dptr, dptr, dptr,
                                     dptr, iptr]),
    "kry_ctri_lyap_blocks": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, dptr,
                                            dptr, dptr, dptr, dptr]),
    "kry_ctri_sylv_blocks": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, dptr,
                                            dptr, ctypes.c_int, dptr, dptr, dptr, dptr, dptr,
                                            dptr, dptr]),
    "kry_true_lyap_residual": (ctypes.c_int, [_P, dptr, ctypes.c_int, dptr, dptr]),
    "kry_sylv1_setup": (ctypes.c_int, [_P, ctypes.c_int, dptr, dptr, dptr]),
    "kry_check_sylv1": (ctypes.c_int, [_P, ctypes.c_double, dptr, dptr]),
    "kry_finalize_sylv1": (ctypes.c_int, [_P, ctypes.c_double, iptr, dptr, dptr, ctypes.c_int]),
    "kry_profile_enable": (ctypes.c_int, [_P, ctypes.c_int]),
    "kry_profile_read": (ctypes.c_int, [_P, dptr, iptr, dptr, iptr]),
    "kry_timer": (ctypes.c_int, [_P, ctypes.c_int, dptr]),
}

_lib = None


def load():
    """Load the in-tree shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("KRY_LIB_PATH", LIB_PATH)   # experiments: alternative build
    if not os.path.exists(path):
        raise KrymatError(
            "libkrymat_b200.so is not built (expected at %s); run "
            "`python -c 'import __graft_entry__ as g; g.build()'`" % LIB_PATH)
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error():
    msg = load().kry_last_error()
    return msg.decode() if msg else ""


def check(code, history=None):
    """Raise the reference exception class for a C-ABI status code."""
    if code == KRY_OK:
        return
    exc = _EXC.get(code, KrymatError)
    msg = last_error()
    if exc is ConvergenceError:
        raise ConvergenceError(msg, history)
    raise exc(msg)


_device_checked = False


def require_device():
    """Fail loudly when no CUDA device is visible (no CPU fallback)."""
    global _device_checked
    if _device_checked:
        return
    n = ctypes.c_int(0)
    rc = load().kry_device_count(ctypes.byref(n))
    if rc != KRY_OK or n.value < 1:
        raise KrymatError("no CUDA device available: the B200 solver has no CPU path (%s)"
                          % last_error())
    _device_checked = True


def as_dptr(a):
    return a.ctypes.data_as(dptr)


def c_double_array(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def launch_count():
    return int(load().kry_launch_count())


def reset_launch_count():
    load().kry_reset_launch_count()
