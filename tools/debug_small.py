"""Debug: compare device projection blocks / residuals with the oracle."""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1602_05033_b200 as kb
from paper_1602_05033_b200 import _lib
from oracle import krymat_oracle as ko, problems as P

n, s, steps = 12, 2, 8
a = P.laplacian2d(n)
c = np.random.default_rng(5).standard_normal((n * n, s))
op = kb.SparseOperator(a)
print("kind", op.kind)
ctx = op.context(s, 60)
lib = _lib.load()
gamma = np.zeros((s, s)); b2 = ctypes.c_double()
_lib.check(lib.kry_init_basis(ctx.ptr, _lib.as_dptr(c), _lib.as_dptr(gamma), ctypes.byref(b2)))
bs = ko.Basis(ko.SparseOperator(a), c)
print("gamma dev\n", gamma, "\ngamma ref\n", bs.gamma, "\nbeta2", b2.value, np.linalg.norm(c)**2)
for it in range(1, steps + 1):
    ex = ctypes.c_int()
    _lib.check(lib.kry_lanczos_step(ctx.ptr, 1, ctypes.byref(ex)))
    bs.step()
    m = ctypes.c_int()
    dr = np.zeros((it, s, s)); ds = np.zeros((it, s, s)); of = np.zeros((it, s, s)); sb = np.zeros((it, s, s))
    _lib.check(lib.kry_get_projection(ctx.ptr, ctypes.byref(m), _lib.as_dptr(dr), _lib.as_dptr(ds), _lib.as_dptr(of), _lib.as_dptr(sb)))
    res, rel = ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.kry_check_lyap(ctx.ptr, b2.value, ctypes.byref(res), ctypes.byref(rel)))
    _, rrel = ko.ctri_lyapunov(bs.projection(), bs.gamma, bs.coupling(), np.linalg.norm(c)**2)
    print("it", it, "m", m.value, "diag err", np.abs(ds[-1] - 0.5*(bs.diag_raw[-1]+bs.diag_raw[-1].T)).max(),
          "sub err", np.abs(sb[-1] - bs.sub[-1]).max(), "rel", rel.value, rrel)
    if it <= 2:
        print(" dev diag", ds[-1].ravel(), "\n ref diag", (0.5*(bs.diag_raw[-1]+bs.diag_raw[-1].T)).ravel())
        print(" dev sub", sb[-1].ravel(), "\n ref sub", bs.sub[-1].ravel())
t = kb.BlockTridiagonal(s, [0.5*(d+d.T) for d in bs.diag_raw], list(bs.sub[:-1]))
pe = kb.partial_eig_blocktridiag(t)
lam = np.linalg.eigvalsh(t.to_dense())
print("partial eig lam err", np.abs(pe.eigenvalues - lam).max(), "lam", lam[:3], pe.eigenvalues[:3])
ctx.close()
