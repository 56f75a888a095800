"""Time and check the dense block Jacobi kernels (csrc/dense.cu) on the
finalisation matrices of the reference goldens: T_m, Ytilde (c1, c2, c4) and
the Sylvester Ytilde (c3)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1602_05033_b200 import _lib

lib = _lib.load()
G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def dense(d, o):
    m, s = d.shape[0], d.shape[1]
    k = m * s
    t = np.zeros((k, k))
    for j in range(m):
        t[j*s:(j+1)*s, j*s:(j+1)*s] = d[j]
        if j < m - 1:
            t[(j+1)*s:(j+2)*s, j*s:(j+1)*s] = o[j]
            t[j*s:(j+1)*s, (j+1)*s:(j+2)*s] = o[j].T
    return t


def eigh(a, semidefinite=1):
    k = a.shape[0]
    q = np.asfortranarray(a).copy(order="F")
    w = np.zeros(k)
    sw = ctypes.c_int(0)
    t = time.perf_counter()
    _lib.check(lib.kry_dense_eigh(0, k, q.ctypes.data_as(_lib.dptr), _lib.as_dptr(w), ctypes.byref(sw), semidefinite))
    return w, q, sw.value, time.perf_counter() - t


def svd(a):
    m, n = a.shape
    af = np.asfortranarray(a)
    u = np.zeros((m, n), order="F"); vt = np.zeros((n, n), order="F"); sig = np.zeros(n)
    sw = ctypes.c_int(0)
    t = time.perf_counter()
    _lib.check(lib.kry_dense_svd(0, m, n, af.ctypes.data_as(_lib.dptr), u.ctypes.data_as(_lib.dptr),
                                 _lib.as_dptr(sig), vt.ctypes.data_as(_lib.dptr), ctypes.byref(sw)))
    return u, sig, vt, sw.value, time.perf_counter() - t


def report(name, a):
    for rep in range(2):
        w, q, sw, dt = eigh(a)
    ref = np.linalg.eigvalsh(a)
    k = a.shape[0]
    print("%s eigh k=%d sweeps %d wall %.1f ms  max|dw|/|w|max %.2e  orth %.2e  res %.2e" % (
        name, k, sw, dt * 1e3, np.abs(w - ref).max() / np.abs(ref).max(),
        np.linalg.norm(q.T @ q - np.eye(k)), np.linalg.norm(a @ q - q * w) / np.abs(ref).max()), flush=True)
    return w, q


for c in sys.argv[1:] or ["c1", "c2", "c4"]:
    g = np.load(os.path.join(G, c + ".npz"))
    if "j_diag" in g.files:
        ta, tb = dense(g["t_diag"], g["t_off"]), dense(g["j_diag"], g["j_off"])
        la, qa = report(c + " T", ta)
        lb, qb = report(c + " J", tb)
        s = g["gamma1"].shape[0]
        u = qa[:s].T @ g["gamma1"]; v = qb[:s].T @ g["gamma2"]
        y = -(u @ v.T) / (la[:, None] + lb[None, :])
        for rep in range(2):
            uu, sig, vt, sw, dt = svd(y)
        ref = np.linalg.svd(y, compute_uv=False)
        tail = np.sqrt(np.cumsum(sig[::-1] ** 2))[::-1]
        print("%s svd %s sweeps %d wall %.1f ms max|ds| %.2e (s0 %.2e) rank %d ref %d recon %.2e" % (
            c, y.shape, sw, dt * 1e3, np.abs(sig - ref).max(), ref[0], int((tail > 1e-12).sum()),
            int(g["rank"]), np.linalg.norm((uu * sig) @ vt - y)), flush=True)
    else:
        t = dense(g["t_diag"], g["t_off"])
        lam, q = report(c + " T", t)
        s = g["gamma"].shape[0]
        u = q[:s].T @ g["gamma"]
        y = -(u @ u.T) / (lam[:, None] + lam[None, :]); y = 0.5 * (y + y.T)
        mu, _ = report(c + " Y", y)
        mu = mu[::-1]
        tail = np.sqrt(np.cumsum(mu[::-1] ** 2))[::-1]
        r = int((tail > 1e-12).sum())
        print("%s rank %d (ref %d) discarded %.4e (ref %.4e)" % (c, r, int(g["rank"]), tail[r] if r < len(tail) else 0, float(g["discarded"])), flush=True)
