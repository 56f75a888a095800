"""CPU ORACLE -- test infrastructure, never the product path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  It restates, in plain
numpy/scipy, the reference algorithm of the hot path so the GPU results can
be checked on the same seeded inputs without /root/reference (which does not
exist on the GPU box).  Each function cites the reference code it follows
(paths relative to /root/reference/pkg/src/krymat/).

Pinned against the reference itself: tests/golden/*.npz were produced by
running the reference package (tests/golden/make_golden.py) and
tests/test_oracle.py checks this restatement against them (histories,
iteration counts, ranks, factor sketches, projected blocks) plus the
reference tests' hand-derived known answers.
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp

RANK_TOL = 1e-12        # kernels.py:22
TRUNC_EPS = 1e-12       # kernels.py:25
DENOM_TOL = 1e-14       # kernels.py:28
ZERO_BLOCK_TOL = 1e-13  # basis.py:30
REPLAY_TOL = 1e-8       # solvers.py:37


class OracleError(Exception):
    pass


class DeflationError(OracleError):
    pass


class IndefiniteError(OracleError):
    pass


class NoConvergence(OracleError):
    def __init__(self, msg, history):
        super().__init__(msg)
        self.history = history


# ----------------------------------------------------------------- operators
class SparseOperator:
    """CSR apply (operators.py:82-101); symmetric input assumed."""

    def __init__(self, a):
        self.matrix = sp.csr_matrix(a)
        self.n = self.matrix.shape[0]

    def apply(self, v):
        return self.matrix @ np.asarray(v, dtype=float)


# ----------------------------------------------------------------- dense kernels
def economy_qr(w):
    """Householder QR with diag(R) >= 0 (kernels.py:134-148)."""
    q, r = np.linalg.qr(np.asarray(w, dtype=float))
    sgn = np.where(np.diag(r) < 0.0, -1.0, 1.0)
    return q * sgn, r * sgn[:, None]


def rank_deficient(r, tol=RANK_TOL):
    """min |r_ii| < tol ||R||_F (kernels.py:151-160)."""
    nrm = np.linalg.norm(r)
    return nrm == 0.0 or bool(np.min(np.abs(np.diag(r))) < tol * nrm)


def guarded_denominators(left, right, tol=DENOM_TOL):
    """kernels.py:31-45."""
    den = np.add.outer(left, right)
    scale = max(np.abs(left).max(), np.abs(right).max())
    if np.abs(den).min() < tol * scale:
        raise IndefiniteError("eigenvalue-sum denominator is numerically singular")
    return den


@dataclass
class BlockTri:
    """Lower block bands of a symmetric block tridiagonal (kernels.py:48-108)."""

    ell: int
    diag: list
    off: list

    @property
    def dim(self):
        return self.ell * len(self.diag)

    def dense(self):
        e, k = self.ell, self.dim
        out = np.zeros((k, k))
        for i, d in enumerate(self.diag):
            out[i * e:(i + 1) * e, i * e:(i + 1) * e] = d
        for i, b in enumerate(self.off):
            out[(i + 1) * e:(i + 2) * e, i * e:(i + 1) * e] = b
            out[i * e:(i + 1) * e, (i + 1) * e:(i + 2) * e] = b.T
        return out


def _bandwidth(t):
    """Largest nonzero sub-diagonal distance (kernels.py:163-181)."""
    e = t.ell
    rr, cc = np.meshgrid(np.arange(e), np.arange(e), indexing="ij")
    bw = 1
    for d in t.diag:
        m = d != 0.0
        if m.any():
            bw = max(bw, int(np.abs(rr - cc)[m].max()))
    for b in t.off:
        m = b != 0.0
        if m.any():
            bw = max(bw, int((e + rr - cc)[m].max()))
    return min(bw, max(t.dim - 1, 1))


def band_to_tridiagonal(t):
    """Givens bulge chasing from the top, tracking only the first and last
    ell rows of the orthogonal transform (kernels.py:184-261)."""
    e, k = t.ell, t.dim
    bw = _bandwidth(t)
    if bw == 1:
        a = t.dense()
        pf = np.zeros((e, k)); pf[:, :e] = np.eye(e)
        pl = np.zeros((e, k)); pl[:, k - e:] = np.eye(e)
        return np.diag(a).copy(), np.diag(a, -1).copy(), pf, pl
    a = t.dense()
    rows = np.zeros((2 * e, k))
    rows[:e, :e] = np.eye(e)
    rows[e:, k - e:] = np.eye(e)
    for b in range(bw, 1, -1):
        for j in range(k - b):
            r, c = j + b, j
            planes, cs, sn = [], [], []
            while r < k:
                p = r - 1
                x, y = a[p, c], a[r, c]
                if y == 0.0:
                    break
                h = np.hypot(x, y)
                co, si = x / h, y / h
                g = np.array([[co, si], [-si, co]])
                lo, hi = max(0, r - b - 1), min(k, r + b + 1)
                a[p:p + 2, lo:hi] = g @ a[p:p + 2, lo:hi]
                a[lo:hi, p:p + 2] = a[lo:hi, p:p + 2] @ g.T
                a[r, c] = a[c, r] = 0.0
                planes.append(p); cs.append(co); sn.append(si)
                c, r = r - 1, r + b
            if planes:
                pi = np.array(planes)
                cv, sv = np.array(cs), np.array(sn)
                u, v = rows[:, pi].copy(), rows[:, pi + 1].copy()
                rows[:, pi] = cv * u + sv * v
                rows[:, pi + 1] = cv * v - sv * u
    return np.diag(a).copy(), np.diag(a, -1).copy(), rows[:e], rows[e:]


def tridiagonal_eig(d, e):
    """stemr -> stebz -> stev fallback chain with the sign rule
    (kernels.py:264-293)."""
    if d.size == 1:
        return d.copy(), np.ones((1, 1))
    for drv in ("stemr", "stebz", "stev"):
        try:
            lam, g = scipy.linalg.eigh_tridiagonal(d, e, lapack_driver=drv)
            break
        except np.linalg.LinAlgError:
            lam = None
    if lam is None:
        raise OracleError("tridiagonal eigensolver failed")
    piv = np.argmax(np.abs(g), axis=0)
    g[:, g[piv, np.arange(g.shape[1])] < 0.0] *= -1.0
    return lam, g


def partial_eig(t):
    """(lam, E1^T Q, Em^T Q) (kernels.py:296-306)."""
    d, e, pf, pl = band_to_tridiagonal(t)
    lam, g = tridiagonal_eig(d, e)
    return lam, pf @ g, pl @ g


def ctri_lyapunov(t, gamma, tau, beta2=None):
    """sqrt(2) ||((u u^T) / (lam_i + lam_j)) w||_F (residual.py:40-59)."""
    gamma = np.atleast_2d(gamma)
    lam, f1, fm = partial_eig(t)
    den = guarded_denominators(lam, lam)
    u = f1.T @ gamma
    w = fm.T @ np.atleast_2d(tau).T
    res = float(np.sqrt(2.0) * np.linalg.norm(((u @ u.T) / den) @ w))
    b2 = float(np.sum(gamma ** 2)) if beta2 is None else float(beta2)
    return res, res / b2


def ctri_sylvester(t, j, g1, g2, tau, iota, rhs=None):
    """residual.py:62-84 (no sqrt(2); both coupling terms)."""
    lt, ft, lt_last = partial_eig(t)
    lj, fj, lj_last = partial_eig(j)
    den = guarded_denominators(lt, lj)
    sd = ((ft.T @ np.atleast_2d(g1)) @ (fj.T @ np.atleast_2d(g2)).T) / den
    f = lt_last.T @ np.atleast_2d(tau).T
    g = lj_last.T @ np.atleast_2d(iota).T
    res = float(np.hypot(np.linalg.norm(sd.T @ f), np.linalg.norm(sd @ g)))
    if rhs is None:
        rhs = np.linalg.norm(g1) * np.linalg.norm(g2)
    return res, res / float(rhs)


def truncated_spd(y, eps=TRUNC_EPS):
    """kernels.py:309-331: descending eigen-split with the exact tail rule."""
    lam, w = np.linalg.eigh(y)
    if lam.size and lam[0] < -1e-10 * np.abs(lam).max():
        raise IndefiniteError("significantly indefinite")
    lam, w = lam[::-1], w[:, ::-1]
    tail = np.sqrt(np.cumsum(lam[::-1] ** 2))[::-1]
    r = int(np.count_nonzero(tail > eps))
    disc = float(tail[r]) if r < lam.size else 0.0
    return w[:, :r] * np.sqrt(np.clip(lam[:r], 0.0, None)), disc


def truncated_svd(y, eps=TRUNC_EPS):
    """kernels.py:334-345."""
    u, sg, vt = np.linalg.svd(y, full_matrices=False)
    tail = np.sqrt(np.cumsum(sg[::-1] ** 2))[::-1]
    r = int(np.count_nonzero(tail > eps))
    disc = float(tail[r]) if r < sg.size else 0.0
    root = np.sqrt(sg[:r])
    return u[:, :r] * root, vt[:r].T * root, disc


# ----------------------------------------------------------------- basis
def mgs_twice(w, older, current):
    """Block MGS performed twice, returning the summed coefficients
    (basis.py:164-180)."""
    a_sum = None if older is None else np.zeros((older.shape[1], w.shape[1]))
    b_sum = np.zeros((current.shape[1], w.shape[1]))
    for _ in (0, 1):
        if older is not None:
            coef = older.T @ w
            a_sum += coef
            w = w - older @ coef
        coef = current.T @ w
        b_sum += coef
        w = w - current @ coef
    return w, a_sum, b_sum


class Basis:
    """Three-block window + projection coefficients (basis.py:33-161,
    standard space only)."""

    def __init__(self, op, c):
        c = np.asarray(c, dtype=float)
        if c.ndim != 2 or c.shape[0] != op.n:
            raise OracleError("rhs shape mismatch")
        q, r = economy_qr(c)
        if rank_deficient(r):
            raise DeflationError("initial QR of C")
        self.op, self.rhs, self.s = op, c, c.shape[1]
        self.gamma = r
        self.blocks = [q]           # at most the last three are needed
        self.diag_raw, self.off_mgs, self.sub = [], [], []
        self.exhausted = False

    @property
    def m(self):
        return len(self.diag_raw)

    def step(self, finalize=True):
        """basis.py:223-252."""
        older = self.blocks[-2] if len(self.blocks) > 1 else None
        cur = self.blocks[-1]
        w = self.op.apply(cur)
        scale = np.linalg.norm(w)
        w, a, b = mgs_twice(w, older, cur)
        self.off_mgs.append(a)
        self.diag_raw.append(b)
        if finalize and np.linalg.norm(w) <= ZERO_BLOCK_TOL * scale:
            self.sub.append(np.zeros((self.s, self.s)))
            self.exhausted = True
            return
        q, r = economy_qr(w)
        if rank_deficient(r):
            raise DeflationError("Lanczos step %d" % self.m)
        self.sub.append(r)
        self.blocks = self.blocks[-1:] + [q]

    def projection(self):
        """basis.py:131-147."""
        m = self.m
        return BlockTri(self.s, [0.5 * (d + d.T) for d in self.diag_raw[:m]],
                        list(self.sub[:m - 1]))

    def coupling(self):
        return self.sub[self.m - 1]


def two_pass_recover(op, basis, qy):
    """Regenerate V_2..V_m with recomputed MGS/QR, check the couplings and
    accumulate Z (solvers.py:130-169)."""
    e, m = basis.s, basis.m
    v, _ = economy_qr(basis.rhs)
    z = v @ qy[:e]
    older = None
    for i in range(2, m + 1):
        w, _, _ = mgs_twice(op.apply(v), older, v)
        vn, tau = economy_qr(w)
        ref = basis.sub[i - 2]
        if np.linalg.norm(tau - ref) > REPLAY_TOL * max(np.linalg.norm(ref), 1e-300):
            raise OracleError("replay mismatch at step %d" % i)
        z += vn @ qy[(i - 1) * e:i * e]
        older, v = v, vn
    return z


# ----------------------------------------------------------------- drivers
@dataclass
class SolveOptions:
    tol: float = 1e-6
    max_m: int = 500
    check_period: int = 1
    storage: str = "windowed"
    trunc_eps: float = TRUNC_EPS


@dataclass
class Solution:
    z1: np.ndarray
    z2: np.ndarray = None
    rank: int = 0
    iterations: int = 0
    final_residual: float = np.inf
    history: list = field(default_factory=list)
    discarded: float = 0.0
    basis: object = None

    @property
    def z(self):
        return self.z1


def solve_lyapunov(op, c, opts=None, keep_basis=False):
    """solvers.py:200-285 (standard space, two-pass recovery)."""
    opts = opts or SolveOptions()
    c = np.atleast_2d(np.asarray(c, dtype=float))
    beta2 = float(np.linalg.norm(c) ** 2)
    bs = Basis(op, c)
    hist, done, rel = [], None, None
    for it in range(1, opts.max_m + 1):
        bs.step()
        if it % opts.check_period == 0 or bs.exhausted:
            _, rel = ctri_lyapunov(bs.projection(), bs.gamma, bs.coupling(), beta2)
            hist.append((it, it * bs.s, rel))
            if rel <= opts.tol:
                done = it
                break
            if bs.exhausted:
                raise NoConvergence("invariant", hist)
    if done is None:
        raise NoConvergence("max_m", hist)
    lam, q = np.linalg.eigh(bs.projection().dense())
    if lam[-1] >= 0.0:
        raise IndefiniteError("projected matrix is not negative definite")
    u = q[:bs.s].T @ bs.gamma
    y = -(u @ u.T) / guarded_denominators(lam, lam)
    fac, disc = truncated_spd(0.5 * (y + y.T), opts.trunc_eps)
    z = two_pass_recover(op, bs, q @ fac)
    return Solution(z, rank=fac.shape[1], iterations=done, final_residual=rel,
                    history=hist, discarded=disc, basis=bs if keep_basis else None)


def solve_sylvester(op_a, op_b, c1, c2, opts=None):
    """solvers.py:288-383 (standard space, two-pass recovery)."""
    opts = opts or SolveOptions()
    c1 = np.atleast_2d(np.asarray(c1, dtype=float))
    c2 = np.atleast_2d(np.asarray(c2, dtype=float))
    rhs = float(np.linalg.norm(c1) * np.linalg.norm(c2))
    ba, bb = Basis(op_a, c1), Basis(op_b, c2)
    hist, done, rel = [], None, None
    for it in range(1, opts.max_m + 1):
        if not ba.exhausted:
            ba.step()
        if not bb.exhausted:
            bb.step()
        both = ba.exhausted and bb.exhausted
        if it % opts.check_period == 0 or both:
            _, rel = ctri_sylvester(ba.projection(), bb.projection(), ba.gamma, bb.gamma,
                                    ba.coupling(), bb.coupling(), rhs)
            hist.append((it, it * ba.s, rel))
            if rel <= opts.tol:
                done = it
                break
            if both:
                raise NoConvergence("invariant", hist)
    if done is None:
        raise NoConvergence("max_m", hist)
    la, qa = np.linalg.eigh(ba.projection().dense())
    lb, qb = np.linalg.eigh(bb.projection().dense())
    if la[-1] >= 0.0 or lb[-1] >= 0.0:
        raise IndefiniteError("a projected matrix is not negative definite")
    u = qa[:ba.s].T @ ba.gamma
    v = qb[:bb.s].T @ bb.gamma
    y = -(u @ v.T) / guarded_denominators(la, lb)
    f1, f2, disc = truncated_svd(y, opts.trunc_eps)
    z1 = two_pass_recover(op_a, ba, qa @ f1)
    z2 = two_pass_recover(op_b, bb, qb @ f2)
    return Solution(z1, z2, rank=f1.shape[1], iterations=done, final_residual=rel,
                    history=hist, discarded=disc)


def residual_one_sided(t, tau, s_input, ups, rhs=None):
    """residual.py:87-104: ||((s_input F) / (ups_i + lam_j)) (L^T tau^T)||_F."""
    lam, f1, fm = partial_eig(t)
    den = guarded_denominators(np.asarray(ups, dtype=float), lam)
    m = ((np.asarray(s_input, dtype=float) @ f1) / den) @ (fm.T @ np.atleast_2d(tau).T)
    res = float(np.linalg.norm(m))
    return res, res / float(rhs) if rhs is not None else res


def solve_sylvester_one_sided(op_a, b, c1, c2, opts=None):
    """solvers.py:386-481 (standard space, two-pass recovery): B small and
    dense, eigendecomposed once; only A is projected."""
    opts = opts or SolveOptions()
    b = np.asarray(b, dtype=float)
    c1 = np.atleast_2d(np.asarray(c1, dtype=float))
    c2 = np.atleast_2d(np.asarray(c2, dtype=float))
    if not np.array_equal(b, b.T):
        raise OracleError("small coefficient matrix B must be symmetric")
    rhs = float(np.linalg.norm(c1) * np.linalg.norm(c2))
    ups, p = np.linalg.eigh(b)
    if ups[-1] >= 0.0:
        raise IndefiniteError("B must be negative definite")
    bs = Basis(op_a, c1)
    s_input = (p.T @ c2) @ bs.gamma.T
    hist, done, rel = [], None, None
    for it in range(1, opts.max_m + 1):
        bs.step()
        if it % opts.check_period == 0 or bs.exhausted:
            _, rel = residual_one_sided(bs.projection(), bs.coupling(), s_input, ups, rhs)
            hist.append((it, it * bs.s, rel))
            if rel <= opts.tol:
                done = it
                break
            if bs.exhausted:
                raise NoConvergence("invariant", hist)
    if done is None:
        raise NoConvergence("max_m", hist)
    lam, q = np.linalg.eigh(bs.projection().dense())
    if lam[-1] >= 0.0:
        raise IndefiniteError("projected matrix is not negative definite")
    u = q[:bs.s].T @ bs.gamma
    y = -(u @ (c2.T @ p)) / guarded_denominators(lam, ups)
    f1, f2, disc = truncated_svd(y, opts.trunc_eps)
    z1 = two_pass_recover(op_a, bs, q @ f1)
    return Solution(z1, p @ f2, rank=f1.shape[1], iterations=done, final_residual=rel,
                    history=hist, discarded=disc)


# ----------------------------------------------------------------- comparison helpers
def factor_distance(za, zb, za2=None, zb2=None):
    """||Za Za2^T - Zb Zb2^T||_F / ||Zb Zb2^T||_F without forming n x n
    matrices: thin QR of [Za, Zb] (and of the right factors) reduces the
    difference to small cores."""
    if za2 is None:
        za2, zb2 = za, zb
    ql, rl = np.linalg.qr(np.hstack([za, zb]))
    qr_, rr = np.linalg.qr(np.hstack([za2, zb2]))
    ta = za.shape[1]
    a = rl[:, :ta] @ rr[:, :ta].T
    b = rl[:, ta:] @ rr[:, ta:].T
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
