"""The slab-sharded multi-GPU path executed for real.

Every rank owns a slab of z-planes of the grid; the library exchanges one
halo plane per neighbour after each new basis block and sums each Gram
reduction over the ranks before the replicated coefficient solve
(halo_exchange / allreduce_gram in csrc/api.cu).  Without a multi-GPU node
the ranks run as threads of one process on one GPU with the loopback
transport (kry_loop): the same sharded kernels, POST_NONE reductions and
post routines as with NCCL, only the transport differs.  The reference has
no sharded counterpart; its single-process run (tests/golden/c2.npz,
c4.npz) is the oracle: iterations and rank exact, history within 1e-9 rel +
floor (the ranks sum the Gram partials in another order), factor sketch to
1e-8, and every rank reports the same history.
"""

import os

import numpy as np
import pytest

import paper_1602_05033_b200 as kb
from oracle import problems as P
from paper_1602_05033_b200.operators import StencilOperator, detect_stencil
from paper_1602_05033_b200.parallel import local_rows, run_ranks, slab_partition

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    path = os.path.join(GOLD, name + ".npz")
    if not os.path.exists(path):
        pytest.skip("golden %s not generated" % name)
    return np.load(path)


def _sharded_solve(a, grid, c, opts, nranks):
    st = detect_stencil(a)
    assert st is not None and st["constant"]

    def rank(r, comm):
        z = slab_partition(grid[2], nranks, r)
        op = StencilOperator(grid, st["c_diag"], st["c_x"], st["c_y"], st["c_z"],
                             slab=z, comm=comm)
        return kb.solve_lyapunov(op, local_rows(c, grid, z), opts)

    return run_ranks(nranks, rank)


def _check(sols, g, floor):
    h0 = [r[2] for r in sols[0].history]
    for s in sols[1:]:
        assert [r[2] for r in s.history] == h0          # replicated projection
        assert s.iterations == sols[0].iterations and s.rank == sols[0].rank
    ref = g["history"][:, 2]
    h = np.array(h0)
    assert sols[0].iterations == int(g["iterations"])
    assert sols[0].rank == int(g["rank"])
    assert np.all(np.abs(h - ref) <= 1e-9 * ref + floor), np.max(np.abs(h - ref) / ref)
    return np.vstack([s.z for s in sols])


@pytest.mark.parametrize("nranks", [2, 4])
def test_c2_slab_sharded_matches_reference(nranks):
    g = gold("c2")
    cfg = P.build_config("c2")
    opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
    sols = _sharded_solve(cfg["a"], (50, 50, 50), cfg["c"], opts, nranks)
    z = _check(sols, g, 2e-16)
    om = P.sketch_omega(z.shape[0], 2)
    sk = z @ (z.T @ om)
    assert np.linalg.norm(sk - g["sketch"]) <= 1e-8 * np.linalg.norm(g["sketch"])


def test_c4_slab_sharded_two_ranks_matches_reference():
    import bench
    g = gold("c4")
    cfg, _, _ = bench.build_problem("c4")
    from paper_1602_05033_b200 import problems as PP
    opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")

    def rank(r, comm):
        z = slab_partition(200, 2, r)
        op = PP.stencil_operator((200, 200, 200), slab=z, comm=comm)
        return kb.solve_lyapunov(op, local_rows(cfg["c"], (200, 200, 200), z), opts)

    sols = run_ranks(2, rank)
    z = _check(sols, g, 2e-16)
    rows = g["sketch_rows"]
    om = P.sketch_omega(z.shape[0], 2)
    sk = (z @ (z.T @ om))[rows]
    assert np.linalg.norm(sk - g["sketch"]) <= 1e-8 * np.linalg.norm(g["sketch"])
