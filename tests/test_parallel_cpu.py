"""CPU (gloo, world size 2/3): the slab-sharded block-Lanczos step.

The library shards a grid operator into z-slabs (paper_1602_05033_b200.parallel),
exchanges one plane per neighbour after each basis block and all-reduces the
Gram partials before the replicated coefficient solve.  Here the same
partition and halo plan drive a NumPy model of that step with torch.distributed
(gloo) as the transport; the projected blocks must match the unsharded
oracle, which is what makes the sharded GPU path correct by construction.
"""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1602_05033_b200.parallel import halo_plan, local_rows, slab_partition


def test_slab_partition_covers_and_balances():
    for nz, n in ((200, 1), (200, 2), (200, 8), (50, 3), (7, 7), (40, 6)):
        parts = [slab_partition(nz, n, r) for r in range(n)]
        assert parts[0][0] == 0 and parts[-1][1] == nz
        assert all(parts[r][1] == parts[r + 1][0] for r in range(n - 1))
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab_partition(3, 4, 0)


def test_halo_plan_is_symmetric():
    for n in (2, 3, 5):
        plans = [halo_plan(20, n, r) for r in range(n)]
        for r, p in enumerate(plans):
            for peer, plane in p["send"].items():
                # what r sends to peer is what peer receives from r
                assert plans[peer]["recv"][r] == plane


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _laplacian3d(n):
    h = 1.0 / (n + 1)
    lap = sp.diags([np.full(n - 1, 1 / h**2), np.full(n, -2 / h**2), np.full(n - 1, 1 / h**2)],
                   (-1, 0, 1)).tocsr()
    eye = sp.identity(n, format="csr")
    a = sp.kron(eye, sp.kron(eye, lap)) + sp.kron(eye, sp.kron(lap, eye))
    return (a + sp.kron(lap, sp.kron(eye, eye))).tocsr()


def _allreduce(x):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _sharded_run(rank, nranks, port, n, s, steps, out):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        a = _laplacian3d(n)
        grid = (n, n, n)
        nxy = n * n
        c = np.random.default_rng(11).standard_normal((n ** 3, s))
        z0, z1 = slab_partition(n, nranks, rank)
        plan = halo_plan(n, nranks, rank)
        lo, hi = max(z0 - 1, 0), min(z1 + 1, n)
        a_loc = a[z0 * nxy:z1 * nxy, lo * nxy:hi * nxy]

        def apply(v):
            # halo exchange per the plan, then the local rows of A
            reqs, recv = [], {}
            for peer, plane in plan["send"].items():
                buf = torch.from_numpy(np.ascontiguousarray(v[(plane - z0) * nxy:(plane - z0 + 1) * nxy]))
                reqs.append(dist.isend(buf, peer))
            for peer, plane in plan["recv"].items():
                recv[plane] = torch.zeros((nxy, s), dtype=torch.float64)
                reqs.append(dist.irecv(recv[plane], peer))
            for r in reqs:
                r.wait()
            ext = [recv[z0 - 1].numpy()] if z0 > 0 else []
            ext.append(v)
            if z1 < n:
                ext.append(recv[z1].numpy())
            return a_loc @ np.vstack(ext)

        def cholqr2(w):
            r1 = np.linalg.cholesky(_allreduce(w.T @ w)).T
            q = np.linalg.solve(r1.T, w.T).T
            r2 = np.linalg.cholesky(_allreduce(q.T @ q)).T
            return np.linalg.solve(r2.T, q.T).T, r2 @ r1

        v, gamma = cholqr2(local_rows(c, grid, (z0, z1)))
        older, diag, sub = None, [], []
        for _ in range(steps):
            w = apply(v)
            b_sum = np.zeros((s, s))
            for _sweep in range(2):
                if older is not None:
                    al = _allreduce(older.T @ w)
                    w = w - older @ al
                be = _allreduce(v.T @ w)
                b_sum += be
                w = w - v @ be
            vn, r = cholqr2(w)
            diag.append(0.5 * (b_sum + b_sum.T))
            sub.append(r)
            older, v = v, vn
        if rank == 0:
            out.put((np.array(diag), np.array(sub), gamma))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_lanczos_matches_unsharded_oracle(nranks):
    from oracle import krymat_oracle as ko

    n, s, steps = 6, 2, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_run, args=(r, nranks, port, n, s, steps, q))
             for r in range(nranks)]
    for p in procs:
        p.start()
    diag, sub, gamma = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = _laplacian3d(n)
    c = np.random.default_rng(11).standard_normal((n ** 3, s))
    bs = ko.Basis(ko.SparseOperator(a), c)
    for _ in range(steps):
        bs.step()
    t = bs.projection()
    scale = np.abs(a.diagonal()).max()
    assert np.allclose(np.abs(gamma), np.abs(bs.gamma), rtol=1e-12, atol=1e-12)
    for j in range(steps):
        ref_d = 0.5 * (bs.diag_raw[j] + bs.diag_raw[j].T)
        assert np.abs(diag[j] - ref_d).max() <= 1e-10 * scale
        assert np.abs(sub[j] - bs.sub[j]).max() <= 1e-10 * scale
    assert np.allclose(t.diag[0], diag[0], rtol=1e-12)
