"""Row-slab sharding of grid operators across GPUs (one process per GPU).

SURVEY.md §8(e): the grid is cut into contiguous slabs of planes along its
slowest axis (z for 3-D, y for 2-D); every n-sized vector (basis blocks, C,
Z) is partitioned the same way while T_m, gamma and the eigen data stay
replicated.  Per Lanczos step the library (csrc/api.cu) exchanges one plane
per neighbour after each new basis block (NCCL send/recv) and sums each Gram
reduction across ranks (one ncclAllReduce of <= 192 doubles) before the
replicated coefficient solve.  This module holds the host-side pieces:
the partition, the NCCL communicator bootstrap over ``torch.distributed`` and
helpers to cut a global right-hand side into the local slab.
"""

import ctypes

import numpy as np

from . import _lib


def slab_partition(n_planes, nranks, rank):
    """Contiguous, balanced plane range [p0, p1) owned by ``rank``."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / world size")
    if n_planes < nranks:
        raise ValueError("fewer planes (%d) than ranks (%d)" % (n_planes, nranks))
    base, extra = divmod(n_planes, nranks)
    p0 = rank * base + min(rank, extra)
    p1 = p0 + base + (1 if rank < extra else 0)
    return p0, p1


def halo_plan(n_planes, nranks, rank):
    """Which planes a rank sends / receives each exchange (mirrors
    ``halo_exchange`` in csrc/api.cu): it sends its first owned plane to
    rank-1 and its last to rank+1, and receives the neighbours' boundary
    planes into its two halo planes."""
    p0, p1 = slab_partition(n_planes, nranks, rank)
    plan = {"own": (p0, p1), "send": {}, "recv": {}}
    if rank > 0:
        plan["send"][rank - 1] = p0
        plan["recv"][rank - 1] = p0 - 1
    if rank < nranks - 1:
        plan["send"][rank + 1] = p1 - 1
        plan["recv"][rank + 1] = p1
    return plan


def local_rows(c, grid, z_range):
    """Rows of a global n x s block owned by the slab z_range (x fastest)."""
    nxy = grid[0] * grid[1] if grid[2] > 1 else grid[0]
    z0, z1 = z_range
    return np.ascontiguousarray(np.asarray(c)[z0 * nxy:z1 * nxy])


class Communicator:
    """NCCL communicator for the library, bootstrapped through an existing
    ``torch.distributed`` process group (rank 0 creates the unique id and
    broadcasts it; every rank then calls kry_comm_init on its context)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self._id = None

    def unique_id(self):
        if self._id is None:
            buf = [None]
            if self.rank == 0:
                raw = ctypes.create_string_buffer(128)
                _lib.check(_lib.load().kry_nccl_unique_id(raw))
                buf[0] = bytes(raw.raw)
            self.dist.broadcast_object_list(buf, src=0, group=self.group)
            self._id = buf[0]
        return self._id

    def attach(self, ctx):
        uid = ctypes.create_string_buffer(self.unique_id(), 128)
        _lib.check(_lib.load().kry_comm_init(ctx.ptr, self.nranks, self.rank, uid))
        self._id = None  # a fresh id for the next communicator


class LoopbackGroup:
    """In-process transport for the sharded path (``kry_loop`` in
    csrc/api.cu): the P slab contexts of one process -- typically all on one
    GPU -- exchange halos and all-reduce their Gram partials through
    event-ordered device copies and a host rendezvous instead of NCCL.  The
    library runs exactly the code of the NCCL path (POST_NONE reductions,
    replicated post routines, halo planes), so the multi-rank solve can be
    exercised and parity-tested without a multi-GPU node.  Each rank must be
    driven from its own host thread (the library releases the GIL)."""

    def __init__(self, nranks):
        self.nranks = int(nranks)
        self.ptr = ctypes.c_void_p()
        _lib.check(_lib.load().kry_loop_create(self.nranks, ctypes.byref(self.ptr)))

    def comm(self, rank):
        return _LoopComm(self, rank)

    def close(self):
        if self.ptr is not None and self.ptr.value:
            _lib.load().kry_loop_destroy(self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _LoopComm:
    """Per-rank handle with the Communicator interface used by operators."""

    def __init__(self, group, rank):
        self.group = group
        self.rank = int(rank)
        self.nranks = group.nranks

    def attach(self, ctx):
        _lib.check(_lib.load().kry_comm_init_loopback(ctx.ptr, self.group.ptr, self.rank))


def run_ranks(nranks, fn):
    """Run ``fn(rank, comm)`` for every rank of a loopback group, one host
    thread per rank; returns the per-rank results (re-raises the first
    rank failure)."""
    import threading

    group = LoopbackGroup(nranks)
    out = [None] * nranks
    err = [None] * nranks

    def body(r):
        try:
            out[r] = fn(r, group.comm(r))
        except BaseException as e:  # noqa: B902 - reported below
            err[r] = e

    threads = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    import gc
    gc.collect()   # contexts of the finished solves go before their group
    group.close()
    for e in err:
        if e is not None:
            raise e
    return out
