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
