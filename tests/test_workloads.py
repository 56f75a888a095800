"""CPU: the package's workload generators (paper_1602_05033_b200.problems,
used by bench.py) reproduce the reference's own CSR matrices bit for bit
(digests recorded from the reference generators in tests/golden/*.npz), and
the device stencil constants equal the CSR entries."""

import os

import numpy as np
import pytest

from oracle import problems as OP
from paper_1602_05033_b200 import problems as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


@pytest.mark.parametrize("name,builder,key", [
    ("c1", lambda: P.gen_fd2d("laplacian2d", 100), "digest_a"),
    ("c2", lambda: P.laplacian3d(50), "digest_a"),
    ("c3", lambda: P.gen_fd2d("varcoef2d", 300), "digest_a"),
    ("c3", lambda: P.laplacian3d(40), "digest_b"),
])
def test_generators_match_reference_digests(name, builder, key):
    assert OP.csr_digest(builder()) == str(gold(name)[key])


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_workload_inputs_match_oracle_builders(name):
    w = P.workload(name)
    o = OP.build_config(name)
    for k in ("c", "c1", "c2"):
        if k in o:
            assert np.array_equal(w[k], o[k])
    assert w["tol"] == o["tol"] and w["max_m"] == o["max_m"]


@pytest.mark.parametrize("dims,n", [(3, 7), (3, 11), (2, 9), (2, 30)])
def test_stencil_constants_equal_csr_entries(dims, n):
    cd, co = P.laplacian_constants(dims, n)
    a = P.laplacian3d(n) if dims == 3 else P.gen_fd2d("laplacian2d", n)
    # Dirichlet cuts couplings, not the diagonal: every diagonal entry is cd
    assert np.all(a.diagonal() == cd)
    off = a.copy()
    off.setdiag(0.0)
    off.eliminate_zeros()
    assert np.all(off.data == co)


def test_large_workloads_shapes_without_matrix():
    w = P.workload("c5", with_matrix=False)
    assert w["a"] is None and w["c"].shape == (4_000_000, 4)
    assert w["grid_a"] == (2000, 2000)
