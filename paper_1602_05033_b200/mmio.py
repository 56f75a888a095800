"""Matrix Market files for the command line (reference ``mmio.py``).

Sparse matrices in coordinate format (``symmetric`` stores the lower
triangle), dense blocks in array format (column-major, as the format
prescribes); values with 17 significant digits so a write-then-read round
trip is exact in binary64.
"""

import numpy as np
import scipy.sparse as sp

from .errors import KrymatError


class MatrixMarketError(KrymatError):
    """Malformed Matrix Market content."""


def write_coordinate(path, a, symmetric=True):
    a = sp.coo_matrix(a)
    r, c, v = a.row, a.col, a.data
    if symmetric:
        low = r >= c
        r, c, v = r[low], c[low], v[low]
    with open(path, "w") as f:
        f.write("%%%%MatrixMarket matrix coordinate real %s\n"
                % ("symmetric" if symmetric else "general"))
        f.write("%d %d %d\n" % (a.shape[0], a.shape[1], v.size))
        for i, j, x in zip(r, c, v):
            f.write("%d %d %.16e\n" % (i + 1, j + 1, x))


def write_array(path, m):
    m = np.atleast_2d(np.asarray(m, dtype=float))
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix array real general\n")
        f.write("%d %d\n" % m.shape)
        np.savetxt(f, m.reshape(-1, order="F"), fmt="%.16e")


def _read(path):
    with open(path) as f:
        head = f.readline()
        if not head.startswith("%%MatrixMarket"):
            raise MatrixMarketError("%s: missing MatrixMarket header" % path)
        tok = [t.lower() for t in head.split()]
        if len(tok) < 5:
            raise MatrixMarketError("%s: incomplete header %r" % (path, head.strip()))
        body = [ln for ln in f if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:
        raise MatrixMarketError("%s: missing size line" % path)
    return tok, body[0].split(), body[1:]


def read_coordinate(path):
    """Sparse matrix (CSR) from a coordinate file (real, symmetric or general)."""
    tok, size, lines = _read(path)
    if tok[2] != "coordinate" or tok[3] not in ("real", "integer"):
        raise MatrixMarketError("%s: expected a real coordinate matrix" % path)
    nr, nc, nnz = (int(x) for x in size[:3])
    if len(lines) != nnz:
        raise MatrixMarketError("%s: expected %d entries, found %d" % (path, nnz, len(lines)))
    data = np.array([ln.split()[:3] for ln in lines], dtype=float).reshape(-1, 3)
    i = data[:, 0].astype(np.int64) - 1
    j = data[:, 1].astype(np.int64) - 1
    v = data[:, 2]
    if tok[4] == "symmetric":
        off = i != j
        i, j, v = np.concatenate([i, j[off]]), np.concatenate([j, i[off]]), \
            np.concatenate([v, v[off]])
    elif tok[4] != "general":
        raise MatrixMarketError("%s: unsupported symmetry %r" % (path, tok[4]))
    return sp.coo_matrix((v, (i, j)), shape=(nr, nc)).tocsr()


def read_array(path):
    """Dense matrix from an array file (column-major values)."""
    tok, size, lines = _read(path)
    if tok[2] != "array":
        raise MatrixMarketError("%s: expected an array matrix" % path)
    nr, nc = (int(x) for x in size[:2])
    vals = np.array([float(ln.split()[0]) for ln in lines])
    if vals.size != nr * nc:
        raise MatrixMarketError("%s: expected %d values, found %d" % (path, nr * nc, vals.size))
    return vals.reshape((nr, nc), order="F")
