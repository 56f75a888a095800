"""Self-noise of the reference ALGORITHM on config 3 (SURVEY.md §8(c) protocol).

Runs the oracle restatement (pinned to the reference by tests/test_oracle.py)
with a reordered-summation operator (U v + D v) + L v instead of the CSR
product; the difference to the reference's own history (tests/golden/c3.npz)
is the roundoff floor any implementation must be judged against.  ~35 min on
one CPU core:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_selfnoise.py
"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import numpy as np  # noqa: E402
from oracle import krymat_oracle as ko, problems as P  # noqa: E402
from tests.helpers import ReorderedOperator  # noqa: E402

if __name__ == "__main__":
    cfg = P.build_config("c3")
    t = time.time()
    per = ko.solve_sylvester(ReorderedOperator(cfg["a"]), ReorderedOperator(cfg["b"]),
                             cfg["c1"], cfg["c2"],
                             ko.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"]))
    np.savez_compressed(os.path.join(HERE, "c3_selfnoise.npz"),
                        history=np.array(per.history), iterations=per.iterations)
    print("done", per.iterations, time.time() - t)
