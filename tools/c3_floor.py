"""Reference-algorithm self-noise on config 3: oracle with the CSR operator vs
the oracle with a reordered-summation operator (SURVEY §8(c) protocol)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from oracle import krymat_oracle as ko, problems as P
from tests.helpers import ReorderedOperator
cfg = P.build_config("c3")
t = time.time()
per = ko.solve_sylvester(ReorderedOperator(cfg["a"]), ReorderedOperator(cfg["b"]), cfg["c1"], cfg["c2"],
                         ko.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"]))
np.savez("/tmp/c3_perturbed.npz", history=np.array(per.history), iterations=per.iterations)
print("done", per.iterations, time.time() - t)
