import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1602_05033_b200 as kb
from paper_1602_05033_b200 import problems as PP
g = np.load("tests/golden/sylv1_lap40.npz")
a = PP.gen_fd2d("laplacian2d", 40)
sol = kb.solve_sylvester_one_sided(kb.SparseOperator(a), g["b"], g["c1"], g["c2"],
                                   kb.SolveOptions(tol=float(g["tol"]), max_m=300, storage="windowed"))
h = np.array([r[2] for r in sol.history]); r = g["history"][:, 2]
for i in range(len(h)):
    print(i + 1, "%.12e %.12e %.2e" % (h[i], r[i], abs(h[i] - r[i]) / r[i]))
