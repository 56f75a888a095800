import sys; sys.path.insert(0, ".")
import numpy as np
import paper_1602_05033_b200 as kb
from oracle import krymat_oracle as ko, problems as P
a, b = P.varcoef2d(11), P.laplacian3d(5)
rng = np.random.default_rng(2)
c1, c2 = rng.standard_normal((121, 2)), rng.standard_normal((125, 2))
sol = kb.solve_sylvester_two_sided(kb.SparseOperator(a), kb.SparseOperator(b), c1, c2, kb.SolveOptions(tol=1e-8, max_m=100))
ref = ko.solve_sylvester(ko.SparseOperator(a), ko.SparseOperator(b), c1, c2, ko.SolveOptions(tol=1e-8, max_m=100))
h = np.array([r[2] for r in sol.history]); hr = np.array([r[2] for r in ref.history])
print(sol.iterations, ref.iterations)
for i in range(len(h)):
    print(i + 1, hr[i], h[i], abs(h[i] - hr[i]) / hr[i], abs(h[i]-hr[i]))
print("factor", ko.factor_distance(sol.z1, ref.z1, sol.z2, ref.z2))
