import sys; sys.path.insert(0, ".")
import numpy as np
import paper_1602_05033_b200 as kb
from oracle import problems as P
g = np.load("tests/golden/c3.npz")
cfg = P.build_config("c3")
sol = kb.solve_sylvester_two_sided(kb.SparseOperator(cfg["a"]), kb.SparseOperator(cfg["b"]), cfg["c1"], cfg["c2"],
                                   kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed"))
h = np.array([r[2] for r in sol.history]); hr = g["history"][:, 2]
rel = np.abs(h - hr) / hr
np.save("gpurun_out/c3_hist_gpu.npy", h)
for m in [1, 5, 10, 20, 50, 100, 150, 200, 250, 300, 350, 400, 450, 500, 550, 600, 650, 681]:
    print(m, hr[m-1], h[m-1], rel[m-1])
print("worst", rel.max(), rel.argmax() + 1)
