import faulthandler, sys
faulthandler.enable()
sys.path.insert(0, ".")
import numpy as np, scipy.sparse as sp
import paper_1602_05033_b200 as kb
c = np.zeros((6, 1)); c[0] = 1.0
op = kb.SparseOperator(sp.diags([-1.0] * 6).tocsr())
print("kind", op.kind, op.stencil.grid, op.stencil.slab, op.n, flush=True)
sol = kb.solve_lyapunov(op, c, kb.SolveOptions(tol=1e-10, max_m=5))
print("ok", sol.iterations)
