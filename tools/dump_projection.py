"""Diagnostics: run a config's pass 1 on the GPU and save the device's own
projected blocks (kry_get_projection), gamma and history to gpurun_out/, so
the residual history can be re-evaluated offline on the device's T_m and
compared block by block with the reference's.

    python tools/dump_projection.py c5
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1602_05033_b200 as kb  # noqa: E402
from paper_1602_05033_b200 import _lib  # noqa: E402
from paper_1602_05033_b200.solvers import _Pass1  # noqa: E402

OUT = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")


def main(name):
    cfg, op, _ = bench.build_problem(name)
    opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
    lib = _lib.load()
    p1 = _Pass1(op, np.ascontiguousarray(cfg["c"]), opts)
    hist = np.zeros((opts.max_m + 1, 5))
    nh, its, reason = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    rel = ctypes.c_double(0.0)
    lib.kry_solve_lyap_pass1(p1.ctx.ptr, opts.tol, opts.max_m, 1, _lib.as_dptr(hist),
                             ctypes.byref(nh), ctypes.byref(its), ctypes.byref(rel),
                             ctypes.byref(reason))
    m = ctypes.c_int(0)
    s = p1.s
    cap = opts.max_m + 4
    draw = np.zeros(cap * s * s)
    dsym = np.zeros(cap * s * s)
    off = np.zeros(cap * s * s)
    sub = np.zeros(cap * s * s)
    _lib.check(lib.kry_get_projection(p1.ctx.ptr, ctypes.byref(m), _lib.as_dptr(draw),
                                      _lib.as_dptr(dsym), _lib.as_dptr(off), _lib.as_dptr(sub)))
    mm = m.value
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "proj_%s.npz" % name),
                        diag=dsym[:mm * s * s].reshape(mm, s, s),
                        sub=sub[:mm * s * s].reshape(mm, s, s), gamma=p1.gamma,
                        beta2=p1.beta2, history=hist[:nh.value])
    p1.ctx.close()
    print("saved", mm, "blocks", flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
