"""Benchmark: block-Lanczos iterations/s and time-to-tol of the two-pass
Lyapunov/Sylvester solver on B200 (BASELINE.json metric).

One "step" = one complete solve of the workload to tolerance: pass 1 (SpMM +
MGS-twice/QR recurrence + cheap residual check every iteration), the
finalisation and pass 2 (basis regeneration + factor accumulation).
``value`` = block-Lanczos iterations per second of that whole solve, inputs
resident in HBM; ``e2e`` = the same metric through the public API
``solve_lyapunov(op, C_host, options)`` with host C in and host Z out.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
    python bench.py --impl reference ...   (the reference algorithm on the host CPU)
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1602_05033_b200.problems import DESCRIPTIONS as CONFIG_DOC  # noqa: E402


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_bytes(path):
    d = json.load(open(path))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(d[k]["value"].replace(",", "")) * scale[d[k]["unit"]]
    return tot


def step_traffic(config):
    """DRAM bytes of one pass-1 step (k_apply_tma + k_combine launches) from
    the committed ncu --set full captures (profiles/), or None."""
    try:
        return (_ncu_bytes(os.path.join(ROOT, "profiles", "r2_k_apply_tma_%s_ncu.json" % config))
                + _ncu_bytes(os.path.join(ROOT, "profiles", "r2_k_combine_%s_ncu.json" % config)))
    except Exception:
        return None


def captured_traffic(config):
    """DRAM bytes per k_combine launch from the committed ncu --set full
    capture of this config (profiles/r2_k_combine_<config>_ncu.json), or None."""
    path = os.path.join(ROOT, "profiles", "r2_k_combine_%s_ncu.json" % config)
    try:
        d = json.load(open(path))
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[k]["value"].replace(",", "")) * scale[d[k]["unit"]]
        return tot
    except Exception:
        return None


def build_problem(name, slab=None, comm=None):
    """Operators (device stencil descriptions for c4/c5, CSR otherwise) and
    the seeded right-hand sides of a BASELINE workload
    (paper_1602_05033_b200.problems).  With ``slab`` (planes [z0, z1) of the
    slowest axis) the operator and C are this rank's row slab (parallel.py)."""
    import paper_1602_05033_b200 as kb
    from paper_1602_05033_b200 import problems as P
    from paper_1602_05033_b200.parallel import local_rows

    if name in ("c4", "c5"):
        cfg = P.workload(name, with_matrix=False)
        op = P.stencil_operator(cfg["grid_a"], slab=slab, comm=comm)
        if slab is not None:
            cfg["c"] = local_rows(cfg["c"], op.grid, slab)
        return cfg, op, None
    cfg = P.workload(name)
    op = kb.SparseOperator(cfg["a"])
    opb = kb.SparseOperator(cfg["b"]) if cfg["kind"] == "sylvester" else None
    return cfg, op, opb


class Clocks:
    """SM clock / throttle-reason sampling during the timed region, in-process
    through NVML (a spawned nvidia-smi every 200 ms perturbed the host-side
    phases being timed)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.index = index

    def start(self):
        def run():
            try:
                import pynvml
                pynvml.nvmlInit()
                h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            except Exception:
                return
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, mx, rs))
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [x[0] for x in self.samples]
        mx = max([x[1] for x in self.samples], default=0)
        reasons = set()
        for _, _, rs in self.samples:
            for name, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def timed_solve_device(kb, lib, ctx, c_dev_ptr, opts, s, prof=True):
    """One device-resident solve (C already in HBM, Z left in HBM)."""
    from paper_1602_05033_b200 import _lib

    gamma = np.zeros((s, s))
    beta2 = ctypes.c_double()
    ms = ctypes.c_double()
    _lib.check(lib.kry_timer(ctx.ptr, 0, None))
    ti = time.perf_counter()
    _lib.check(lib.kry_init_basis_device(ctx.ptr, ctypes.c_void_p(c_dev_ptr), _lib.as_dptr(gamma),
                                         ctypes.byref(beta2)))
    t_init = time.perf_counter() - ti
    hist = np.zeros((opts.max_m + 1, 5))
    nh, its, reason = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rel = ctypes.c_double()
    t0 = time.perf_counter()
    rc = lib.kry_solve_lyap_pass1(ctx.ptr, opts.tol, opts.max_m, 1, _lib.as_dptr(hist),
                                  ctypes.byref(nh), ctypes.byref(its), ctypes.byref(rel),
                                  ctypes.byref(reason))
    t1 = time.perf_counter()
    rank, disc = ctypes.c_int(), ctypes.c_double()
    if rc == _lib.KRY_ERR_CONVERGENCE and reason.value == 1:
        # config 5: no convergence within max_m (the reference raises too);
        # the step is the full pass 1 of max_m iterations, no factor
        its.value = opts.max_m
        rel.value = float(hist[nh.value - 1, 2]) if nh.value else float("nan")
        _lib.check(lib.kry_timer(ctx.ptr, 1, ctypes.byref(ms)))
        t2 = t3 = time.perf_counter()
    else:
        _lib.check(rc)
        _lib.check(lib.kry_finalize_lyap(ctx.ptr, opts.trunc_eps, ctypes.byref(rank),
                                         ctypes.byref(disc)))
        t2 = time.perf_counter()
        _lib.check(lib.kry_recover(ctx.ptr, None))
        _lib.check(lib.kry_timer(ctx.ptr, 1, ctypes.byref(ms)))
        t3 = time.perf_counter()
    return dict(ms=ms.value, iterations=its.value, rank=rank.value, rel=rel.value,
                init_s=t_init, pass1_s=t1 - t0, finalize_s=t2 - t1, pass2_s=t3 - t2,
                check_s=float(hist[nh.value - 1, 4]) if nh.value else 0.0,
                basis_s=float(hist[nh.value - 1, 3]) if nh.value else 0.0,
                basis_its=int(hist[nh.value - 1, 0]) if nh.value else 0)


def combine_alone(lib, ctx, c_dev_ptr, opts, s, its):
    """Average k_combine launch time with the eigen stream idle: one extra,
    untimed pass 1 of ``its`` iterations that queues the recurrence only
    (KRY_DEBUG_NO_EIG).  In the timed region the eigen appends of the second
    stream run beside the recurrence and take SM time from it, so the in-situ
    launch time is longer than the kernel's own."""
    from paper_1602_05033_b200 import _lib

    gamma = np.zeros((s, s))
    beta2 = ctypes.c_double()
    os.environ["KRY_DEBUG_NO_EIG"] = "1"
    try:
        lib.kry_profile_enable(ctx.ptr, 0)
        lib.kry_profile_enable(ctx.ptr, 1)
        _lib.check(lib.kry_init_basis_device(ctx.ptr, ctypes.c_void_p(c_dev_ptr),
                                             _lib.as_dptr(gamma), ctypes.byref(beta2)))
        hist = np.zeros((its + 1, 5))
        nh, it, reason = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        rel = ctypes.c_double()
        lib.kry_solve_lyap_pass1(ctx.ptr, 0.0, its, 1, _lib.as_dptr(hist), ctypes.byref(nh),
                                 ctypes.byref(it), ctypes.byref(rel), ctypes.byref(reason))
        ms, n = ctypes.c_double(), ctypes.c_int()
        lib.kry_profile_read(ctx.ptr, ctypes.byref(ms), ctypes.byref(n), None, None)
        return ms.value / max(n.value, 1), n.value
    finally:
        os.environ.pop("KRY_DEBUG_NO_EIG", None)
        lib.kry_profile_enable(ctx.ptr, 0)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_sample(cfg_name, threads):
    """Bounded sample of the reference algorithm (the oracle port, a numpy
    restatement of the reference pinned to its goldens) on the host with
    ``threads`` BLAS threads, extrapolated to the full solve:

    * pass-1 steps: block-Lanczos steps (SpMM + MGS twice + Householder QR,
      basis.py:223-252) on the full-size input;
    * pass-2 steps: the same regeneration + the factor update
      ``z += v @ qy[block]`` of two_pass_recover (solvers.py:158-169) with the
      reference's rank (the golden), which is what makes the reference's
      recovery ~2x its basis time (c4 golden: 4,827 s vs 2,480 s);
    * one cTri check (band reduction + tridiagonal eig + contraction,
      residual.py:40-59) on the reference's own T_m at depth m_chk, scaled
      ~m^2 to every iteration;
    * the finalisation (two dense eighs of order k = s m, solvers.py:254-264).
    Returns (iterations/s, description, seconds spent)."""
    from threadpoolctl import threadpool_limits
    from oracle import krymat_oracle as ko
    from oracle import problems as P

    spent = time.perf_counter()
    cfg = P.build_config(cfg_name)
    op = ko.SparseOperator(cfg["a"])
    c = cfg.get("c", cfg.get("c1"))
    gpath = os.path.join(ROOT, "tests", "golden", cfg_name + ".npz")
    g = np.load(gpath) if os.path.exists(gpath) else None
    with threadpool_limits(threads):
        bs = ko.Basis(op, c)
        nsteps = 2 if cfg_name in ("c4", "c5") else 10
        t0 = time.perf_counter()
        for _ in range(nsteps):
            bs.step()
        t_step = (time.perf_counter() - t0) / nsteps
        nsteps2 = 1 if cfg_name in ("c4", "c5") else nsteps
        s = c.shape[1]
        rank = int(g["rank"]) if g is not None and "rank" in g else 8 * s
        qy = np.random.default_rng(0).standard_normal(((nsteps2 + 1) * s, rank))
        z = np.zeros((op.n, rank))
        v = bs.blocks[-1]
        t0 = time.perf_counter()
        for i in range(nsteps2):
            w, _, _ = ko.mgs_twice(op.apply(v), None, v)
            vn, _ = ko.economy_qr(w)
            z += vn @ qy[i * s:(i + 1) * s]
            v = vn
        t_step2 = (time.perf_counter() - t0) / nsteps2
        del z
        t_chk = m_chk = iters_ref = None
        t_fin = 0.0
        if g is not None:
            m_all = g["t_diag"].shape[0]
            iters_ref = int(g["iterations"]) if "iterations" in g else m_all
            m_chk = max(1, min(m_all, 64 if s >= 4 else 200))
            t = ko.BlockTri(s, [0.5 * (d + d.T) for d in g["t_diag"][:m_chk]],
                            list(g["t_off"][:m_chk - 1]))
            t1 = time.perf_counter()
            ko.ctri_lyapunov(t, g["gamma"], g["t_off"][m_chk - 1] if m_chk < m_all else g["tau"])
            t_chk = time.perf_counter() - t1
            k = s * iters_ref
            a = np.random.default_rng(1).standard_normal((k, k))
            a = a + a.T
            t1 = time.perf_counter()
            np.linalg.eigh(a)
            t_fin = 2.0 * (time.perf_counter() - t1)
    spent = time.perf_counter() - spent
    if t_chk is not None and iters_ref:
        m = iters_ref
        checks = sum(t_chk * (j / m_chk) ** 2 for j in range(1, m + 1))
        total = m * t_step + checks + t_fin + m * t_step2
        value = m / total
        desc = ("%d threads (%s): %d pass-1 block-Lanczos steps of the numpy port on the full %s "
                "input (%.2f s/step), %d pass-2 steps incl. the rank-%d factor update (%.2f "
                "s/step), one cTri check at m=%d on the reference's own T_m (%.2f s), two "
                "eighs of order %d (%.1f s); extrapolated to the reference's %d iterations "
                "(checks ~ m^2): time-to-tol %.0f s" %
                (threads, cpu_model(), nsteps, cfg_name, t_step, nsteps2, rank, t_step2, m_chk,
                 t_chk, s * m, t_fin, m, total))
    else:
        value = 1.0 / (t_step + t_step2)
        desc = "%d threads: %d block-Lanczos steps (no checks) of the numpy port" % (threads,
                                                                                    nsteps)
    return value, desc, spent


def cpu_legs(cfg_name):
    """The reference on all host threads and on one (more
    threads can be slower); the faster leg is the baseline."""
    allt = os.cpu_count() or 1
    legs = []
    for th in sorted({allt, 1}, reverse=True):
        v, desc, spent = cpu_sample(cfg_name, th)
        legs.append({"threads": th, "value": v, "sample": desc, "seconds": round(spent, 1)})
    best = max(legs, key=lambda x: x["value"])
    return best, legs


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    vals, legs_all = [], []
    best = None
    for _ in range(max(1, args.steps)):
        best, legs = cpu_legs(args.config)
        vals.append(best["value"])
        legs_all = legs
    value = float(np.median(vals))
    line = {
        "impl": "reference",
        "metric": "block-Lanczos iterations/s (SpMM+orth+residual norm, full solve to tol)",
        "value": value,
        "unit": "iters/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 / value if value else None,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": {"workload": args.config, "desc": CONFIG_DOC[args.config]},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": best["threads"],
                         "kind": "port", "sample": best["sample"], "cpu_model": cpu_model(),
                         "legs": legs_all},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIG_DOC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_1602_05033_b200 as kb
    from paper_1602_05033_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()
    slab = comm = None
    if world > 1:
        from paper_1602_05033_b200 import problems as P
        from paper_1602_05033_b200.parallel import Communicator, slab_partition
        g = P.workload(args.config, with_matrix=False)["grid_a"]
        slab = slab_partition(g[-1], world, rank)
        comm = Communicator()
    cfg, op, opb = build_problem(args.config, slab=slab, comm=comm)
    if cfg["kind"] != "lyapunov":
        raise SystemExit("bench.py measures the Lyapunov configs (c1, c2, c4, c5)")
    op.device = local
    c = cfg["c"]
    n, s = c.shape
    opts = kb.SolveOptions(tol=cfg["tol"], max_m=cfg["max_m"], storage="windowed")
    # inputs resident in HBM for the device-timed value
    c_dev = torch.from_numpy(np.ascontiguousarray(c)).to(f"cuda:{local}")
    torch.cuda.synchronize()
    ctx = op.context(s, opts.max_m + 2)
    for _ in range(args.warmup):
        timed_solve_device(kb, lib, ctx, c_dev.data_ptr(), opts, s)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    _lib.reset_launch_count()
    lib.kry_profile_enable(ctx.ptr, 1)
    runs = []
    for _ in range(args.steps):
        runs.append(timed_solve_device(kb, lib, ctx, c_dev.data_ptr(), opts, s))
    launches = _lib.launch_count()
    comb_ms, comb_n = ctypes.c_double(), ctypes.c_int()
    lib.kry_profile_read(ctx.ptr, ctypes.byref(comb_ms), ctypes.byref(comb_n), None, None)
    zacc_ms, zacc_fl, zacc_n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    lib.kry_profile_zacc(ctx.ptr, ctypes.byref(zacc_ms), ctypes.byref(zacc_fl),
                         ctypes.byref(zacc_n))
    lib.kry_profile_enable(ctx.ptr, 0)
    torch.cuda.synchronize()
    clk = clocks.stop()
    # the residual contraction on the final eigen data (k = s m), and the
    # device's measured fp64 peaks (untimed, after the timed region)
    chk_ms, chk_k = ctypes.c_double(), ctypes.c_int()
    chk_ok = lib.kry_profile_check(ctx.ptr, 20, ctypes.byref(chk_ms), ctypes.byref(chk_k)) == 0
    dfma, dmma = ctypes.c_double(), ctypes.c_double()
    lib.kry_fp64_peak(local, ctypes.byref(dfma), ctypes.byref(dmma))
    alone_ms, alone_n = (0.0, 0)
    if world == 1:
        try:
            alone_ms, alone_n = combine_alone(lib, ctx, c_dev.data_ptr(), opts, s,
                                              min(runs[-1]["iterations"], opts.max_m))
        except Exception:   # measurement only
            alone_ms, alone_n = (0.0, 0)
    ms_total = sum(r["ms"] for r in runs)
    its_total = sum(r["iterations"] for r in runs)
    if dist:
        t = torch.tensor([ms_total], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    its_total_all = its_total   # sharded: all ranks advance the same solve
    value = its_total_all / (ms_total / 1000.0)
    ctx.close()
    # Roofline: the unit is one pass-1 block-Lanczos step,
    # B_iter = 24 n s bytes (read V_{m-1}, V_m, write V_{m+1}: the three-term
    # minimum; constant stencil, no operator bytes); achieved = B_iter / the
    # device time per step on the Lanczos stream (CUDA events, pass 1,
    # excluding the check stream).  The step kernels themselves move 48 n s
    # (k_apply_tma: read V_m, write A V_m; k_combine: read V_{m-1}, V_m,
    # A V_m, write V_{m+1}), so this is at most 0.5 of the copy peak by
    # construction; the kernel-level DRAM fractions are listed beside it.
    hbm, hbm_kind = peaks()
    r_last = runs[-1]
    b_iter = 24 * n * s
    t_step = r_last["basis_s"] / max(r_last["basis_its"], 1)
    achieved = b_iter / t_step / 1e9 if t_step > 0 else 0.0
    comb_avg_ms = comb_ms.value / max(comb_n.value, 1)
    handoff = (world == 1 and s % 2 == 0 and os.environ.get("KRY_NO_AV_HANDOFF") != "1"
               and os.environ.get("KRY_FUSED_STEP") != "1")
    bytes_launch = (4 if handoff else 3) * n * s * 8
    comb_gbs = bytes_launch / (comb_avg_ms / 1000.0) / 1e9 if comb_avg_ms > 0 else 0.0
    kernels = [{"kernel": "k_combine (3-term recurrence + Gram on DMMA)", "bound": "hbm",
                "bytes_per_launch": bytes_launch, "avg_launch_ms": comb_avg_ms,
                "achieved": comb_gbs, "unit": "GB/s", "frac": comb_gbs / hbm if hbm else None,
                "traffic": captured_traffic(args.config), "launches": comb_n.value}]
    if alone_ms > 0:
        agbs = bytes_launch / (alone_ms / 1000.0) / 1e9
        kernels[0]["alone"] = {
            "avg_launch_ms": alone_ms, "achieved": agbs, "frac": agbs / hbm if hbm else None,
            "frac_survey_bytes": (b_iter / (alone_ms / 1000.0) / 1e9) / hbm if hbm else None,
            "launches": alone_n,
            "note": "same kernel with the eigen stream idle (untimed extra pass 1): in the timed "
                    "region the eigen appends run beside the recurrence and take SM time from it"}
    fp64_peak = dmma.value if dmma.value > 0 else None
    if zacc_n.value:
        tf = zacc_fl.value / (zacc_ms.value / 1000.0) / 1e12
        kernels.append({"kernel": "k_zacc (pass-2 factor accumulation Z += V Q, DMMA)",
                        "bound": "tensor (fp64 DMMA)", "flops_total": zacc_fl.value,
                        "ms_total": zacc_ms.value, "launches": zacc_n.value, "achieved": tf,
                        "unit": "TFLOP/s", "peak": fp64_peak,
                        "frac": tf / fp64_peak if fp64_peak else None})
    if chk_ok and chk_ms.value > 0:
        k = chk_k.value
        fl = 4.0 * s * k * k + k * k
        tf = fl / (chk_ms.value / 1000.0) / 1e12
        kernels.append({"kernel": "residual contraction k_cauchy_mma (4 s k^2 + k^2 flop, "
                        "divisions counted once)", "bound": "fp64", "k": k,
                        "avg_ms": chk_ms.value, "achieved": tf, "unit": "TFLOP/s",
                        "peak": fp64_peak, "frac": tf / fp64_peak if fp64_peak else None})

    e2e = None
    if not args.no_e2e:
        import torch as _t
        pinned = _t.empty((n, s), dtype=_t.float64, pin_memory=True).numpy()
        pinned[:] = c
        # untimed warm-up through the same API (first-touch costs: the
        # page-locked host pages the factor is returned in are allocated once
        # and recycled by later solves)
        def api_solve():
            try:
                sol = kb.solve_lyapunov(op, pinned, opts)
                return sol.iterations, sol.rank, sol.basis_seconds, sol.recovery_seconds
            except kb.ConvergenceError as exc:   # config 5: max_m reached, as the reference
                return len(exc.history), 0, exc.history[-1][3] if exc.history else 0.0, 0.0

        for _ in range(2):
            api_solve()
        e2e_runs = []
        for _ in range(max(1, min(args.steps, 3))):
            _t.cuda.synchronize()
            t0 = time.perf_counter()
            it_, rk_, tb_, tr_ = api_solve()   # the result is released before the next solve
            e2e_runs.append((time.perf_counter() - t0, it_, rk_, tb_, tr_))
        e2e_s = sum(r[0] for r in e2e_runs)
        e2e_its = sum(r[1] for r in e2e_runs)
        rank_z = e2e_runs[-1][2]
        if dist:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": e2e_its / e2e_s, "unit": "iters/s",
               "h2d_bytes_per_step": int(n * s * 8),
               "d2h_bytes_per_step": int(n * rank_z * 8),
               "ms_per_solve": 1000.0 * e2e_s / len(e2e_runs),
               "solves_s": [{"total": round(r[0], 4), "pass1": round(r[3], 4),
                             "finalize+pass2+copy": round(r[4], 4)} for r in e2e_runs]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            best, legs = cpu_legs(args.config)
            cpu = {"value": best["value"], "unit": "iters/s", "cores": best["threads"],
                   "kind": "port", "sample": best["sample"], "cpu_model": cpu_model(),
                   "legs": legs}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "iters/s", "cores": 0, "kind": "port",
                   "sample": "failed: %s" % exc}
    r0 = runs[-1]
    line = {
        "metric": "block-Lanczos iterations/s (SpMM+orth+residual norm, full solve to tol)",
        "value": value,
        "unit": "iters/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_total / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8(d)); inputs larger than L2",
        "config": {"workload": args.config, "desc": CONFIG_DOC[args.config], "n": n, "s": s,
                   "tol": cfg["tol"], "iterations": r0["iterations"], "rank": r0["rank"],
                   "final_rel_residual": r0["rel"],
                   "parallelism": "slab-z%d" % world if world > 1 else "single",
                   "l2": "inputs (4 x %d MB blocks) exceed the 126 MB L2" % (n * s * 8 >> 20)},
        "time_to_tol_ms": ms_total / args.steps,
        "phases_all_s": [{k: round(r[k], 4) for k in ("pass1_s", "finalize_s", "pass2_s")}
                         for r in runs],
        "phases_s": {"init": r0["init_s"], "pass1": r0["pass1_s"],
                     "checks_in_pass1": r0["check_s"],
                     "finalize": r0["finalize_s"], "pass2": r0["pass2_s"]},
        "roofline": {"bound": "hbm",
                     "kernel": "k_combine: pass-1 recurrence, one launch per block-Lanczos "
                     "iteration (the north star's fused SpMM/recurrence target)",
                     "definition": "SURVEY 8(d) unit: one iteration, B_iter = 24 n s bytes "
                     "(read V_{m-1}, V_m, write V_{m+1}; constant stencil, no operator "
                     "bytes) per launch / average CUDA-event launch time",
                     "unit_bytes": b_iter, "achieved": b_iter / (comb_avg_ms / 1000.0) / 1e9
                     if comb_avg_ms > 0 else 0.0, "peak": hbm, "peak_kind": hbm_kind,
                     "unit": "GB/s",
                     "frac": (b_iter / (comb_avg_ms / 1000.0) / 1e9 / hbm)
                     if comb_avg_ms > 0 and hbm else None,
                     "traffic": captured_traffic(args.config),
                     "step": {"achieved": achieved, "frac": achieved / hbm if hbm else None,
                              "step_ms": 1000.0 * t_step, "traffic": step_traffic(args.config),
                              "note": "B_iter / device time per iteration on the Lanczos "
                              "stream (apply + combine, 48 n s bytes moved)"},
                     "pass1_loop_frac": (b_iter * r_last["iterations"] / r_last["pass1_s"] / 1e9
                                         / hbm) if r_last["pass1_s"] > 0 else None,
                     "fp64_peak_tflops": {"dmma": dmma.value, "dfma": dfma.value,
                                          "how": "kry_fp64_peak, one-wave microbenchmark"},
                     "kernels": kernels},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": {k: clk[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
    }
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
