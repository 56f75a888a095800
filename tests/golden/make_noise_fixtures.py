"""Noise-floor fixtures for the chaotic / long configs.

Input: the reference block sequences and their surrogate histories written by
make_golden_blocks.py (``lanczos`` + ``residuals`` stages) for the plain run
(variant ``csr``) and an ensemble of variants of the SAME reference
algorithm: reordered SpMM summations (``upd``, ``ldu``, ``dlu``, ``lud``,
``rev``) and the QR of new blocks done by Cholesky QR twice (``cholqr*``,
the QR algorithm the device uses).  Output ``tests/golden/<cfg>_noise.npz``:

* ``surrogate``: the plain run's history (the paper's formula on a dense
  eigendecomposition of the reference's own T_m at every m);
* ``env``: per m, max over the ensemble of |rel_variant - rel_plain|;
* ``variants``, ``variant_iters`` (first m below tol per variant).

The test floor is 2 x the running maximum of ``env`` (an 8-member ensemble
envelope underestimates the spread of a chaotic deviation; the factor 2 is
that allowance).  Test infrastructure only (build container).

    python tests/golden/make_noise_fixtures.py c3 /tmp/gt upd ldu dlu lud rev cholqr cholqr-upd cholqr-dlu
    python tests/golden/make_noise_fixtures.py --golden-base=/tmp/gt/lapack/c5_blocks_csr_hist.npz \
        c5 /tmp/gt upd ldu dlu cholqr cholqr-upd
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main(cfg, src, variants, golden_base=None):
    """``golden_base``: the plain run's history evaluated with LAPACK (stored
    as the golden "surrogate"); the ensemble deviations are always taken
    between runs evaluated the same way (files in ``src``)."""
    base = np.load(os.path.join(src, "%s_blocks_csr_hist.npz" % cfg))["surrogate_history"]
    tol = float(np.load(os.path.join(src, "%s_blocks_csr.npz" % cfg))["tol"])
    devs, iters = [], []
    for v in variants:
        h = np.load(os.path.join(src, "%s_blocks_%s_hist.npz" % (cfg, v)))["surrogate_history"]
        n = min(len(h), len(base))
        dv = np.abs(h[:n] - base[:n])
        # strided variant histories (NaN between samples): the deviation at an
        # unsampled m is bounded by the larger of its sampled neighbours
        have = np.nonzero(np.isfinite(dv))[0]
        if len(have) < n:
            nxt = np.searchsorted(have, np.arange(n))
            prv = np.clip(nxt - 1, 0, len(have) - 1)
            nxt = np.clip(nxt, 0, len(have) - 1)
            dv = np.where(np.isfinite(dv), dv, np.maximum(dv[have[prv]], dv[have[nxt]]))
        devs.append(dv)
        below = np.nonzero(h <= tol)[0]
        iters.append(int(below[0]) + 1 if len(below) else -1)
    n = min(len(d) for d in devs)
    env = np.max([d[:n] for d in devs], axis=0)
    out = os.path.join(HERE, "%s_noise.npz" % cfg)
    gold = base if golden_base is None else np.load(golden_base)["surrogate_history"]
    np.savez_compressed(out, surrogate=gold, env=env, variants=np.array(variants),
                        variant_iters=np.array(iters))
    print("wrote", out, "max rel env", float(np.max(env / base[:n])), "iters", iters)


if __name__ == "__main__":
    args = sys.argv[1:]
    gb = None
    if args and args[0].startswith("--golden-base="):
        gb = args[0].split("=", 1)[1]
        args = args[1:]
    main(args[0], args[1], args[2:], gb)
