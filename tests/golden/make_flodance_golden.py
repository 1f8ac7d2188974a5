"""Golden vectors for FLODANCE from the UNMODIFIED reference (`oocdet.flodance`, 0.1.0).

Run in the build container, where /root/reference is mounted (it is not on the GPU box):

    python tests/golden/make_flodance_golden.py

Inputs are prefix sequences computed here by the oracle (the reference's own memdet algorithm,
oracle/memdet_oracle.py) on seeded BASELINE-family Gram matrices, plus a synthetic power-law
sequence; the reference fits and extrapolates each.  Only the reference's outputs are stored
(tests/golden/flodance.npz + flodance.json).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import memdet_oracle as O  # noqa: E402
from paper_2503_04424_b200 import gen  # noqa: E402


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from oocdet import flodance as F  # the reference

    seqs = {
        "rbf600": O.memdet_cholesky(gen.rbf(600, seed=11), 2)[0],
        "ntk500": O.memdet_cholesky(gen.ntk_like(500, 1000, 0.75, seed=12), 2)[0],
        "wishart400": O.memdet_cholesky(gen.spd_wishart(400, 400, seed=13, shift=1e-3), 1)[0],
    }
    j = np.arange(1, 801, dtype=np.float64)
    # synthetic: ell_n = n (2 - 0.7 log(n!) / n^2 + 0.1 (1 - 1/n)) + small deterministic wiggle
    from scipy.special import gammaln
    seqs["powerlaw800"] = j * (2.0 + 0.1 * (1 - 1 / j) - 0.7 * gammaln(j + 1) / j ** 2) + 1e-3 * np.sin(j)
    cases = []
    arrays = {}
    specs = [("rbf600", 1, 5, 500, 0, 600), ("rbf600", 1, 20, 550, 2, 600), ("ntk500", 1, 10, 450, 1, 500),
             ("ntk500", 2, 3, 240, 3, 250), ("wishart400", 1, 2, 380, 0, 400), ("powerlaw800", 1, 1, 700, 1, 800),
             ("powerlaw800", 1, 50, 790, 4, 800)]
    for name, d, n0, ns, q, n in specs:
        fit = F.fit_prefix(seqs[name], d, n0, ns, q)
        L_hat, ell_hat = F.predict(fit, np.arange(ns + 1, n + 1))
        lo, hi = F.predict_interval(fit, n, 0.9)
        key = f"{name}_d{d}_n0{n0}_ns{ns}_q{q}"
        arrays[key + "_L_hat"] = np.asarray(L_hat)
        arrays[key + "_ell_hat"] = np.asarray(ell_hat)
        arrays[key + "_residuals"] = np.asarray(fit.residuals)
        cases.append({"key": key, "seq": name, "d": d, "n0": n0, "ns": ns, "q": q, "n": n,
                      "fit": fit.to_json_dict(), "interval90": [lo, hi]})
    burn = []
    for name, d, ns, q in [("rbf600", 1, 600, 0), ("powerlaw800", 1, 800, 1)]:
        burn.append({"seq": name, "d": d, "ns": ns, "q": q,
                     "n0": int(F.select_burn_in(seqs[name], d, ns, q, candidates=(1, 10, 50, 100)))})
    traces = {f"{k}_trace_d{d}": F.scaling_ratio_trace(seqs[k], d) for k in ("rbf600", "ntk500") for d in (1, 2)}
    for k, v in seqs.items():
        arrays["seq_" + k] = v
    arrays.update(traces)
    np.savez_compressed(os.path.join(HERE, "flodance.npz"), **arrays)
    import scipy
    with open(os.path.join(HERE, "flodance.json"), "w") as f:
        json.dump({"generator": "oocdet.flodance (reference 0.1.0, unmodified)", "numpy": np.__version__,
                   "scipy": scipy.__version__, "cases": cases, "burn_in": burn}, f, indent=1)
    print(f"{len(cases)} fits, {len(burn)} burn-in selections, {len(traces)} traces")


if __name__ == "__main__":
    main()
