"""Golden vectors for the full-size configs C3, C4L (C4's leading 65536 block) and C5S (C5's recipe
at n = 98304) from the CPU ORACLE (oracle/memdet_oracle.py: the reference's _memdet_symmetric
restated over the same SciPy LAPACK / NumPy BLAS calls, pinned to the unmodified reference's own
outputs by tests/test_oracle_golden.py and, at C2 size, by tests/golden/c2.*).

Runs ON THE GPU BOX (the inputs are formed on the device; the reference package is not there,
and these orders exceed this container's memory):

    python tests/golden/make_big_golden.py --config C3 [--out gpurun_out/golden]

Steps: form the config's matrix on the device (gen.big_config_device), copy it to host memory,
record gen.sha_rows of the bytes, run the engine once on the device copy (a diagnostic recorded
beside the golden, not the golden), free the device, then run the oracle on all host cores:
memdet_cholesky, and memdet_ldl where its scalar pivoted tile kernel finishes (C3, C4L; C5S's
19661-row tiles would take hours).  Writes <config>.npz (prefixes, perm, signs) and
<config>.json (SHA, versions, host, timings, counters).  The -m gpu test
tests/test_big_configs_gpu.py regenerates the input, checks the SHA and compares.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True, choices=["C3", "C4L", "C5S"])
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "golden"))
    ap.add_argument("--no-ldl", action="store_true")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    import scipy
    import torch

    import paper_2503_04424_b200 as eng
    from oracle import memdet_oracle as O
    from paper_2503_04424_b200 import gen

    cfg = gen.BIG_CONFIGS[args.config]
    n, nb = cfg["n"], cfg["num_blocks"]
    secs = {}
    t0 = time.perf_counter()
    a = gen.big_config_device(args.config)
    torch.cuda.synchronize()
    secs["formation"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = a.cpu().numpy()
    digest = gen.sha_rows(host)
    secs["d2h_sha"] = time.perf_counter() - t0
    print(f"{args.config}: n={n} formed in {secs['formation']:.1f} s, sha {digest}", flush=True)
    with_ldl = not args.no_ldl and args.config != "C5S"
    eng_out = {}
    t0 = time.perf_counter()
    ec = eng.memdet_cholesky(a, num_blocks=nb)
    eng_out["chol"] = ec.prefix.copy()
    secs["engine_chol"] = time.perf_counter() - t0
    if with_ldl:
        t0 = time.perf_counter()
        el = eng.memdet_ldl(a, num_blocks=nb)
        eng_out["ldl"] = (el.prefix.copy(), el.perm.copy(), el.prefix_signs.copy())
        secs["engine_ldl"] = time.perf_counter() - t0
    eng.release_engine_cache()
    del a
    torch.cuda.empty_cache()
    threads = os.environ.get("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    manifest = {"oracle": "oracle/memdet_oracle.py (reference memdet.py:322-433 over SciPy LAPACK / NumPy BLAS)",
                "config": args.config, "spec": cfg, "input_sha_rows": digest, "m": n, "num_blocks": nb,
                "numpy": np.__version__, "scipy": scipy.__version__, "torch": torch.__version__,
                "python": platform.python_version(), "cores": os.cpu_count(), "openblas_threads": threads,
                "cpu": platform.processor() or platform.machine(), "seconds": secs, "runs": {}}
    try:
        with open("/proc/cpuinfo") as f:
            manifest["cpu"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    arrays = {}
    if with_ldl:
        t0 = time.perf_counter()
        perm, prefix, signs, info = O.memdet_ldl(host, nb)
        secs["oracle_ldl"] = time.perf_counter() - t0
        arrays.update(ldl__prefix=prefix, ldl__perm=perm, ldl__signs=signs)
        manifest["runs"]["ldl"] = dict(logdet=float(prefix[-1]), n_b=info.n_b, b=info.b,
                                       blocks_read=info.blocks_read, blocks_written=info.blocks_written,
                                       scratch_slots=info.scratch_slots)
        ep, eperm, esig = eng_out["ldl"]
        rel = np.max(np.abs(ep - prefix) / np.maximum(1, np.abs(prefix)))
        diff = int(np.sum(eperm != perm))
        manifest["runs"]["ldl"]["engine_check"] = dict(max_rel=float(rel), perm_positions_differing=diff,
                                                       signs_equal=bool(np.array_equal(esig, signs)))
        print(f"oracle ldl {secs['oracle_ldl']:.0f} s logdet {prefix[-1]!r}; engine max rel {rel:.3e}, "
              f"perm differs at {diff}", flush=True)
    t0 = time.perf_counter()
    prefix, info = O.memdet_cholesky(host, nb, inplace=True)
    secs["oracle_chol"] = time.perf_counter() - t0
    arrays["chol__prefix"] = prefix
    manifest["runs"]["chol"] = dict(logdet=float(prefix[-1]), n_b=info.n_b, b=info.b,
                                    blocks_read=info.blocks_read, blocks_written=info.blocks_written,
                                    scratch_slots=info.scratch_slots)
    rel = np.max(np.abs(eng_out["chol"] - prefix) / np.maximum(1, np.abs(prefix)))
    manifest["runs"]["chol"]["engine_check"] = dict(max_rel=float(rel))
    print(f"oracle chol {secs['oracle_chol']:.0f} s logdet {prefix[-1]!r}; engine max rel {rel:.3e}", flush=True)
    name = args.config.lower()
    np.savez_compressed(os.path.join(args.out, f"{name}.npz"), **arrays)
    with open(os.path.join(args.out, f"{name}.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print(f"wrote {args.out}/{name}.npz / .json", secs, flush=True)


if __name__ == "__main__":
    main()
