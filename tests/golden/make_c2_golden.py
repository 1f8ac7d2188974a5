"""Golden vectors for C2 at full size (n = 32768 RBF, num_blocks = 8) from the UNMODIFIED
reference (`oocdet` 0.1.0): every prefix of memdet_cholesky and memdet_ldl, the LDL
permutation and signs, and the reference's counters.

Run in the build container, where /root/reference is mounted (it is not on the GPU box):

    python tests/golden/make_c2_golden.py [--ref-src /tmp/refpkg/src] [--threads 8]

`--ref-src` should point at a /tmp copy of /root/reference/pkg/src with the Cython `_ldl`
built in place (`python setup.py build_ext --inplace`): the NumPy LDL fallback needs hours
for eight 4096-wide tiles.  The input is `gen.rbf(32768, seed=0)` (host NumPy, 8.6 GB); its
SHA-256 is recorded so the GPU test proves it factors the same bytes.  Only outputs are
stored (`tests/golden/c2.npz` + `c2.json`); nothing from the reference is copied.
Measured here: ~70 s input, ~65 s memdet_cholesky, ~165 s memdet_ldl (8 cores).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2503_04424_b200 import gen  # noqa: E402

N, NB = 32768, 8


def sha(a: np.ndarray) -> str:
    h = hashlib.sha256()
    for r0 in range(0, a.shape[0], 1024):
        h.update(np.ascontiguousarray(a[r0:r0 + 1024]).tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    default_src = "/tmp/refpkg/src" if os.path.isdir("/tmp/refpkg/src") else "/root/reference/pkg/src"
    ap.add_argument("--ref-src", default=default_src)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--tmp", default=None)
    args = ap.parse_args()
    sys.path.insert(0, args.ref_src)
    import oocdet  # the reference
    from oocdet import kernels as rk

    t0 = time.perf_counter()
    a = gen.rbf(N, seed=0, threads=args.threads)
    digest = sha(a)
    t_gen = time.perf_counter() - t0
    tmp = tempfile.mkdtemp(prefix="c2golden-", dir=args.tmp)
    path = os.path.join(tmp, "c2.mdm")
    mf = oocdet.MatrixFile.create(path, N, a.dtype, "spd")
    mm = mf.memmap("r+")
    for r0 in range(0, N, 1024):
        mm[r0:r0 + 1024] = a[r0:r0 + 1024]
    mm.flush()
    del mm, a
    manifest = {"reference": "oocdet " + oocdet.__version__, "compiled_ldl": bool(rk.HAVE_COMPILED_LDL),
                "numpy": np.__version__, "scipy": __import__("scipy").__version__,
                "python": platform.python_version(), "cores": os.cpu_count(),
                "input": f"gen.rbf({N}, d=16, ell=4.0, jitter=1e-6, seed=0)", "input_sha256": digest,
                "m": N, "num_blocks": NB, "seconds": {"input": t_gen}, "runs": {}}
    arrays = {}
    for name, driver in (("chol", oocdet.memdet_cholesky), ("ldl", oocdet.memdet_ldl)):
        t0 = time.perf_counter()
        res = driver(path, num_blocks=NB)
        manifest["seconds"][name] = time.perf_counter() - t0
        arrays[f"{name}__prefix"] = res.prefix
        if hasattr(res, "perm"):
            arrays[f"{name}__perm"] = res.perm
            arrays[f"{name}__signs"] = res.prefix_signs
        manifest["runs"][name] = {"logdet": float(res.prefix[-1]), "n_b": res.info.n_b, "b": res.info.b,
                                  "blocks_read": res.info.blocks_read, "blocks_written": res.info.blocks_written,
                                  "scratch_slots": res.info.scratch_slots}
        print(name, manifest["seconds"][name], res.prefix[-1], flush=True)
    os.remove(path)
    np.savez_compressed(os.path.join(HERE, "c2.npz"), **arrays)
    with open(os.path.join(HERE, "c2.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print("wrote c2.npz / c2.json", manifest["seconds"])


if __name__ == "__main__":
    main()
