"""Golden vectors for the generic (LU) path from the UNMODIFIED reference (`oocdet` 0.1.0):
memdet_lu results (log|det|, sign, block counters) on seeded generic matrices, and the generic
schedule tables.  Run in the build container (/root/reference mounted):

    python tests/golden/make_lu_golden.py

Only the reference's outputs are stored (tests/golden/lu.npz + lu.json)."""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    import oocdet

    tmp = tempfile.mkdtemp(prefix="lu-golden-")
    rng_cases = []

    def mat(kind, m, seed, dtype=np.float64):
        rng = np.random.default_rng(seed)
        if kind == "gauss":  # generic, well conditioned enough: N(0,1) + 2 sqrt(m) I
            a = rng.standard_normal((m, m)) + 2.0 * np.sqrt(m) * np.eye(m)
        elif kind == "needs_pivot":  # tiny diagonal: partial pivoting is required
            a = rng.standard_normal((m, m))
            a[np.diag_indices(m)] *= 1e-8
        elif kind == "negdet":  # an odd number of negative eigen-directions
            a = rng.standard_normal((m, m)) + 2.0 * np.sqrt(m) * np.eye(m)
            a[0] = -a[0]
        elif kind == "singular":  # two equal rows
            a = rng.standard_normal((m, m))
            a[m // 2] = a[m // 3]
        elif kind == "perm":  # a permutation matrix (sign = parity)
            a = np.eye(m)[rng.permutation(m)]
        else:
            raise ValueError(kind)
        return a.astype(dtype)

    specs = [("gauss", 1, [1]), ("gauss", 2, [1, 2]), ("gauss", 37, [1, 2, 3]), ("gauss", 130, [1, 2, 3, 4]),
             ("gauss", 300, [1, 3, 5, 7]), ("needs_pivot", 200, [1, 2, 4]), ("negdet", 257, [1, 3, 6]),
             ("singular", 150, [1, 2, 4]), ("perm", 64, [1, 4]), ("gauss", 1000, [4, 8])]
    arrays, cases = {}, []
    for kind, m, nbs in specs:
        name = f"{kind}{m}"
        a = mat(kind, m, seed=m + 7)
        arrays[name] = a
        path = os.path.join(tmp, name + ".mdm")
        mf = oocdet.MatrixFile.create(path, m, a.dtype, "generic")
        mm = mf.memmap("r+")
        mm[:] = a
        mm.flush()
        del mm
        runs = {}
        for nb in nbs:
            r = oocdet.memdet_lu(path, num_blocks=nb)
            runs[str(nb)] = {"logabsdet": float(r.logabsdet), "sign": int(r.sign), "n_b": r.info.n_b,
                             "b": r.info.b, "blocks_read": r.info.blocks_read,
                             "blocks_written": r.info.blocks_written, "scratch_slots": r.info.scratch_slots}
        cases.append({"name": name, "m": m, "runs": runs})
    f32 = mat("gauss", 96, seed=5, dtype=np.float32)
    arrays["gauss96_f32"] = f32
    path = os.path.join(tmp, "f32.mdm")
    mf = oocdet.MatrixFile.create(path, 96, f32.dtype, "generic")
    mm = mf.memmap("r+")
    mm[:] = f32
    mm.flush()
    del mm
    r = oocdet.memdet_lu(path, num_blocks=3)
    cases.append({"name": "gauss96_f32", "m": 96, "runs": {"3": {
        "logabsdet": float(r.logabsdet), "sign": int(r.sign), "n_b": r.info.n_b, "b": r.info.b,
        "blocks_read": r.info.blocks_read, "blocks_written": r.info.blocks_written,
        "scratch_slots": r.info.scratch_slots}}})
    sched = {}
    for nb in range(2, 8):
        for k in range(1, nb):
            sched[f"{nb}_{k}"] = [[e.i, e.j, list(e.loads), e.target] for e in oocdet.schedule(nb, "generic", k)]
    np.savez_compressed(os.path.join(HERE, "lu.npz"), **arrays)
    with open(os.path.join(HERE, "lu.json"), "w") as f:
        json.dump({"generator": "oocdet.memdet_lu / schedule (reference 0.1.0, unmodified)",
                   "numpy": np.__version__, "cases": cases, "schedule_generic": sched}, f, indent=1)
    print(f"{len(cases)} matrices, {sum(len(c['runs']) for c in cases)} runs, {len(sched)} schedule stages")


if __name__ == "__main__":
    main()
