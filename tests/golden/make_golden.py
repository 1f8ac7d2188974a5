"""Generate golden vectors from the UNMODIFIED reference (`oocdet` 0.1.0).

Run in the build container, where /root/reference is mounted (it is not on the GPU box):

    python tests/golden/make_golden.py [--ref-src /tmp/refpkg/src]

`--ref-src` may point at a /tmp copy of /root/reference/pkg/src with the Cython `_ldl`
built in place (`python setup.py build_ext --inplace`), which is much faster for the
4096-wide LDL tiles; the compiled and NumPy LDL paths are pinned equal by the reference's
own test (tests/test_kernels.py:94-105).  Nothing from the reference is copied: only its
outputs on seeded inputs are stored, in `tests/golden/*.npz` + `manifest.json`.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2503_04424_b200 import gen  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    default_src = "/tmp/refpkg/src" if os.path.isdir("/tmp/refpkg/src") else "/root/reference/pkg/src"
    ap.add_argument("--ref-src", default=default_src)
    ap.add_argument("--skip-c1", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, args.ref_src)
    import oocdet  # the reference
    from oocdet import kernels as rk
    from oocdet.cost import predicted_reads, predicted_writes, scratch_slots

    tmp = tempfile.mkdtemp(prefix="golden-")

    def write(values, symmetry):
        path = os.path.join(tmp, f"m{len(os.listdir(tmp))}.mdm")
        mf = oocdet.MatrixFile.create(path, values.shape[0], values.dtype, symmetry)
        mm = mf.memmap("r+")
        mm[:] = values
        mm.flush()
        del mm
        return path

    def run(driver, path, nb):
        try:
            res = driver(path, num_blocks=nb)
        except oocdet.NotSpdError:
            return {"error": "NotSpdError"}
        except oocdet.IndefiniteBlockError as exc:
            return {"error": "IndefiniteBlockError", "msg": str(exc)}
        out = {"prefix": res.prefix, "n_b": res.info.n_b, "b": res.info.b,
               "blocks_read": res.info.blocks_read, "blocks_written": res.info.blocks_written,
               "scratch_slots": res.info.scratch_slots}
        if hasattr(res, "perm"):
            out["perm"] = res.perm
            out["signs"] = res.prefix_signs
        return out

    manifest = {
        "reference": "oocdet " + oocdet.__version__,
        "ref_src": args.ref_src,
        "compiled_ldl": bool(rk.HAVE_COMPILED_LDL),
        "numpy": np.__version__,
        "scipy": __import__("scipy").__version__,
        "python": platform.python_version(),
        "cases": {},
    }

    arrays = {}

    def store(name, inp, symmetry, nbs, drivers, keep_input=True):
        path = write(inp, symmetry)
        case = {"m": int(inp.shape[0]), "dtype": str(inp.dtype), "symmetry": symmetry,
                "input_sha256": sha(inp), "runs": {}}
        if keep_input:
            arrays[f"{name}__input"] = inp
        for dname in drivers:
            driver = {"chol": oocdet.memdet_cholesky, "ldl": oocdet.memdet_ldl}[dname]
            for nb in nbs:
                out = run(driver, path, nb)
                key = f"{dname}_nb{nb}"
                meta = {}
                for k, v in out.items():
                    if isinstance(v, np.ndarray):
                        arrays[f"{name}__{key}__{k}"] = v
                    else:
                        meta[k] = v
                case["runs"][key] = meta
        manifest["cases"][name] = case

    # A. random SPD, small and ragged sizes, every driver, n_b 1..8
    for m, seed in [(1, 11), (2, 12), (5, 13), (30, 14), (48, 15), (64, 16), (120, 17), (200, 18)]:
        store(f"spd{m}", gen.random_spd(m, seed=seed), "spd", range(1, 9), ["chol", "ldl"])
    # B. symmetric indefinite (pivoting matters; Cholesky must fail)
    for m, seed in [(24, 21), (30, 22), (48, 23), (64, 24), (120, 25)]:
        store(f"sym{m}", gen.random_symmetric(m, seed=seed), "symmetric", [1, 2, 3, 4], ["chol", "ldl"])
    # C. hand-checked cases
    store("eye50", np.eye(50), "spd", [1, 3], ["chol", "ldl"])
    store("diag8", np.diag(np.arange(1.0, 9.0)), "symmetric", [1, 2], ["chol", "ldl"])
    store("hand2", np.array([[4.0, 2.0], [2.0, 5.0]]), "spd", [1], ["chol", "ldl"])
    store("notspd2", np.array([[1.0, 2.0], [2.0, 1.0]]), "symmetric", [1], ["chol", "ldl"])
    store("hardindef2", np.array([[0.0, 1.0], [1.0, 0.0]]), "symmetric", [1], ["chol", "ldl"])
    # D. float32 file
    store("spd40_f32", gen.random_spd(40, seed=31).astype(np.float32), "spd", [1, 3], ["chol", "ldl"])
    # E. mid size: RBF and NTK-like spectra (the C2 / C3 families at test scale)
    store("rbf512", gen.rbf(512, seed=41), "spd", [1, 2, 4, 8], ["chol", "ldl"], keep_input=False)
    store("ntk384", gen.ntk_like(384, 768, 0.75, seed=42), "spd", [1, 3, 6], ["chol", "ldl"],
          keep_input=False)
    # F. C1 at full size (n=4096, num_blocks=4): every prefix, both drivers
    if not args.skip_c1:
        c1 = gen.spd_wishart(4096, 4096, seed=0, shift=1e-3)
        store("C1", c1, "spd", [4], ["chol", "ldl"], keep_input=False)

    # G. host-side planner / schedule / cost tables
    sched = {}
    for nb in range(2, 11):
        for k in range(1, nb):
            sched[f"{nb}_{k}"] = [[e.i, e.j, list(e.loads), e.target]
                                  for e in oocdet.schedule(nb, "symmetric", k)]
    blocking = []
    for m, c, beta in [(1000, 8_000_000, 8), (1100, 8_000_000, 8), (1200, 8_000_000, 8),
                       (1024, 1024 * 1024 * 8, 8), (1024, 1024 * 1024 * 8 - 1, 8),
                       (196608, 64_000_000_000, 8), (196608, 64 * 2 ** 30, 8),
                       (32768, 2 ** 30, 8), (4096, 10 ** 7, 4), (7, 24, 8)]:
        nb, lay = oocdet.select_blocking(m, oocdet.Budget(c, beta))
        blocking.append([m, c, beta, nb, lay.b, lay.tail])
    grids = []
    for m, nb in [(1, 1), (5, 8), (10, 4), (10, 9), (120, 7), (4096, 4), (196608, 5), (100, 99)]:
        lay = oocdet.BlockLayout.from_grid(m, nb)
        grids.append([m, nb, lay.n_b, lay.b, lay.tail])
    cost = []
    for nb in range(1, 17):
        cost.append([nb, predicted_reads(nb, "symmetric"), predicted_writes(nb, "symmetric"),
                     scratch_slots(nb, "symmetric")])
    flops = []
    for m, nb in [(4096, 4), (32768, 8), (65536, 16), (120, 5)]:
        pc = oocdet.predicted_cost(m, nb, "symmetric")
        flops.append([m, nb, str(pc.total_flops), str(pc.gramian_multiply.total),
                      str(pc.full_multiply.total), str(pc.lower_solve.total),
                      str(pc.decomposition.total)])
    manifest["tables"] = {"schedule": sched, "select_blocking": blocking, "from_grid": grids,
                          "cost_counts": cost, "cost_flops": flops}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(manifest["cases"]), "cases")


if __name__ == "__main__":
    main()
