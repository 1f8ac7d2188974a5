"""Pin the CPU oracle (oracle/memdet_oracle.py) to the reference's own outputs.

The golden vectors were produced by the unmodified reference (tests/golden/make_golden.py);
the oracle must reproduce every prefix to 1e-12 (it calls the same LAPACK/BLAS), every LDL
permutation and sign bit-exactly, and every transfer counter exactly."""

import numpy as np
import pytest

from conftest import rel_err
from oracle import memdet_oracle as O

CASES = ["spd1", "spd2", "spd5", "spd30", "spd48", "spd64", "spd120", "spd200", "sym24", "sym30",
         "sym48", "sym64", "sym120", "eye50", "diag8", "hand2", "notspd2", "hardindef2",
         "spd40_f32", "rbf512", "ntk384", "C1"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(golden, name):
    inp = golden.input(name)
    for key, meta in golden.cases[name]["runs"].items():
        drv, nb = key.split("_nb")
        nb = int(nb)
        ref = golden.run(name, key)
        try:
            if drv == "chol":
                prefix, info = O.memdet_cholesky(inp, nb)
                perm = signs = None
            else:
                perm, prefix, signs, info = O.memdet_ldl(inp, nb)
        except O.OracleNotSpd:
            assert ref.get("error") == "NotSpdError", (name, key)
            continue
        except O.OracleIndefinite:
            assert ref.get("error") == "IndefiniteBlockError", (name, key)
            continue
        assert "error" not in ref, (name, key, ref)
        tol = 1e-5 if inp.dtype == np.float32 else 1e-12
        assert rel_err(prefix, ref["prefix"]) <= tol, (name, key)
        assert (info.n_b, info.b) == (ref["n_b"], ref["b"])
        assert (info.blocks_read, info.blocks_written, info.scratch_slots) == \
            (ref["blocks_read"], ref["blocks_written"], ref["scratch_slots"]), (name, key)
        if perm is not None:
            np.testing.assert_array_equal(perm, ref["perm"])
            np.testing.assert_array_equal(signs, ref["signs"])


def test_hand_cases(golden):
    # reference tests/test_kernels.py:114-118 and tests/test_memdet.py:100-105
    p = golden.run("hand2", "chol_nb1")["prefix"]
    assert p[-1] == pytest.approx(np.log(16.0), rel=1e-15)
    p = golden.run("diag8", "ldl_nb2")["prefix"]
    assert p[-1] == pytest.approx(np.log(40320.0), rel=1e-13)
    assert golden.run("notspd2", "chol_nb1")["error"] == "NotSpdError"
    assert golden.run("hardindef2", "ldl_nb1")["error"] == "IndefiniteBlockError"


def test_ldl_tile_restatement_is_exact_on_pivot_order():
    # reference tests/test_kernels.py:59-64: largest diagonal first
    a = np.diag([2.0, 3.0])
    swaps, d = O.ldl_tile(a)
    assert d[0] == 3.0 and float(np.prod(d)) == 6.0
    with pytest.raises(O.OracleIndefinite):
        O.ldl_tile(np.zeros((2, 2)))


def _ref_ldl():
    import importlib
    import os
    import sys

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
    if not os.path.isdir(ref):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        return importlib.import_module("_ldl")
    except ImportError:
        return None


@pytest.mark.parametrize("n,seed", [(5, 1), (33, 2), (64, 3), (200, 4)])
def test_ldl_restatement_bit_exact_vs_reference_compiled_kernel(n, seed):
    """oracle/ldl_tile.c vs the reference's own compiled _ldl.pyx (built by oracle/build_ref.sh
    from /root/reference): identical swaps and bit-identical pivots and factors."""
    ref = _ref_ldl()
    if ref is None:
        pytest.skip("oracle/_ref not built (reference not mounted)")
    from paper_2503_04424_b200 import gen

    a0 = gen.random_symmetric(n, seed=seed)
    tol = 64.0 * np.finfo(np.float64).eps * np.max(np.abs(a0))
    a1 = a0.copy()
    sw1, d1, w1 = np.empty(n, np.int64), np.empty(n), np.empty(n)
    assert ref.ldl_factor(a1, sw1, d1, w1, tol) == -1
    a2 = a0.copy()
    sw2, d2 = O.ldl_tile(a2)
    np.testing.assert_array_equal(sw1, sw2)
    np.testing.assert_array_equal(d1, d2)
    np.testing.assert_array_equal(np.tril(a1, -1), np.tril(a2, -1))


def _f32_golden():
    import json
    import os
    import sys

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    from make_f32_golden import CASES

    with open(os.path.join(here, "f32.json")) as f:
        meta = json.load(f)
    return CASES, meta, np.load(os.path.join(here, "f32.npz"))


def _f32_cases():
    cases, meta, _ = _f32_golden()
    return [(name, nb) for name, (_, nbs) in cases.items() for nb in nbs]


@pytest.mark.parametrize("name,nb", _f32_cases())
def test_f32_model_bit_exact_vs_reference_goldens(name, nb):
    """oracle/ldl32_model.c (the reference's memdet_ldl on a float32 file with the f32 rounding
    sequence of its LDL kernel, STRSM and SGEMM) reproduces the unmodified reference's outputs
    bit for bit: permutation, signs and the float32 prefix (NumPy's own log / cumsum of d)."""
    import hashlib

    cases, meta, arr = _f32_golden()
    a = cases[name][0]().astype(np.float32)
    assert hashlib.sha256(a.tobytes()).hexdigest() == meta["cases"][name]["input_sha256"]
    run = meta["cases"][name]["runs"][f"ldl_nb{nb}"]
    perm, d, fail = O.memdet_ldl32(a, nb)
    if "error" in run:
        assert fail >= 0, run
        return
    assert fail == -1
    key = f"{name}__ldl_nb{nb}"
    np.testing.assert_array_equal(perm, arr[key + "__perm"])
    np.testing.assert_array_equal(np.cumsum(np.log(np.abs(d))), arr[key + "__prefix"])
    np.testing.assert_array_equal(np.cumprod(np.sign(d)).astype(np.int64), arr[key + "__signs"])


@pytest.mark.parametrize("n,seed", [(33, 2), (200, 4)])
def test_ldl_restatement_f32_bit_exact_vs_reference_compiled_kernel(n, seed):
    """The float32 instance of the restated tile kernel vs the reference's compiled `floating`
    kernel on float32 input."""
    ref = _ref_ldl()
    if ref is None:
        pytest.skip("oracle/_ref not built (reference not mounted)")
    from paper_2503_04424_b200 import gen

    a0 = gen.random_symmetric(n, seed=seed).astype(np.float32)
    tol = 64.0 * float(np.finfo(np.float32).eps) * float(np.max(np.abs(a0)))
    a1 = a0.copy()
    sw1, d1, w1 = np.empty(n, np.int64), np.empty(n, np.float32), np.empty(n, np.float32)
    assert ref.ldl_factor(a1, sw1, d1, w1, tol) == -1
    a2 = a0.copy()
    sw2, d2 = O.ldl_tile(a2)
    np.testing.assert_array_equal(sw1, sw2)
    np.testing.assert_array_equal(d1, d2)
    np.testing.assert_array_equal(np.tril(a1, -1), np.tril(a2, -1))
