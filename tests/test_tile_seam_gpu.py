"""The tile seam (paper_2503_04424_b200/kernels.py): the reference's kernel module on the GPU.

1. Tile level: ldl_inplace against the C restatement of the reference's compiled kernel
   (oracle/ldl_tile.c, itself bit-checked against _ldl.pyx) in float64 and float32 -- swaps, d
   and L bit-identical, the strict upper triangle untouched; cholesky_inplace / solve_lower /
   schur_update against the oracle's LAPACK / BLAS calls to rounding.
2. Driver level: the reference's symmetric driver (restated in oracle/memdet_oracle.py, which
   calls the tile kernels by name as memdet.py:36-44 does) with the GPU seam kernels bound in
   place of LAPACK / BLAS reproduces the UNMODIFIED reference's stored outputs bit for bit
   (tests/golden/golden.npz float64 and tests/golden/f32.npz float32): the seam follows the
   golden host's BLAS rounding sequence."""

import json
import os

import numpy as np
import pytest

from conftest import rel_err
from oracle import memdet_oracle as O
from paper_2503_04424_b200 import _native, gen
from paper_2503_04424_b200 import kernels as K

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if _native.load().b2d_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("n,seed", [(1, 1), (33, 2), (200, 3), (700, 4)])
def test_ldl_tile_bit_identical_to_reference_kernel(dtype, n, seed):
    a0 = gen.random_symmetric(n, seed=seed).astype(dtype)
    a1, a2 = a0.copy(), a0.copy()
    sw1, d1 = O.ldl_tile(a1)
    sw2, d2 = K.ldl_inplace(a2)
    np.testing.assert_array_equal(sw1, sw2)
    np.testing.assert_array_equal(d1, d2)
    np.testing.assert_array_equal(np.tril(a1), np.tril(a2))
    np.testing.assert_array_equal(np.triu(a2, 1), np.triu(a0, 1))  # never touched, as _ldl.pyx


def test_ldl_tile_errors_and_strided_views():
    with pytest.raises(K.IndefiniteBlockError):
        K.ldl_inplace(np.zeros((8, 8)))
    with pytest.raises(K.IndefiniteBlockError):
        K.ldl_inplace(np.array([[0.0, 1.0], [1.0, 0.0]]))
    big = gen.random_symmetric(300, seed=9)
    view = big[:200, :200]  # a strided tile, as the reference's ragged blocks
    ref = view.copy()
    sw1, d1 = O.ldl_tile(ref)
    sw2, d2 = K.ldl_inplace(view)
    np.testing.assert_array_equal(d1, d2)
    np.testing.assert_array_equal(np.tril(ref), np.tril(big[:200, :200]))


def test_cholesky_solve_and_schur_tiles():
    a = gen.spd_wishart(500, 500, seed=5, shift=1e-2)
    l1, l2 = a.copy(), a.copy()
    d1 = O.chol_tile(l1)
    d2 = K.cholesky_inplace(l2)
    assert rel_err(d2, d1) <= 1e-13 and np.all(np.triu(l2, 1) == 0)
    np.testing.assert_allclose(l2, l1, rtol=0, atol=1e-12)
    b1 = np.random.default_rng(1).standard_normal((500, 300))
    b2 = b1.copy()
    O.lower_solve(l1, b1, unit=False)
    K.solve_lower_inplace(l1, b2, unit_diag=False)
    np.testing.assert_allclose(b2, b1, rtol=1e-12, atol=1e-12)
    s1 = np.random.default_rng(2).standard_normal((300, 280))
    s2 = s1.copy()
    c = np.random.default_rng(3).standard_normal((500, 300))
    bb = np.random.default_rng(4).standard_normal((500, 280))
    O.schur_update(s1, c, bb)
    K.schur_update(s2, c, bb, "ct_b")
    np.testing.assert_allclose(s2, s1, rtol=1e-12, atol=1e-11)
    with pytest.raises(K.NotSpdError):
        K.cholesky_inplace(-np.eye(4))


class _Bound:
    """The oracle driver with the seam kernels bound by name (as memdet.py:36-44 imports them)."""

    def __init__(self):
        self.saved = {}

    def __enter__(self):
        def ldl(a):
            try:
                return K.ldl_inplace(a)
            except K.IndefiniteBlockError as exc:
                raise O.OracleIndefinite(str(exc), 0) from exc

        def chol(a):
            try:
                return K.cholesky_inplace(a)
            except K.NotSpdError as exc:
                raise O.OracleNotSpd(str(exc)) from exc

        new = {"ldl_tile": ldl, "chol_tile": chol,
               "lower_solve": lambda l, b, unit: K.solve_lower_inplace(l, b, unit_diag=unit),
               "schur_update": lambda t, c, b: K.schur_update(t, c, b, "ct_b")}
        for k, v in new.items():
            self.saved[k] = getattr(O, k)
            setattr(O, k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            setattr(O, k, v)


def test_reference_driver_on_seam_matches_reference_f64(golden):
    checked = 0
    with _Bound():
        for name, case in golden.cases.items():
            for key, run in case["runs"].items():
                if not key.startswith("ldl_nb") or "error" in run or name == "C1":
                    continue
                inp = golden.input(name)
                if inp.dtype != np.float64:
                    continue
                perm, prefix, signs, info = O.memdet_ldl(inp, run["n_b"])
                ref = golden.run(name, key)
                np.testing.assert_array_equal(perm, ref["perm"])
                np.testing.assert_array_equal(prefix, ref["prefix"])  # bit for bit
                np.testing.assert_array_equal(signs, ref["signs"])
                checked += 1
    assert checked >= 6


def test_reference_driver_on_seam_matches_reference_f32():
    import sys

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    from make_f32_golden import CASES

    with open(os.path.join(here, "f32.json")) as f:
        meta = json.load(f)
    arr = np.load(os.path.join(here, "f32.npz"))
    checked = 0
    with _Bound():
        for name in ("wish512s4", "sym300", "rbf600", "lowrank300"):
            a = CASES[name][0]().astype(np.float32)
            for key, run in meta["cases"][name]["runs"].items():
                nb = int(key.split("nb")[1])
                if "error" in run:
                    with pytest.raises(O.OracleIndefinite):
                        O.memdet_ldl(a, nb)
                    continue
                perm, prefix, signs, _ = O.memdet_ldl(a, nb)
                np.testing.assert_array_equal(perm, arr[f"{name}__{key}__perm"])
                np.testing.assert_array_equal(prefix, arr[f"{name}__{key}__prefix"])
                checked += 1
    assert checked >= 8
