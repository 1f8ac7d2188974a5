"""float32 memdet_ldl in f32 arithmetic vs the unmodified reference (tests/golden/f32.*).

The reference factors a float32 file in float32 (memdet.py:337-338; _ldl.pyx `floating`; SciPy's
f32 ?trtrs; NumPy's f32 matmul; tolerance 64 eps(f32) max|A|, dense.py:73), so its pivots differ
from the same values factored in f64 (79 positions at
spd_wishart(512, 512, seed=4, shift=1e-3), num_blocks=2).  The engine's f32 path (ldl32.cu)
follows the same rounding sequence: permutation and signs bit-exact, D bit-identical to the
oracle model (oracle/ldl32_model.c, itself bit-exact vs the goldens), prefixes within the
reference's own float32 bar 1e-4 (tests/test_memdet.py:247-256; measured ~1e-7: the engine sums
log|d| in double-double, the reference in float32), IndefiniteBlockError where it raises."""

import hashlib

import numpy as np
import pytest

import paper_2503_04424_b200 as eng
from conftest import rel_err
from oracle import memdet_oracle as O
from paper_2503_04424_b200 import _native
from test_oracle_golden import _f32_cases, _f32_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if _native.load().b2d_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    yield
    eng.release_engine_cache()


_inputs = {}


def _input(name):
    cases, meta, _ = _f32_golden()
    if name not in _inputs:
        a = cases[name][0]().astype(np.float32)
        assert hashlib.sha256(a.tobytes()).hexdigest() == meta["cases"][name]["input_sha256"]
        _inputs[name] = a
    return _inputs[name]


@pytest.mark.parametrize("name,nb", _f32_cases())
def test_f32_ldl_matches_reference(name, nb):
    _, meta, arr = _f32_golden()
    a = _input(name)
    run = meta["cases"][name]["runs"][f"ldl_nb{nb}"]
    if "error" in run:
        with pytest.raises(eng.IndefiniteBlockError):
            eng.memdet_ldl(a, num_blocks=nb)
        return
    res = eng.memdet_ldl(a, num_blocks=nb)
    key = f"{name}__ldl_nb{nb}"
    assert res.prefix.dtype == np.float32
    np.testing.assert_array_equal(res.perm, arr[key + "__perm"])
    np.testing.assert_array_equal(res.prefix_signs, arr[key + "__signs"])
    assert rel_err(res.prefix, arr[key + "__prefix"]) <= 1e-4, rel_err(res.prefix, arr[key + "__prefix"])
    if a.shape[0] <= 1000:  # D bit-identical to the model (the reference's f32 values)
        perm, d, fail = O.memdet_ldl32(a, nb)
        assert fail == -1
        np.testing.assert_array_equal(res.d.astype(np.float32), d)
        assert np.all(res.d == d.astype(np.float64))


def test_f32_device_tensor_equals_host():
    torch = pytest.importorskip("torch")
    a = _input("wish512s4")
    host = eng.memdet_ldl(a, num_blocks=2)
    dev = eng.memdet_ldl(torch.from_numpy(a).cuda(), num_blocks=2)
    np.testing.assert_array_equal(host.perm, dev.perm)
    np.testing.assert_array_equal(host.prefix, dev.prefix)


def test_f32_one_shot_c_abi_matches_reference():
    """b2d_memdet_sym with dtype B2D_F32, mode LDL_PIV (the entry INTEGRATION.md tells reference
    maintainers to bind) takes the f32 path too."""
    import ctypes

    _, _, arr = _f32_golden()
    a = _input("wish512s4")
    m = a.shape[0]
    d = np.empty(m)
    perm = np.empty(m, np.int64)
    prefix = np.empty(m)
    signs = np.empty(m, np.int64)
    info = _native.RunInfoC()
    fail = ctypes.c_int64(-1)
    rc = _native.load().b2d_memdet_sym(a.ctypes.data, m, m, _native.B2D_F32, _native.MODE_LDL_PIV, 2, 0, None, 0,
                                       d.ctypes.data, perm.ctypes.data, prefix.ctypes.data, signs.ctypes.data,
                                       ctypes.byref(info), ctypes.byref(fail))
    assert rc == 0, _native.last_error()
    np.testing.assert_array_equal(perm, arr["wish512s4__ldl_nb2__perm"])
    assert rel_err(prefix, arr["wish512s4__ldl_nb2__prefix"]) <= 1e-4
