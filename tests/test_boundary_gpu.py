"""The one-shot C entry INTEGRATION.md §B tells reference maintainers to bind, called exactly as
that stub does (ctypes, host buffers, every mode, the error codes, sign_out, devices / ndev)."""

import ctypes

import numpy as np
import pytest

from conftest import rel_err
from oracle import memdet_oracle as O
from paper_2503_04424_b200 import _native, gen

pytestmark = pytest.mark.gpu


class _Info(ctypes.Structure):  # the stub's own copy of b2d_run_info
    _fields_ = [(n, ctypes.c_int64) for n in (
        "m", "n_b", "b", "tail", "blocks_read", "blocks_written", "scratch_slots", "tile",
        "n_tiles", "h2d_bytes", "d2h_bytes", "kernel_launches")] + [
        ("device_ms", ctypes.c_double), ("wall_seconds", ctypes.c_double)] + [
        (n, ctypes.c_int64) for n in ("ooc_blocks", "ooc_block", "ooc_reads", "ooc_writes", "ooc_scratch")]


def _lib():
    lib = ctypes.CDLL(_native.LIB_PATH)
    lib.b2d_memdet_sym.restype = ctypes.c_int
    lib.b2d_memdet_sym.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.POINTER(_Info), ctypes.POINTER(ctypes.c_int64)]
    lib.b2d_last_error.restype = ctypes.c_char_p
    return lib


def _call(a, mode, num_blocks=0, max_mem=0, devices=None):
    lib = _lib()
    m = a.shape[0]
    d, prefix = np.empty(m), np.empty(m)
    perm, sign = np.empty(m, np.int64), np.empty(m, np.int64)
    info, fail = _Info(), ctypes.c_int64(-1)
    dev_arr = (ctypes.c_int * len(devices))(*devices) if devices else None
    rc = lib.b2d_memdet_sym(a.ctypes.data, m, m, 0 if a.dtype == np.float64 else 1, mode, num_blocks, max_mem,
                            dev_arr, len(devices) if devices else 0, d.ctypes.data, perm.ctypes.data,
                            prefix.ctypes.data, sign.ctypes.data, ctypes.byref(info), ctypes.byref(fail))
    return rc, d, perm, prefix, sign, info, fail.value, lib.b2d_last_error().decode()


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if _native.load().b2d_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


@pytest.mark.parametrize("devices", [None, [0], [0, 0]])
def test_memdet_sym_cholesky_and_unpivoted_ldl(devices):
    a = gen.spd_wishart(1500, 1500, seed=21, shift=1e-2)
    ref, oinfo = O.memdet_cholesky(a, 3)
    for mode in (_native.MODE_CHOLESKY, _native.MODE_LDL_NOPIV):
        rc, d, perm, prefix, sign, info, fail, err = _call(a, mode, num_blocks=3, devices=devices)
        assert rc == 0, err
        assert rel_err(prefix, ref) <= 1e-10
        assert (info.n_b, info.b, info.blocks_read, info.blocks_written, info.scratch_slots) == \
            (oinfo.n_b, oinfo.b, oinfo.blocks_read, oinfo.blocks_written, oinfo.scratch_slots)
        assert np.all(sign == 1) and fail == -1
        np.testing.assert_array_equal(perm, np.arange(1500))
        if mode == _native.MODE_LDL_NOPIV:
            np.testing.assert_allclose(np.cumsum(np.log(d)), ref, rtol=1e-10)


def test_memdet_sym_pivoted_ldl_perm_and_signs():
    a = gen.random_symmetric(900, seed=8)
    perm_ref, prefix_ref, signs_ref, _ = O.memdet_ldl(a, 3)
    rc, d, perm, prefix, sign, info, fail, err = _call(a, _native.MODE_LDL_PIV, num_blocks=3)
    assert rc == 0, err
    np.testing.assert_array_equal(perm, perm_ref)
    np.testing.assert_array_equal(sign, signs_ref)
    assert rel_err(prefix, prefix_ref) <= 1e-10
    # max_mem instead of num_blocks (memdet.py:63-80): same tiling as the oracle's rule
    nb = O.select_blocking(900, 900 * 900 * 8 // 4)
    rc, d, perm, prefix, sign, info, fail, err = _call(a, _native.MODE_LDL_PIV, max_mem=900 * 900 * 8 // 4)
    assert rc == 0, err and info.n_b == nb


def test_memdet_sym_error_codes():
    a = gen.spd_wishart(600, 600, seed=3, shift=1e-2)
    bad = a.copy()
    bad[300, 300] = -5.0
    rc, d, perm, prefix, sign, info, fail, err = _call(bad, _native.MODE_CHOLESKY, num_blocks=2)
    assert rc == _native.B2D_ERR_NOT_SPD and fail == 300, (rc, fail, err)
    z = np.zeros((64, 64))
    rc, *_, fail, err = _call(z, _native.MODE_LDL_PIV, num_blocks=1)
    assert rc == _native.B2D_ERR_INDEFINITE, err
    rc, *_, err = _call(a, _native.MODE_CHOLESKY)  # neither num_blocks nor max_mem
    assert rc == _native.B2D_ERR_USAGE, err
    rc, *_, err = _call(a, 9, num_blocks=2)  # unknown mode
    assert rc == _native.B2D_ERR_USAGE, err
    rc, *_, err = _call(a, _native.MODE_CHOLESKY, num_blocks=2, devices=[0] * 9)
    assert rc == _native.B2D_ERR_USAGE, err
