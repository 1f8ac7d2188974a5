"""memdet_cholesky / memdet_ldl(pivoting="none") with devices=[...]: one process, several devices,
1-D block-cyclic outer panels, each device ingesting only its own panels (engine mgpu.cu).

On the one-GPU test box the ranks share cuda:0 (devices=[0, 0] / [0, 0, 0]): every dependency
between ranks is a stream-event wait, so this exercises the whole multi-device schedule --
panel ownership, sharded ingest, the cross-rank panel copies and event ordering, the gather of
2 log L_ii and the prefix -- with the real kernels.  Parity: the CPU oracle (reference
memdet.py:415-433) and the single-device engine on the same bytes."""

import numpy as np
import pytest

import paper_2503_04424_b200 as eng
from conftest import rel_err
from oracle import memdet_oracle as O
from paper_2503_04424_b200 import _native, gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if _native.load().b2d_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    yield
    eng.release_engine_cache()


@pytest.mark.parametrize("m,devices", [(5000, [0, 0]), (5000, [0, 0, 0]), (9000, [0, 0]), (12345, [0, 0, 0, 0])])
def test_multidevice_cholesky_matches_oracle(m, devices):
    a = gen.spd_wishart(m, m, seed=m, shift=1e-2)
    ref, _ = O.memdet_cholesky(a, 2)
    res = eng.memdet_cholesky(a, num_blocks=2, devices=devices)
    assert rel_err(res.prefix, ref) <= 1e-10, rel_err(res.prefix, ref)
    single = eng.memdet_cholesky(a, num_blocks=2)
    assert rel_err(res.prefix, single.prefix) <= 1e-12
    np.testing.assert_allclose(res.d, single.d, rtol=1e-12)
    assert res.info.h2d_bytes > 0


def test_multidevice_inputs_pinned_pageable_device_and_ldl():
    torch = pytest.importorskip("torch")
    m = 7000
    a = gen.spd_wishart(m, m, seed=77, shift=1e-2)
    ref, _ = O.memdet_cholesky(a, 4)
    pinned = torch.from_numpy(a).pin_memory()
    for inp in (a, pinned.numpy(), torch.from_numpy(a).cuda()):
        res = eng.memdet_cholesky(inp, num_blocks=4, devices=[0, 0])
        assert rel_err(res.prefix, ref) <= 1e-10
    ldl = eng.memdet_ldl(a, num_blocks=4, pivoting="none", devices=[0, 0, 0])
    assert rel_err(ldl.prefix, ref) <= 1e-10
    assert list(ldl.perm) == list(range(m))
    # float32 file: computed in FP64 from the f32 values, as the single-device Cholesky
    a32 = a.astype(np.float32)
    r32 = eng.memdet_cholesky(a32, num_blocks=4, devices=[0, 0])
    s32 = eng.memdet_cholesky(a32, num_blocks=4)
    assert r32.prefix.dtype == np.float32 and rel_err(r32.prefix, s32.prefix) <= 1e-6


def test_multidevice_not_spd_reports_the_global_pivot():
    m = 6000
    a = gen.spd_wishart(m, m, seed=5, shift=1e-2)
    a[4500, 4500] = -1.0  # the leading minor of order 4501 is indefinite
    with pytest.raises(eng.NotSpdError, match="4501"):
        eng.memdet_cholesky(a, num_blocks=2, devices=[0, 0])
    with pytest.raises(eng.NotSpdError, match="4501"):
        eng.memdet_cholesky(a, num_blocks=2)


def test_multidevice_c2_full_size_equals_single_device():
    """C2 (n = 32768 RBF, device-formed) over two ranks vs one device: every prefix 1e-12."""
    torch = pytest.importorskip("torch")
    import ctypes

    n = 32768
    x = torch.from_numpy(gen.rbf_points(n, 16, seed=0)).cuda()
    a = torch.empty((n, n), dtype=torch.float64, device="cuda")
    _native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6,
                                             ctypes.c_void_p(a.data_ptr()), None))
    torch.cuda.synchronize()
    single = eng.memdet_cholesky(a, num_blocks=8)
    eng.release_engine_cache()
    multi = eng.memdet_cholesky(a, num_blocks=8, devices=[0, 0])
    eng.release_engine_cache()
    assert rel_err(multi.prefix, single.prefix) <= 1e-12, rel_err(multi.prefix, single.prefix)
    # the north star's LDL^T (block-pivoted, 8 blocks): bit-identical to one device
    lsingle = eng.memdet_ldl(a, num_blocks=8)
    eng.release_engine_cache()
    lmulti = eng.memdet_ldl(a, num_blocks=8, devices=[0, 0, 0])
    eng.release_engine_cache()
    np.testing.assert_array_equal(lmulti.perm, lsingle.perm)
    np.testing.assert_array_equal(lmulti.prefix, lsingle.prefix)


@pytest.mark.parametrize("m,nb,devices", [(3072, 3, [0, 0]), (4096, 4, [0, 0, 0]), (2560, 5, [0, 0]), (1000, 1, [0, 0])])
def test_multidevice_block_pivoted_ldl_matches_oracle_and_single_device(m, nb, devices):
    """Stages on their owners, row-k block grids copied across ranks: perm / signs exact vs the
    oracle (the reference's pivoting), and every output bit-identical to one device."""
    a = gen.random_symmetric(m, seed=m + nb)
    perm, prefix, signs, _ = O.memdet_ldl(a, nb)
    res = eng.memdet_ldl(a, num_blocks=nb, devices=devices)
    np.testing.assert_array_equal(res.perm, perm)
    np.testing.assert_array_equal(res.prefix_signs, signs)
    assert rel_err(res.prefix, prefix) <= 1e-10
    single = eng.memdet_ldl(a, num_blocks=nb)
    np.testing.assert_array_equal(res.d, single.d)
    np.testing.assert_array_equal(res.prefix, single.prefix)


def test_multidevice_ldl_indefinite_and_unaligned_blocks():
    z = gen.random_symmetric(2048, seed=1)
    z[1024:, :] = 0.0
    z[:, 1024:] = 0.0  # the second block is all zero after no updates: the reference raises
    with pytest.raises(eng.IndefiniteBlockError):
        eng.memdet_ldl(z, num_blocks=2, devices=[0, 0])
    with pytest.raises(NotImplementedError):  # b = 1000 is not on a 128-row boundary
        eng.memdet_ldl(gen.random_symmetric(3000, seed=2), num_blocks=3, devices=[0, 0])
