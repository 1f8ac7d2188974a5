"""The out-of-core scratchpad (reference storage.py:147-204): a temp file under scratch_dir /
$OOCDET_SCRATCH_DIR (mkstemp + ftruncate, memory-mapped, unlinked), lazily touched host memory by
default, or pinned memory (B2D_SCRATCH=pinned) -- the same kernels on the same bytes, so every
mode gives bit-identical results, equal to the oracle's."""

import os

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
    # small orders' scratchpads would fit in HBM beside the slots: keep them in host memory
    old = os.environ.get("B2D_HOST_SCRATCH")
    os.environ["B2D_HOST_SCRATCH"] = "1"
    eng.release_engine_cache()
    yield
    eng.release_engine_cache()
    if old is None:
        os.environ.pop("B2D_HOST_SCRATCH", None)
    else:
        os.environ["B2D_HOST_SCRATCH"] = old


def _with_mode(mode, fn):
    old = os.environ.get("B2D_SCRATCH")
    os.environ["B2D_SCRATCH"] = mode
    try:
        eng.release_engine_cache()
        return fn()
    finally:
        eng.release_engine_cache()
        if old is None:
            os.environ.pop("B2D_SCRATCH", None)
        else:
            os.environ["B2D_SCRATCH"] = old


@pytest.mark.parametrize("m,nb", [(1536, 4), (2000, 5)])
def test_scratch_modes_bit_identical_and_match_oracle(tmp_path, m, nb):
    a = gen.spd_wishart(m, m, seed=m, shift=1e-2)
    ref, info = O.memdet_cholesky(a, nb)
    runs = {}
    for mode in ("pinned", "staged"):
        runs[mode] = _with_mode(mode, lambda: eng.memdet_cholesky(a, num_blocks=nb, out_of_core=True))
    runs["file"] = eng.memdet_cholesky(a, num_blocks=nb, out_of_core=True, scratch_dir=str(tmp_path))
    eng.release_engine_cache()
    assert os.listdir(tmp_path) == []  # unlinked as soon as it is mapped
    for mode, res in runs.items():
        assert res.info.out_of_core and not _native.load() is None
        assert (res.info.ooc_reads, res.info.ooc_writes, res.info.ooc_scratch) == \
            (info.blocks_read, info.blocks_written, info.scratch_slots), mode
        np.testing.assert_array_equal(res.prefix, runs["pinned"].prefix)
    assert rel_err(runs["file"].prefix, ref) <= 1e-10


def test_scratch_dir_env_and_errors(tmp_path, monkeypatch):
    a = gen.spd_wishart(1200, 1200, seed=12, shift=1e-2)
    ref, _ = O.memdet_cholesky(a, 4)
    monkeypatch.setenv("OOCDET_SCRATCH_DIR", str(tmp_path))
    eng.release_engine_cache()
    res = eng.memdet_cholesky(a, num_blocks=4, out_of_core=True)
    assert rel_err(res.prefix, ref) <= 1e-10
    eng.release_engine_cache()
    with pytest.raises(eng.StorageError):
        eng.memdet_cholesky(a, num_blocks=4, out_of_core=True, scratch_dir=str(tmp_path / "missing"))


def test_file_scratch_pivoted_ldl_and_lu(tmp_path):
    a = gen.random_symmetric(1500, seed=15)
    perm, prefix, signs, _ = O.memdet_ldl(a, 4)
    res = eng.memdet_ldl(a, num_blocks=4, out_of_core=True, scratch_dir=str(tmp_path))
    np.testing.assert_array_equal(res.perm, perm)
    assert rel_err(res.prefix, prefix) <= 1e-10
    g = np.random.default_rng(3).standard_normal((1100, 1100))
    lu = eng.memdet_lu(g, num_blocks=3, out_of_core=True, scratch_dir=str(tmp_path))
    s, ld = np.linalg.slogdet(g)
    assert lu.sign == s and abs(lu.logabsdet - ld) <= 1e-10 * abs(ld)
    eng.release_engine_cache()
