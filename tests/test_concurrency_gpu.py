"""Concurrent runs (reference SPEC.md:285: runs on distinct files may proceed in parallel) and
the block-local LU grid (advisor finding: the generic walk must keep the reference's blocks)."""

import threading

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


def _run_threads(jobs):
    out, errs = [None] * len(jobs), []

    def work(i, fn):
        try:
            out[i] = fn()
        except BaseException as e:  # noqa: BLE001 -- re-raised in the main thread
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i, fn)) for i, fn in enumerate(jobs)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out


def test_concurrent_runs_on_distinct_matrices_match_oracle():
    """Threads factoring different orders, drivers and blockings at the same time (and two on
    the same order, which must not share a workspace) each match the oracle."""
    mats = {m: gen.spd_wishart(m, m, seed=m, shift=1e-2) for m in (700, 1000, 1300)}
    refs = {m: O.memdet_cholesky(a, 3)[0] for m, a in mats.items()}
    ldl_ref = O.memdet_ldl(mats[1000], 4)
    jobs = []
    for rep in range(3):
        for m, a in mats.items():
            jobs.append(lambda a=a: ("chol", a.shape[0], eng.memdet_cholesky(a, num_blocks=3)))
        jobs.append(lambda: ("ldl", 1000, eng.memdet_ldl(mats[1000], num_blocks=4)))
        jobs.append(lambda: ("ooc", 1300, eng.memdet_cholesky(mats[1300], num_blocks=3, out_of_core=True)))
    for kind, m, res in _run_threads(jobs):
        if kind == "ldl":
            perm, prefix, signs, _ = ldl_ref
            np.testing.assert_array_equal(res.perm, perm)
            assert rel_err(res.prefix, prefix) <= 1e-10
        else:
            assert rel_err(res.prefix, refs[m]) <= 1e-10, (kind, m)


def test_release_while_running_keeps_the_running_workspace():
    """release_engine_cache() from another thread never frees a workspace in use."""
    a = gen.spd_wishart(1500, 1500, seed=9, shift=1e-2)
    ref = O.memdet_cholesky(a, 4)[0]
    stop = threading.Event()

    def releaser():
        while not stop.is_set():
            eng.release_engine_cache()

    t = threading.Thread(target=releaser)
    t.start()
    try:
        for _ in range(6):
            res = eng.memdet_cholesky(a, num_blocks=4)
            assert rel_err(res.prefix, ref) <= 1e-10
    finally:
        stop.set()
        t.join()


def test_lu_keeps_reference_blocks_anti_identity():
    """The anti-identity has a zero leading block under any grid finer than one block: the
    reference (one block, m > 6144) pivots across it and finds |det| = 1, so the engine must not
    refine the grid; it either matches or says it cannot (NotImplementedError), never -inf."""
    m = 6400
    a = np.fliplr(np.eye(m))
    with pytest.raises(NotImplementedError):
        eng.memdet_lu(a, num_blocks=1)
    # two blocks: the reference's leading 3200 block is zero -> singular (memdet.py:293-294)
    res = eng.memdet_lu(a, num_blocks=2)
    assert res.logabsdet == -np.inf and res.sign == 0
    # a grid the engine supports as given: m = 4096 in one block -> |det| = 1, sign of the reversal
    m2 = 4096
    r2 = eng.memdet_lu(np.fliplr(np.eye(m2)), num_blocks=1)
    assert abs(r2.logabsdet) <= 1e-12
    assert r2.sign == (-1) ** (m2 * (m2 - 1) // 2 % 2)
