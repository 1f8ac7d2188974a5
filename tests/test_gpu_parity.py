"""Parity of the CUDA engine (through the C ABI) with the reference.

Small cases compare against the golden vectors the unmodified reference produced
(tests/golden) and against the CPU oracle; the full-size C2 case compares against an
independent GPU factorisation (cuSOLVER via torch, used only as a checker) and through
size-independent properties (nested-generator prefixes, tiling invariance).
Tolerances (BASELINE.json north star): 1e-10 relative (denominator max(1,|x|)) in FP64 on
well-conditioned inputs, 1e-6 on the power-law (NTK-like) spectra, 1e-4 for float32 files
(the reference's own f32 bar, tests/test_memdet.py:247-256)."""

import hashlib
import os
import json

import numpy as np
import pytest

import paper_2503_04424_b200 as eng
from conftest import rel_err
from oracle import memdet_oracle as O
from paper_2503_04424_b200 import _native, gen

pytestmark = pytest.mark.gpu

TOL = {"ntk384": 1e-6, "spd40_f32": 1e-4}

SPD_CASES = ["spd1", "spd2", "spd5", "spd30", "spd48", "spd64", "spd120", "spd200", "eye50",
             "hand2", "spd40_f32", "rbf512", "ntk384", "C1"]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if _native.load().b2d_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    yield
    eng.release_engine_cache()


@pytest.mark.parametrize("name", SPD_CASES)
def test_cholesky_matches_reference_golden(golden, name):
    inp = golden.input(name)
    tol = TOL.get(name, 1e-10)
    for key in golden.cases[name]["runs"]:
        drv, nb = key.split("_nb")
        nb = int(nb)
        ref = golden.run(name, key)
        if drv == "chol":
            res = eng.memdet_cholesky(inp, num_blocks=nb)
            assert res.prefix.dtype == inp.dtype
            assert rel_err(res.prefix, ref["prefix"]) <= tol, (name, key, rel_err(res.prefix, ref["prefix"]))
            assert (res.info.n_b, res.info.b, res.info.blocks_read, res.info.blocks_written,
                    res.info.scratch_slots) == (ref["n_b"], ref["b"], ref["blocks_read"],
                                                ref["blocks_written"], ref["scratch_slots"])
            assert res.sign == 1
        else:
            # unpivoted LDL: natural-order prefixes equal the Cholesky ones everywhere and the
            # reference's pivoted LDL prefixes at block boundaries q = k*b and at q = m
            res = eng.memdet_ldl(inp, num_blocks=nb, pivoting="none")
            chol_ref = golden.run(name, f"chol_nb{nb}")["prefix"]
            assert rel_err(res.prefix, chol_ref) <= tol
            b = ref["b"]
            qs = sorted(set(list(range(b, len(inp) + 1, b)) + [len(inp)]))
            idx = np.array(qs) - 1
            assert rel_err(res.prefix[idx], ref["prefix"][idx]) <= tol, (name, key)
            assert list(res.perm) == list(range(len(inp)))
            np.testing.assert_allclose(res.d, np.asarray(res.d), rtol=0)


@pytest.mark.parametrize("name", ["notspd2", "sym24", "sym48", "sym120"])
def test_not_spd_raises_like_reference(golden, name):
    inp = golden.input(name)
    assert golden.run(name, "chol_nb1")["error"] == "NotSpdError"
    with pytest.raises(eng.NotSpdError):
        eng.memdet_cholesky(inp, num_blocks=1)


@pytest.mark.parametrize("m", [1, 2, 3, 127, 128, 129, 255, 256, 257, 383, 700, 1000])
def test_ragged_orders_vs_oracle(m):
    a = gen.spd_wishart(m, max(m, 8), seed=m, shift=1e-2)
    res = eng.memdet_cholesky(a, num_blocks=3)
    ref, info = O.memdet_cholesky(a, 3)
    assert rel_err(res.prefix, ref) <= 1e-10
    assert (res.info.n_b, res.info.blocks_read) == (info.n_b, info.blocks_read)
    d = res.d
    np.testing.assert_allclose(np.cumsum(2 * np.log(d)), ref, rtol=1e-10, atol=1e-10)


def test_input_unmodified_and_sidecar(tmp_path):
    a = gen.random_spd(300, seed=9)
    p = tmp_path / "a.mdm"
    eng.write_matrix(p, a, "spd")
    h0 = hashlib.sha256(open(p, "rb").read()).hexdigest()
    side = tmp_path / "a.pfx"
    res = eng.memdet_cholesky(p, num_blocks=5, prefix_out=side)
    assert hashlib.sha256(open(p, "rb").read()).hexdigest() == h0
    ell, sg = eng.read_prefix(side)
    np.testing.assert_array_equal(ell, res.prefix)
    assert np.all(sg == 1)


def test_tiling_invariance_is_exact():
    # the engine's tiling is independent of num_blocks: results are bit-identical
    a = gen.rbf(1000, seed=4)
    outs = [eng.memdet_cholesky(a, num_blocks=nb).prefix for nb in (1, 2, 3, 5, 8)]
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])
    outs2 = eng.memdet_cholesky(a, max_mem=8 * 300 * 300).prefix
    np.testing.assert_array_equal(outs2, outs[0])


def test_device_tensor_path_equals_host_path():
    torch = pytest.importorskip("torch")
    a = gen.rbf(1500, seed=6)
    host = eng.memdet_cholesky(a, num_blocks=4)
    t = torch.from_numpy(a).cuda()
    dev = eng.memdet_cholesky(t, num_blocks=4)
    np.testing.assert_array_equal(host.prefix, dev.prefix)
    assert torch.equal(t.cpu(), torch.from_numpy(a))  # input untouched


@pytest.mark.parametrize("nb,dtype", [(4, np.float64), (2, np.float32), (3, np.float64)])
def test_pivoted_ldl_device_tensor_equals_host(nb, dtype):
    """memdet_ldl on a CUDA tensor: tile-aligned blocks run in core straight from the device
    copy (nb = 4, 2); the others move it to host for the block walk (nb = 3); the result is the
    host path's bit for bit and the input is untouched."""
    torch = pytest.importorskip("torch")
    a = gen.random_symmetric(1024, seed=nb).astype(dtype)
    host = eng.memdet_ldl(a, num_blocks=nb)
    t = torch.from_numpy(a).cuda()
    dev = eng.memdet_ldl(t, num_blocks=nb)
    np.testing.assert_array_equal(host.perm, dev.perm)
    np.testing.assert_array_equal(host.prefix, dev.prefix)
    np.testing.assert_array_equal(host.prefix_signs, dev.prefix_signs)
    assert dev.info.out_of_core == (nb == 3)
    assert torch.equal(t.cpu(), torch.from_numpy(a))


def test_f32_matrix_file(tmp_path):
    a = gen.random_spd(200, seed=12).astype(np.float32)
    p = tmp_path / "f.mdm"
    eng.write_matrix(p, a, "spd")
    truth = float(np.sum(np.log(np.linalg.eigvalsh(a.astype(np.float64)))))
    res = eng.memdet_cholesky(p, num_blocks=3)
    assert res.prefix.dtype == np.float32
    assert res.logabsdet == pytest.approx(truth, rel=1e-4)


def test_device_rbf_generator_matches_host():
    torch = pytest.importorskip("torch")
    import ctypes

    n = 777
    x = gen.rbf_points(n, 16, seed=3)
    host = gen.rbf(n, x=x)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty((n, n), dtype=torch.float64, device="cuda")
    _native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(xd.data_ptr()), n, 16, 4.0, 1e-6,
                                             ctypes.c_void_p(out.data_ptr()), None))
    torch.cuda.synchronize()
    dev = out.cpu().numpy()
    np.testing.assert_array_equal(dev, dev.T)
    assert np.max(np.abs(dev - host)) <= 4e-16


@pytest.mark.slow
def test_c2_full_size_vs_independent_gpu_factorisation():
    """C2 (n=32768 RBF) at full size: every prefix against cuSOLVER's potrf (checker only),
    plus the nested-generator property prefix_C2[:4096] == prefix(rbf(4096))."""
    torch = pytest.importorskip("torch")
    import ctypes

    n = 32768
    x = gen.rbf_points(n, 16, seed=0)
    xd = torch.from_numpy(x).cuda()
    a = torch.empty((n, n), dtype=torch.float64, device="cuda")
    _native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(xd.data_ptr()), n, 16, 4.0, 1e-6,
                                             ctypes.c_void_p(a.data_ptr()), None))
    torch.cuda.synchronize()
    res = eng.memdet_cholesky(a, num_blocks=8)
    eng.release_engine_cache()
    low = torch.linalg.cholesky(a)
    ref = torch.cumsum(2.0 * torch.log(torch.diagonal(low)), 0).cpu().numpy()
    del low
    assert rel_err(res.prefix, ref) <= 1e-10, rel_err(res.prefix, ref)
    small = eng.memdet_cholesky(a[:4096, :4096].contiguous(), num_blocks=1)
    assert rel_err(res.prefix[:4096], small.prefix) <= 1e-12


@pytest.mark.slow
def test_c2_full_size_matches_reference_golden():
    """C2 at full size against the UNMODIFIED reference's own outputs on the same bytes
    (tests/golden/c2.*, made by make_c2_golden.py): the host input is regenerated here and its
    SHA-256 must equal the one the reference factored; then every memdet_cholesky prefix and
    every memdet_ldl prefix within 1e-10 (north star), and the LDL pivots and signs."""
    path = os.path.join(os.path.dirname(__file__), "golden", "c2.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c2.json not generated")
    with open(path) as f:
        meta = json.load(f)
    ref = np.load(os.path.join(os.path.dirname(__file__), "golden", "c2.npz"))
    a = gen.rbf(meta["m"], seed=0, threads=os.cpu_count() or 1)
    h = hashlib.sha256()
    for r0 in range(0, a.shape[0], 1024):
        h.update(np.ascontiguousarray(a[r0:r0 + 1024]).tobytes())
    assert h.hexdigest() == meta["input_sha256"]
    chol = eng.memdet_cholesky(a, num_blocks=meta["num_blocks"])
    assert rel_err(chol.prefix, ref["chol__prefix"]) <= 1e-10, rel_err(chol.prefix, ref["chol__prefix"])
    ldl = eng.memdet_ldl(a, num_blocks=meta["num_blocks"])
    eng.release_engine_cache()
    assert rel_err(ldl.prefix, ref["ldl__prefix"]) <= 1e-10, rel_err(ldl.prefix, ref["ldl__prefix"])
    np.testing.assert_array_equal(ldl.perm, ref["ldl__perm"])
    np.testing.assert_array_equal(ldl.prefix_signs, ref["ldl__signs"])
    for r, res in (("chol", chol), ("ldl", ldl)):
        info = meta["runs"][r]
        assert (res.info.n_b, res.info.b) == (info["n_b"], info["b"])
        assert (res.info.blocks_read, res.info.blocks_written, res.info.scratch_slots) == \
            (info["blocks_read"], info["blocks_written"], info["scratch_slots"])


# ------------------------------------------------------------------ out-of-core block streamer


@pytest.mark.parametrize("m,nb", [(700, 3), (1000, 4), (1536, 4), (2000, 5), (640, 1), (900, 2)])
def test_out_of_core_matches_oracle_and_reference_counters(m, nb):
    """Forced out-of-core: the reference tile walk over HBM slots; every prefix matches the
    oracle and the block transfers equal the reference's own counters (cost.py:79-101)."""
    a = gen.spd_wishart(m, m, seed=100 + m, shift=1e-2)
    res = eng.memdet_cholesky(a, num_blocks=nb, out_of_core=True)
    ref, info = O.memdet_cholesky(a, nb)
    assert res.info.out_of_core
    assert rel_err(res.prefix, ref) <= 1e-10, rel_err(res.prefix, ref)
    assert res.info.ooc_blocks == info.n_b
    assert (res.info.ooc_reads, res.info.ooc_writes, res.info.ooc_scratch) == \
        (info.blocks_read, info.blocks_written, info.scratch_slots)
    # and the same numbers as the in-core engine, to rounding
    inc = eng.memdet_cholesky(a, num_blocks=nb)
    assert not inc.info.out_of_core
    assert rel_err(res.prefix, inc.prefix) <= 1e-12


def test_out_of_core_golden_c1(golden):
    """C1 (n=4096, num_blocks=4) through the out-of-core streamer vs the reference's prefixes."""
    inp = golden.input("C1")
    ref = golden.run("C1", "chol_nb4")
    res = eng.memdet_cholesky(inp, num_blocks=4, out_of_core=True)
    assert rel_err(res.prefix, ref["prefix"]) <= 1e-10
    assert (res.info.ooc_reads, res.info.ooc_writes, res.info.ooc_scratch) == \
        (ref["blocks_read"], ref["blocks_written"], ref["scratch_slots"])


def test_out_of_core_budget_planner_grows_grid():
    """A tiny HBM budget forces a finer grid than the requested num_blocks; results unchanged."""
    a = gen.rbf(1500, seed=8)
    res = eng.memdet_cholesky(a, num_blocks=2, hbm_budget=20 << 20,
                              out_of_core=True)
    assert res.info.ooc_blocks > 2
    ref, _ = O.memdet_cholesky(a, 2)
    assert rel_err(res.prefix, ref) <= 1e-10


def test_out_of_core_not_spd():
    a = gen.random_symmetric(500, seed=3)
    with pytest.raises(eng.NotSpdError):
        eng.memdet_cholesky(a, num_blocks=3, out_of_core=True)


# ------------------------------------------------------------------ multi-rank driver on the GPU


def _dist_worker(rank, world, port, backend, m, panel, peer, q, host=False):
    import os
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    kw = dict(device_id=torch.device("cuda", 0)) if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    from paper_2503_04424_b200 import gen
    from paper_2503_04424_b200.distributed import memdet_cholesky_distributed

    a = gen.spd_wishart(m, m, seed=11, shift=1e-2)
    if not host:
        a = torch.from_numpy(a).cuda()
    prefix, fail = memdet_cholesky_distributed(a, panel_tiles=panel, peer=peer)
    q.put((rank, prefix, fail))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,backend,m,panel,peer,host", [(1, "nccl", 1000, 4, None, False),
                                                             (2, "gloo", 1000, 3, False, False),
                                                             (3, "gloo", 777, 2, False, False),
                                                             (2, "gloo", 1000, 3, True, False),
                                                             (3, "gloo", 900, 2, True, False),
                                                             (2, "gloo", 1000, 3, True, True),
                                                             (3, "gloo", 777, 2, True, True),
                                                             (3, "gloo", 900, 2, False, True)])
def test_distributed_driver_cuda_tile_ops(world, backend, m, panel, peer, host):
    """The row-cyclic multi-GPU driver with the real CUDA tile kernels.  One GPU is available,
    so world > 1 runs several ranks on cuda:0 with gloo (collectives and barriers are host-side,
    no rank waits on another's kernels); world = 1 exercises the NCCL path.  peer=True is the
    product exchange: every rank's grid is cudaMalloc'd, mapped into the other ranks with CUDA
    IPC, and the Schur-update kernels read the owners' solved panel tiles in place.  host=True:
    each rank ingests only its own tile rows from a host array (sharded ingest, no replica)."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, backend, m, panel, peer, q, host))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref, _ = O.memdet_cholesky(gen.spd_wishart(m, m, seed=11, shift=1e-2), 1)
    for rank, prefix, fail in results:
        assert fail == -1
        assert rel_err(prefix, ref) <= 1e-10, (rank, rel_err(prefix, ref))


# ------------------------------------------------------------------ block-pivoted LDL (memdet_ldl)

LDL_CASES = ["spd1", "spd2", "spd5", "spd30", "spd48", "spd64", "spd120", "spd200", "sym24", "sym30",
             "sym48", "sym64", "sym120", "eye50", "diag8", "hand2", "hardindef2", "spd40_f32",
             "rbf512", "ntk384", "C1"]


@pytest.mark.parametrize("name", LDL_CASES)
def test_pivoted_ldl_matches_reference_golden(golden, name):
    """memdet_ldl with the reference's block-local 1x1 pivoting: perm and signs exactly, every
    permuted-minor prefix within tolerance, IndefiniteBlockError where the reference raises."""
    inp = golden.input(name)
    tol = TOL.get(name, 1e-10)
    for key in golden.cases[name]["runs"]:
        drv, nb = key.split("_nb")
        if drv != "ldl":
            continue
        nb = int(nb)
        ref = golden.run(name, key)
        if ref.get("error") == "IndefiniteBlockError":
            with pytest.raises(eng.IndefiniteBlockError):
                eng.memdet_ldl(inp, num_blocks=nb)
            continue
        res = eng.memdet_ldl(inp, num_blocks=nb)
        np.testing.assert_array_equal(res.perm, ref["perm"], err_msg=f"{name} {key}")
        np.testing.assert_array_equal(res.prefix_signs, ref["signs"], err_msg=f"{name} {key}")
        assert rel_err(res.prefix, ref["prefix"]) <= tol, (name, key, rel_err(res.prefix, ref["prefix"]))
        assert res.prefix.dtype == inp.dtype
        assert (res.info.blocks_read, res.info.blocks_written, res.info.scratch_slots) == \
            (ref["blocks_read"], ref["blocks_written"], ref["scratch_slots"])
        if res.info.out_of_core:  # the block walk makes exactly the reference's transfers
            assert (res.info.ooc_reads, res.info.ooc_writes, res.info.ooc_scratch) == \
                (ref["blocks_read"], ref["blocks_written"], ref["scratch_slots"])


@pytest.mark.parametrize("m,nb", [(1024, 4), (1022, 4), (1280, 5), (768, 2), (2048, 8), (700, 1), (1536, 12)])
@pytest.mark.parametrize("kchunk", ["8", "1"])
@pytest.mark.parametrize("sched", ["rows", "cols"])
def test_pivoted_ldl_in_core_equals_block_walk(m, nb, kchunk, sched, monkeypatch):
    """B2D_REST_KCHUNK splits the trailing update over K into sequential launches (1 = one
    tile-column each), which must not change a bit; neither may the stage schedule
    (B2D_LDL_ROWS: block rows by distance on prioritised streams, or block columns).
    Tile-aligned reference blocks run in core (the matrix resident, one large update per
    stage, the next block's factor overlapped); every tile gets the walk's updates with the same
    operands and K, so perm, D and the prefixes equal the out-of-core block walk's bit for bit,
    and the walk makes the reference's transfers."""
    monkeypatch.setenv("B2D_REST_KCHUNK", kchunk)
    monkeypatch.setenv("B2D_LDL_ROWS", "1" if sched == "rows" else "0")
    eng.release_engine_cache()
    a = gen.random_symmetric(m, seed=m + nb)
    res = eng.memdet_ldl(a, num_blocks=nb)
    walk = eng.memdet_ldl(a, num_blocks=nb, out_of_core=True)
    assert not res.info.out_of_core and walk.info.out_of_core
    np.testing.assert_array_equal(res.perm, walk.perm)
    np.testing.assert_array_equal(res.prefix_signs, walk.prefix_signs)
    assert np.array_equal(res.prefix.view(np.int64), walk.prefix.view(np.int64)), \
        np.max(np.abs(res.prefix - walk.prefix))
    ref_perm, ref_prefix, ref_signs, rinfo = O.memdet_ldl(a, nb)
    np.testing.assert_array_equal(res.perm, ref_perm)
    assert rel_err(res.prefix, ref_prefix) <= 1e-10
    assert (walk.info.ooc_reads, walk.info.ooc_writes) == (rinfo.blocks_read, rinfo.blocks_written)
    eng.release_engine_cache()


@pytest.mark.parametrize("m,nb", [(2048, 2), (2560, 2), (3072, 3), (1024, 4)])
@pytest.mark.parametrize("la", ["0", "1", "3", "4"])
@pytest.mark.parametrize("sched", ["rows", "cols"])
def test_pivoted_ldl_lookahead_solve_equals_block_walk(m, nb, la, sched, monkeypatch):
    """B2D_LDL_LA: the rows of block k+1 solved in groups of `la` tile-columns with look-ahead
    (the chain on one stream, the rest of each group's updates and the group's K-chunk of the
    diagonal update on two others).  Every tile still receives its K-chunks in increasing order,
    so perm, D and the prefixes equal the block walk's bit for bit."""
    monkeypatch.setenv("B2D_LDL_LA", la)
    monkeypatch.setenv("B2D_LDL_ROWS", "1" if sched == "rows" else "0")
    eng.release_engine_cache()
    a = gen.random_symmetric(m, seed=m + 7 * nb)
    res = eng.memdet_ldl(a, num_blocks=nb)
    walk = eng.memdet_ldl(a, num_blocks=nb, out_of_core=True)
    assert not res.info.out_of_core and walk.info.out_of_core
    np.testing.assert_array_equal(res.perm, walk.perm)
    np.testing.assert_array_equal(res.prefix_signs, walk.prefix_signs)
    assert np.array_equal(res.prefix.view(np.int64), walk.prefix.view(np.int64)), \
        np.max(np.abs(res.prefix - walk.prefix))
    eng.release_engine_cache()


@pytest.mark.parametrize("m,nb", [(2048, 2), (2560, 2), (3072, 3), (2560, 4), (3840, 5)])
@pytest.mark.parametrize("groups,front,ue", [("0", "1", "2"), ("1", "1", "1"), ("2", "1", "2"), ("4", "1", "2"),
                                             ("4", "0", "2"), ("3", "1", "3")])
def test_pivoted_ldl_group_pipeline_equals_block_walk(m, nb, groups, front, ue, monkeypatch):
    """B2D_LDL_GROUPS: the factors hand out their finished column groups (L tile rows, tile
    inverses, permutation entries) while they run; stage 0's block rows (B2D_LDL_FRONT) and every
    stage's chain row solve and apply them group by group (far rows every B2D_LDL_FRONT_UE
    groups).  Every entry still receives its terms in increasing k, so perm, D and the prefixes
    equal the block walk's (and the whole-panel schedule's, groups = 0) bit for bit."""
    monkeypatch.setenv("B2D_LDL_GROUPS", groups)
    monkeypatch.setenv("B2D_LDL_FRONT", front)
    monkeypatch.setenv("B2D_LDL_FRONT_UE", ue)
    eng.release_engine_cache()
    a = gen.random_symmetric(m, seed=3 * m + nb)
    res = eng.memdet_ldl(a, num_blocks=nb)
    again = eng.memdet_ldl(a, num_blocks=nb)  # event / buffer reuse across runs of one context
    walk = eng.memdet_ldl(a, num_blocks=nb, out_of_core=True)
    assert not res.info.out_of_core and walk.info.out_of_core
    for r in (res, again):
        np.testing.assert_array_equal(r.perm, walk.perm)
        np.testing.assert_array_equal(r.prefix_signs, walk.prefix_signs)
        assert np.array_equal(r.prefix.view(np.int64), walk.prefix.view(np.int64)), \
            np.max(np.abs(r.prefix - walk.prefix))
    ref_perm, ref_prefix, _, _ = O.memdet_ldl(a, nb)
    np.testing.assert_array_equal(res.perm, ref_perm)
    assert rel_err(res.prefix, ref_prefix) <= 1e-10
    eng.release_engine_cache()


@pytest.mark.parametrize("m,nb", [(1022, 4), (768, 3)])
def test_in_core_f32_inputs_equal_block_walk(m, nb, monkeypatch):
    """float32 inputs converted to FP64 on the device (B2D_F32_ARITH=0 for the LDL; the default
    float32 arithmetic is tests/test_f32_gpu.py's) through the in-core LDL and LU equal the block
    walks bit for bit."""
    monkeypatch.setenv("B2D_F32_ARITH", "0")
    eng.release_engine_cache()
    a = gen.random_symmetric(m, seed=m).astype(np.float32)
    r1, r2 = eng.memdet_ldl(a, num_blocks=nb), eng.memdet_ldl(a, num_blocks=nb, out_of_core=True)
    assert not r1.info.out_of_core and r2.info.out_of_core
    np.testing.assert_array_equal(r1.perm, r2.perm)
    np.testing.assert_array_equal(r1.prefix, r2.prefix)
    assert r1.prefix.dtype == np.float32
    g = (np.random.default_rng(m).standard_normal((m, m)) + 2.0 * np.sqrt(m) * np.eye(m)).astype(np.float32)
    u1, u2 = eng.memdet_lu(g, num_blocks=nb), eng.memdet_lu(g, num_blocks=nb, out_of_core=True)
    assert not u1.info.out_of_core and u2.info.out_of_core
    assert (u1.sign, u1.logabsdet) == (u2.sign, u2.logabsdet)
    eng.release_engine_cache()


def test_pivoted_ldl_in_core_failing_block_matches_walk():
    """A zero diagonal block at stage 2 (the Schur complement of a block-diagonal matrix):
    in core and the block walk raise IndefiniteBlockError at the same global pivot, as the
    reference's block-local pivoting does."""
    m, nb = 1024, 4
    a = gen.random_symmetric(m, seed=9)
    a[512:768, :] = 0.0
    a[:, 512:768] = 0.0
    msgs = []
    for ooc in (None, True):
        with pytest.raises(eng.IndefiniteBlockError) as e:
            eng.memdet_ldl(a, num_blocks=nb, out_of_core=ooc)
        msgs.append(str(e.value).split(":")[0])
    assert msgs[0] == msgs[1] and msgs[0] == "LDL pivot 512 below tolerance", msgs


def test_lu_in_core_singular_block_matches_walk():
    """A zero diagonal block at stage 2: (-inf, 0) in core and through the walk, with the
    reference's counters of a walk that stops at stage 2 (memdet.py:293-294)."""
    m, nb = 1024, 4
    rng = np.random.default_rng(3)
    a = rng.standard_normal((m, m)) + 2.0 * np.sqrt(m) * np.eye(m)
    a[512:768, 512:768] = 0.0
    a[512:768, :512] = 0.0
    a[:512, 512:768] = 0.0
    r1 = eng.memdet_lu(a, num_blocks=nb)
    r2 = eng.memdet_lu(a, num_blocks=nb, out_of_core=True)
    assert not r1.info.out_of_core and r2.info.out_of_core
    assert (r1.sign, r1.logabsdet) == (0, -np.inf) == (r2.sign, r2.logabsdet)
    assert (r1.info.blocks_read, r1.info.blocks_written, r1.info.scratch_slots) == \
        (r2.info.blocks_read, r2.info.blocks_written, r2.info.scratch_slots)


def _ldl_block_input(m, kind):
    rng = np.random.default_rng(m)
    if kind == "sym":
        return gen.random_symmetric(m, seed=m)
    if kind == "rbf":  # equal diagonal: an exact tie at the first step
        return gen.rbf(m, seed=m)
    if kind == "blocks":  # identical diagonal blocks: exact ties at every step
        b = gen.random_symmetric(16, seed=3)
        return np.kron(np.eye(m // 16), b)
    if kind == "int":  # small integers: many exactly equal candidates
        g = rng.integers(-3, 4, size=(m, m)).astype(np.float64)
        a = np.tril(g) + np.tril(g, -1).T
        a[np.diag_indices(m)] = rng.integers(5, 9, size=m) * np.where(rng.random(m) < 0.5, -1.0, 1.0)
        return a
    raise ValueError(kind)


@pytest.mark.parametrize("panel", ["cluster", "single_cta", "persistent"])
@pytest.mark.parametrize("m,kind", [(31, "sym"), (33, "sym"), (100, "sym"), (257, "sym"), (700, "sym"),
                                    (600, "rbf"), (320, "blocks"), (400, "int")])
def test_pivoted_ldl_diagonal_block_bit_identical_to_reference_kernel(m, kind, panel, monkeypatch):
    """One diagonal block (num_blocks=1): the blocked panel / delayed-update kernels reproduce the
    reference's unblocked loop (_ldl.pyx:21-61, restated in oracle/ldl_tile.c) bit for bit:
    the same interchanges and the same pivots d, across panel boundaries and exact ties; all
    three forms (per-panel 16-CTA cluster kernels, the one-launch cluster factor used beside
    the trailing updates, and the one-CTA kernel used above 6144 rows)."""
    if panel == "single_cta":
        monkeypatch.setenv("B2D_LDL_SINGLE_CTA", "1")
    if panel == "persistent":
        monkeypatch.setenv("B2D_LDL_PERSIST", "2")
    else:
        monkeypatch.setenv("B2D_LDL_PERSIST", "0")
    a = _ldl_block_input(m, kind)
    ctx = _native.Context(m, _native.MODE_LDL_PIV, num_blocks=1)
    ctx.factor_host_async(a.ctypes.data, m, _native.B2D_F64, 0)
    d = np.empty(m)
    rc, fail, info = ctx.fetch(d, None)
    _native.check(rc)
    perm = np.empty(m, np.int64)
    ctx.fetch_perm(perm)
    ctx.close()
    swaps, dref = O.ldl_tile(a.copy())
    np.testing.assert_array_equal(perm, O.perm_from_swaps(swaps))
    assert np.array_equal(d.view(np.int64), np.asarray(dref, np.float64).view(np.int64)), \
        np.max(np.abs(d - dref))


def test_pivoted_ldl_prefix_is_permuted_minor_logdet():
    """reference tests/test_memdet.py:117-129: prefix[q-1] = log|det M[perm[:q], perm[:q]]|."""
    m = 48
    a = gen.random_symmetric(m, seed=5)
    for nb in (1, 2, 4):
        res = eng.memdet_ldl(a, num_blocks=nb)
        assert sorted(res.perm) == list(range(m))
        for q in range(1, m + 1):
            idx = res.perm[:q]
            sign, ld = np.linalg.slogdet(a[np.ix_(idx, idx)])
            assert res.prefix_signs[q - 1] == int(sign)
            assert res.prefix[q - 1] == pytest.approx(ld, rel=1e-9, abs=1e-9)


def test_gram_formation_in_packed_context_matches_dense():
    """K = G G^T / n + jitter I formed in the packed tiles by the engine's DMMA kernel, then
    factored in place, equals the engine's factorisation of the same K formed densely by cuBLAS."""
    torch = pytest.importorskip("torch")
    import ctypes

    n, k = 1000, 3000
    ctx = _native.Context(n)
    gen.gram_into_context(ctx, n, k, 1.0 / n, 1e-4, seed=5, chunk=1024)
    _native.check(_native.load().b2d_ctx_factor_packed_async(ctx.handle, None))
    pre = np.empty(n)
    rc, fail, info = ctx.fetch(None, pre)
    _native.check(rc)
    ctx.close()
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    dense = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    for c0 in range(0, k, 1024):
        z = torch.randn((n, min(k, c0 + 1024) - c0), dtype=torch.float64, device="cuda", generator=g)
        dense.addmm_(z, z.T)
    dense.div_(n)
    dense.diagonal().add_(1e-4)
    ref, _ = O.memdet_cholesky(dense.cpu().numpy(), 1)
    assert rel_err(pre, ref) <= 1e-10, rel_err(pre, ref)


@pytest.mark.parametrize("host_scratch", [False, True])
def test_out_of_core_scratch_placement(host_scratch):
    """Scratchpad in HBM (fits) or pinned host memory: same walk, same numbers, same counters."""
    m, nb = 1100, 5
    a = gen.rbf(m, seed=21)
    ctx = _native.Context(m, num_blocks=nb, force_out_of_core=True, host_scratch=host_scratch)
    assert ctx.out_of_core and ctx.scratch_on_device == (not host_scratch)
    ctx.factor_host_async(a.ctypes.data, m, _native.B2D_F64, 0)
    pre = np.empty(m)
    rc, fail, info = ctx.fetch(None, pre)
    _native.check(rc)
    ctx.close()
    ref, rinfo = O.memdet_cholesky(a, nb)
    assert rel_err(pre, ref) <= 1e-10
    assert (info.ooc_reads, info.ooc_writes, info.ooc_scratch) == (rinfo.blocks_read, rinfo.blocks_written,
                                                                    rinfo.scratch_slots)


# ------------------------------------------------------------------ generic LU (memdet_lu)


def test_lu_matches_reference_golden():
    """memdet_lu against the unmodified reference (tests/golden/lu.*): log|det| within 1e-10
    (1e-4 for the float32 file, the reference's f32 bar), the sign exactly, the reference's
    block counters; (-inf, 0) where block-local pivoting meets a singular diagonal block.
    The exactly rank-deficient matrix's finite value is roundoff (it differs across the
    reference's own block counts), so it is not compared."""
    import json
    import os

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(here, "lu.json")) as f:
        cases = json.load(f)["cases"]
    arrays = np.load(os.path.join(here, "lu.npz"))
    for c in cases:
        a = arrays[c["name"]]
        tol = 1e-4 if a.dtype == np.float32 else 1e-10
        for nb, ref in c["runs"].items():
            res = eng.memdet_lu(a, num_blocks=int(nb))
            key = (c["name"], nb)
            if c["name"].startswith("singular"):
                # exact rank deficiency: whether elimination meets an exact zero pivot (det = 0,
                # the walk stops) or a roundoff-sized one depends on the arithmetic order
                assert res.sign == 0 or np.isfinite(res.logabsdet), key
                continue
            assert (res.info.n_b, res.info.b, res.info.blocks_read, res.info.blocks_written,
                    res.info.scratch_slots) == (ref["n_b"], ref["b"], ref["blocks_read"], ref["blocks_written"],
                                                ref["scratch_slots"]), key
            if ref["sign"] == 0:
                assert res.sign == 0 and res.logabsdet == -np.inf, key
                continue
            assert res.sign == ref["sign"], key
            assert abs(res.logabsdet - ref["logabsdet"]) <= tol * max(1.0, abs(ref["logabsdet"])), \
                (key, res.logabsdet, ref["logabsdet"])


@pytest.mark.parametrize("m,nb", [(1024, 4), (1022, 4), (1280, 5), (2048, 2), (700, 1)])
@pytest.mark.parametrize("kchunk", ["8", "1"])
def test_lu_in_core_equals_block_walk(m, nb, kchunk, monkeypatch):
    """B2D_REST_KCHUNK = 1 splits the trailing update over K into one launch per tile-column.
    Tile-aligned reference blocks run in core (full tile grid resident, one large update per
    stage, the next block's factor overlapped): every tile gets the walk's updates with the
    same operands and K, so log|det|, the sign and the pivots equal the generic walk's bit for
    bit, and agree with numpy's slogdet."""
    monkeypatch.setenv("B2D_REST_KCHUNK", kchunk)
    rng = np.random.default_rng(m + nb)
    a = rng.standard_normal((m, m)) + 2.0 * np.sqrt(m) * np.eye(m)
    a[::3] *= -1.0
    res = eng.memdet_lu(a, num_blocks=nb)
    walk = eng.memdet_lu(a, num_blocks=nb, out_of_core=True)
    assert not res.info.out_of_core and walk.info.out_of_core
    assert res.sign == walk.sign and res.logabsdet == walk.logabsdet, (res.logabsdet, walk.logabsdet)
    sign, ref = np.linalg.slogdet(a)
    assert res.sign == int(sign)
    assert abs(res.logabsdet - ref) <= 1e-10 * abs(ref)
    assert (res.info.blocks_read, res.info.blocks_written) == (walk.info.blocks_read, walk.info.blocks_written)


@pytest.mark.parametrize("m,nb", [(3000, 2), (2900, 3), (5000, 1)])
def test_lu_larger_vs_slogdet(m, nb):
    """Several 32-column panels per block, ragged blocks, the 16-CTA panel at 5000 rows."""
    rng = np.random.default_rng(m)
    a = rng.standard_normal((m, m)) + 3.0 * np.sqrt(m) * np.eye(m)
    a[: m // 2] *= -1.0
    sign, ref = np.linalg.slogdet(a)
    res = eng.memdet_lu(a, num_blocks=nb)
    assert res.sign == int(sign)
    assert abs(res.logabsdet - ref) <= 1e-10 * abs(ref)


# ------------------------------------------------------------------ Ozaki (int8 tcgen05) Schur updates


@pytest.mark.parametrize("m", [4096, 6000, 9000])
def test_ozaki_schur_matches_dmma_and_oracle(m):
    """schur="ozaki": the trailing updates emulated on the int8 tensor cores agree with the
    FP64 DMMA path to 1e-12 and with the CPU oracle to 1e-10 on every prefix."""
    a = gen.rbf(m, seed=m)
    ref, _ = O.memdet_cholesky(a, 4)
    dm = eng.memdet_cholesky(a, num_blocks=4)
    oz = eng.memdet_cholesky(a, num_blocks=4, schur="ozaki")
    eng.release_engine_cache()
    assert rel_err(oz.prefix, dm.prefix) <= 1e-12, rel_err(oz.prefix, dm.prefix)
    assert rel_err(oz.prefix, ref) <= 1e-10, rel_err(oz.prefix, ref)
    assert oz.info.kernel_launches > dm.info.kernel_launches  # the slice kernels ran


@pytest.mark.slow
def test_ozaki_c2_full_size_vs_independent_gpu_factorisation():
    """C2 (n = 32768 RBF) with the int8-emulated Schur updates: every prefix within 1e-10 of
    cuSOLVER's potrf (checker only)."""
    torch = pytest.importorskip("torch")
    import ctypes

    n = 32768
    xd = torch.from_numpy(gen.rbf_points(n, 16, seed=0)).cuda()
    a = torch.empty((n, n), dtype=torch.float64, device="cuda")
    _native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(xd.data_ptr()), n, 16, 4.0, 1e-6,
                                             ctypes.c_void_p(a.data_ptr()), None))
    torch.cuda.synchronize()
    res = eng.memdet_cholesky(a, num_blocks=8, schur="ozaki")
    eng.release_engine_cache()
    low = torch.linalg.cholesky(a)
    ref = torch.cumsum(2.0 * torch.log(torch.diagonal(low)), 0).cpu().numpy()
    del low
    assert rel_err(res.prefix, ref) <= 1e-10, rel_err(res.prefix, ref)


# ------------------------------------------------------------------ pageable (file) inputs


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_memdet01_file_input_staged_equals_pinned(tmp_path, dtype, monkeypatch):
    """A MEMDET01 file (memory-mapped: pageable host memory, the reference's own input form)
    goes through the pinned staging buffers filled by host threads; the bytes, hence every
    result, must equal the pinned-input run and the driver's own pageable copies
    (B2D_HOST_STAGING=0): Cholesky (in core and forced out of core), pivoted LDL, LU."""
    torch = pytest.importorskip("torch")
    from paper_2503_04424_b200.storage import write_matrix

    m = 2304  # 128-row strips of 2.4 MB (f64): above the staging threshold
    spd = gen.spd_wishart(m, m, seed=7, shift=1e-2).astype(dtype)
    sym = gen.random_symmetric(m, seed=8).astype(dtype)
    gen_m = (np.random.default_rng(9).standard_normal((m, m)) + 2.0 * np.sqrt(m) * np.eye(m)).astype(dtype)
    ps, py, pg = tmp_path / "spd.mdm", tmp_path / "sym.mdm", tmp_path / "gen.mdm"
    write_matrix(ps, spd, "spd")
    write_matrix(py, sym, "symmetric")
    write_matrix(pg, gen_m, "generic")

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64 if dtype == np.float64 else torch.float32, pin_memory=True)
        t.numpy()[:] = a
        return t.numpy()

    runs = {
        "chol": (lambda x: eng.memdet_cholesky(x, num_blocks=3).prefix, ps, spd),
        "chol_ooc": (lambda x: eng.memdet_cholesky(x, num_blocks=3, out_of_core=True).prefix, ps, spd),
        "ldl": (lambda x: eng.memdet_ldl(x, num_blocks=3).prefix, py, sym),
        "lu": (lambda x: np.array([eng.memdet_lu(x, num_blocks=3).logabsdet]), pg, gen_m),
    }
    for name, (f, path, arr) in runs.items():
        monkeypatch.setenv("B2D_HOST_STAGING", "1")
        staged = f(str(path))
        ref = f(pinned(arr))
        monkeypatch.setenv("B2D_HOST_STAGING", "0")
        driver = f(str(path))
        eng.release_engine_cache()
        assert np.array_equal(staged.view(np.uint8), ref.view(np.uint8)), name
        assert np.array_equal(staged.view(np.uint8), driver.view(np.uint8)), name


@pytest.mark.parametrize("m", [8192, 6016])
@pytest.mark.parametrize("gbs", ["0.5", "4", "50"])
def test_pinned_input_eager_band_catch_up_is_bit_identical(m, gbs, monkeypatch):
    """B2D_EAGER_CATCH (pinned host input): a band that joins the right-looking updates at step s
    takes the panels of steps < s one by one as they are solved (low-priority streams) instead
    of one catch-up GEMM when it joins.  Same k order, exact FP64 continuation: every prefix must
    equal the one-catch-up schedule's and the device-resident path's bit for bit.  A slow modelled
    PCIe rate (B2D_PCIE_GBS) makes the band plan join bands late, so pieces are really issued."""
    torch = pytest.importorskip("torch")
    a = gen.spd_wishart(m, m, seed=11, shift=1e-2)
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = a
    monkeypatch.setenv("B2D_PCIE_GBS", gbs)
    monkeypatch.setenv("B2D_STAGE_GBS", gbs)
    out = {}
    # pinned: every strip enqueued up front, one piece per solved panel; pageable (a plain ndarray,
    # staged): strips enqueued band by band, a band's first piece covers the panels solved so far
    for kind, inp in (("pinned", t.numpy()), ("pageable", a)):
        for eager in ("1", "0"):
            monkeypatch.setenv("B2D_EAGER_CATCH", eager)
            eng.release_engine_cache()
            first = eng.memdet_cholesky(inp, num_blocks=4).prefix
            again = eng.memdet_cholesky(inp, num_blocks=4).prefix  # events / streams reused
            assert np.array_equal(first.view(np.int64), again.view(np.int64)), (kind, eager)
            out[kind, eager] = first
    dev = eng.memdet_cholesky(t.cuda(), num_blocks=4).prefix
    eng.release_engine_cache()
    for key, val in out.items():
        assert np.array_equal(val.view(np.int64), dev.view(np.int64)), (key, np.max(np.abs(val - dev)))
    out = {"1": out["pinned", "1"]}
    ref, _ = O.memdet_cholesky(a, 4)
    assert rel_err(out["1"], ref) <= 1e-10


def test_pivoted_ldl_out_of_core_keeps_reference_blocks():
    """The out-of-core planner may refine the block grid for Cholesky (results do not depend on
    it), never for the block-pivoted LDL, whose pivots are searched inside the reference's
    blocks: under a budget its walk cannot meet it fails loudly instead of pivoting over other
    blocks; with room, perm and prefixes are the reference's."""
    a = gen.random_symmetric(1536, seed=12)
    with pytest.raises(MemoryError, match="keeps the reference's"):
        eng.memdet_ldl(a, num_blocks=2, hbm_budget=20 << 20, out_of_core=True)
    res = eng.memdet_ldl(a, num_blocks=2, hbm_budget=1 << 30, out_of_core=True)
    ref_perm, ref_prefix, _, _ = O.memdet_ldl(a, 2)
    np.testing.assert_array_equal(res.perm, ref_perm)
    assert rel_err(res.prefix, ref_prefix) <= 1e-10


@pytest.mark.parametrize("m,nb", [(8192, 1), (13000, 2)])
def test_pivoted_ldl_big_blocks_cluster_equals_one_cta(m, nb, monkeypatch):
    """Reference blocks above the shared-memory cluster panel's 16 x 384 rows (the paper's
    memory-sized blocks) run on the big-block cluster panel (the rows' C / W histories in global
    memory); it must reproduce the one-CTA panel (B2D_LDL_BIG=0, itself pinned to the oracle on
    smaller blocks) bit for bit: perm, prefix and signs."""
    a = gen.rbf(m, seed=m)
    eng.release_engine_cache()
    big = eng.memdet_ldl(a, num_blocks=nb)
    monkeypatch.setenv("B2D_LDL_BIG", "0")
    eng.release_engine_cache()
    one = eng.memdet_ldl(a, num_blocks=nb)
    eng.release_engine_cache()
    np.testing.assert_array_equal(big.perm, one.perm)
    np.testing.assert_array_equal(big.prefix_signs, one.prefix_signs)
    assert np.array_equal(big.prefix.view(np.int64), one.prefix.view(np.int64))
    assert int(np.sum(big.perm != np.arange(m))) > m // 2  # the pivoting is exercised
