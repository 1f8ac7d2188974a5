"""Multi-rank host logic of the row-cyclic distributed factorisation (distributed.py) under
gloo on CPU, world sizes 2 and 3, against the CPU oracle.  The tile math is a NumPy stand-in
(tests/dist_numpy_ops.py); the GPU version of the same driver is in test_gpu_parity.py."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import rel_err


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, panel, seed, out_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_numpy_ops import NumpyTileOps

    from paper_2503_04424_b200 import gen
    from paper_2503_04424_b200.distributed import RowCyclic, TorchComm, factor_distributed

    a = gen.spd_wishart(m, m, seed=seed, shift=1e-2)
    nt = -(-m // 128)
    d = RowCyclic(nt, world, rank)
    ops = NumpyTileOps(d, m, panel)
    ops.load(a)
    prefix, fail = factor_distributed(ops, TorchComm(), d, panel)
    out_q.put((rank, prefix.numpy().copy(), fail))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,panel", [(2, 700, 2), (3, 1000, 3), (2, 384, 8)])
def test_row_cyclic_driver_matches_oracle(world, m, panel):
    from oracle import memdet_oracle as O
    from paper_2503_04424_b200 import gen

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, panel, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = gen.spd_wishart(m, m, seed=7, shift=1e-2)
    ref, _ = O.memdet_cholesky(a, 1)
    for rank, prefix, fail in results:
        assert fail == -1
        assert rel_err(prefix, ref) <= 1e-10, (rank, rel_err(prefix, ref))


def test_row_cyclic_layout():
    from paper_2503_04424_b200.distributed import RowCyclic

    d = RowCyclic(10, 3, 1)
    assert list(d.rows) == [1, 4, 7] and d.nloc == 3 and d.maxloc == 4
    assert all(RowCyclic(10, 3, r).owner(i) == i % 3 for r in range(3) for i in range(10))
    # every tile row has exactly one owner and the lower triangle is balanced within one row
    loads = [sum(i + 1 for i in RowCyclic(64, 4, r).rows) for r in range(4)]
    assert max(loads) - min(loads) <= 64


@pytest.mark.parametrize("world,m,panel", [(2, 700, 2), (3, 1000, 3), (4, 900, 2)])
def test_peer_mode_driver_matches_oracle(world, m, panel):
    """Peer mode (the NVLink product path: solved panels read in place from their owners' grids
    after a barrier, no all-gather): ranks as threads sharing memory, NumPy tile math."""
    from dist_numpy_ops import NumpyTileOps, ThreadComm, run_threads
    from oracle import memdet_oracle as O

    from paper_2503_04424_b200 import gen
    from paper_2503_04424_b200.distributed import RowCyclic, factor_distributed

    a = gen.spd_wishart(m, m, seed=9, shift=1e-2)
    nt = -(-m // 128)
    group = ThreadComm.Group(world)
    ops = [NumpyTileOps(RowCyclic(nt, world, r), m, panel) for r in range(world)]
    for o in ops:
        o.load(a)
        o.set_peers(ops)

    def rank(r):
        return factor_distributed(ops[r], ThreadComm(group, r), ops[r].dist, panel)

    res = run_threads(world, rank)
    ref, _ = O.memdet_cholesky(a, 1)
    for r, (prefix, fail) in enumerate(res):
        assert fail == -1
        assert rel_err(prefix.numpy(), ref) <= 1e-10, (r, rel_err(prefix.numpy(), ref))
        assert all(o.panels[0].abs().sum() == 0 for o in ops)  # no panel was ever gathered
