"""TEST INFRASTRUCTURE: a NumPy stand-in for CudaTileOps, so the multi-rank host logic of
paper_2503_04424_b200.distributed runs under gloo on CPU (the container has no GPU).  Tiles are
plain 128x128 row-major blocks here; only the tile-op semantics must match the device ones."""

import contextlib

import numpy as np
import torch
from scipy.linalg import cholesky

from paper_2503_04424_b200.distributed import INT64_MAX, RowCyclic

T = 128


class NumpyTileOps:
    def __init__(self, dist: RowCyclic, m: int, panel_tiles: int = 8):
        self.dist, self.m, self.W = dist, m, panel_tiles
        nt, ml, W = dist.nt, dist.maxloc, self.W
        self.grid = torch.zeros((ml, nt, T, T), dtype=torch.float64)
        self.diag_block = torch.zeros((W, W, T, T), dtype=torch.float64)
        self.inv = torch.zeros((W, T, T), dtype=torch.float64)
        self.panel_loc = torch.zeros((ml, W, T, T), dtype=torch.float64)
        self.panels = [torch.zeros((dist.world * ml, W, T, T), dtype=torch.float64) for _ in range(2)]
        self.ell = torch.zeros(nt * T, dtype=torch.float64)
        self.fail = INT64_MAX
        self.peers = None  # peer mode: every rank's NumpyTileOps (ranks as threads of one process)

    def set_peers(self, ops_by_rank):
        self.peers = list(ops_by_rank)

    def load(self, a: np.ndarray):
        m, nt = self.m, self.dist.nt
        full = np.eye(nt * T)
        full[:m, :m] = a
        for i in self.dist.rows:
            for j in range(i + 1):
                self.grid[self.dist.local(i), j] = torch.from_numpy(full[i * T:(i + 1) * T, j * T:(j + 1) * T])

    def begin(self):
        self.ell.zero_()
        self.fail = INT64_MAX

    def wait_rest(self, s):
        pass

    def fill_diag_block(self, k0, ke):
        self.diag_block.zero_()
        for i in range(k0, ke):
            if self.dist.owner(i) == self.dist.rank:
                for j in range(k0, i + 1):
                    self.diag_block[i - k0, j - k0] = self.grid[self.dist.local(i), j]

    def factor_diag_block(self, k0, ke):
        n = ke - k0
        blk = np.zeros((n * T, n * T))
        for i in range(n):
            for j in range(i + 1):
                blk[i * T:(i + 1) * T, j * T:(j + 1) * T] = self.diag_block[i, j].numpy()
        try:
            low = cholesky(np.tril(blk) + np.tril(blk, -1).T, lower=True)
        except np.linalg.LinAlgError:
            self.fail = min(self.fail, k0 * T)
            low = np.eye(n * T)
        for i in range(n):
            for j in range(i + 1):
                self.diag_block[i, j] = torch.from_numpy(low[i * T:(i + 1) * T, j * T:(j + 1) * T].copy())
        self.low = low
        self.ell[k0 * T:ke * T] = torch.from_numpy(2.0 * np.log(np.diagonal(low)))

    def solve_panel(self, k0, ke):
        n = ke - k0
        linv_t = np.linalg.inv(self.low).T
        for i in self.dist.rows:
            if i >= ke:
                li = self.dist.local(i)
                row = np.concatenate([self.grid[li, k0 + q].numpy() for q in range(n)], axis=1)
                x = row @ linv_t
                for q in range(n):
                    self.grid[li, k0 + q] = torch.from_numpy(x[:, q * T:(q + 1) * T].copy())

    def local_panel(self, k0, ke):
        self.panel_loc.zero_()
        self.panel_loc[:, : ke - k0] = self.grid[:, k0:ke]
        return self.panel_loc

    def panel_buffer(self, s):
        return self.panels[s % 2]

    def update_trailing(self, s, k0, ke, j0, j1):
        P, ml = self.dist.world, self.dist.maxloc
        g = self.panels[s % 2]
        for i in self.dist.rows:
            li = self.dist.local(i)
            for j in range(j0, min(j1, i + 1)):
                if self.peers:  # the owner's grid, read in place
                    row = self.peers[j % P].grid[j // P]
                    for p in range(k0, ke):
                        self.grid[li, j] -= self.grid[li, p] @ row[p].T
                else:
                    gj = g[(j % P) * ml + j // P]
                    for p in range(k0, ke):
                        self.grid[li, j] -= self.grid[li, p] @ gj[p - k0].T

    def mark_panel(self, s):
        pass

    def side(self):
        return contextlib.nullcontext()

    def wait_panel(self, s):
        pass

    def mark_rest(self, s):
        pass

    def join(self):
        pass

    def fail_tensor(self):
        return torch.tensor([self.fail], dtype=torch.int64)

    def fail_value(self, fail):
        v = int(fail.item())
        return -1 if v == INT64_MAX else v

    def prefix(self):
        return torch.cumsum(self.ell[: self.m], 0)


class ThreadComm:
    """TEST INFRASTRUCTURE: the collectives of paper_2503_04424_b200.distributed.TorchComm for
    ranks run as threads of one process (CPU tensors, or CUDA tensors on one GPU with one stream
    per thread).  Host barriers only: no kernel ever waits on another rank's kernel."""

    class Group:
        def __init__(self, world):
            import threading

            self.world = world
            self.bar = threading.Barrier(world)
            self.slots = [None] * world
            self.result = None

    ReduceOp = torch.distributed.ReduceOp

    def __init__(self, group, rank):
        self.g, self.rank = group, rank

    @staticmethod
    def _sync(t):
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()

    def _exchange(self, t, combine):
        g = self.g
        self._sync(t)
        g.slots[self.rank] = t
        g.bar.wait()
        if self.rank == 0:
            g.result = combine(g.slots)
            self._sync(g.result)
        g.bar.wait()
        return g.result

    def all_reduce(self, t, op=None):
        if op is None or op == self.ReduceOp.SUM:
            r = self._exchange(t, lambda xs: torch.stack([x.to(xs[0].device) for x in xs]).sum(0))
        elif op == self.ReduceOp.MIN:
            r = self._exchange(t, lambda xs: torch.stack([x.to(xs[0].device) for x in xs]).min(0).values)
        else:
            raise ValueError(op)
        t.copy_(r)
        self._sync(t)
        self.g.bar.wait()

    def broadcast(self, t, src):
        r = self._exchange(t, lambda xs: xs[src].clone())
        t.copy_(r)
        self._sync(t)
        self.g.bar.wait()

    def all_gather_into_tensor(self, out, inp):
        r = self._exchange(inp, lambda xs: torch.cat([x.reshape(-1) for x in xs]))
        out.copy_(r.reshape(out.shape))
        self._sync(out)
        self.g.bar.wait()

    def barrier(self):
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        self.g.bar.wait()


def run_threads(world, fn):
    """Run fn(rank) for every rank in its own thread; returns the results by rank (re-raises)."""
    import threading

    out, err = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 - surfaced below
            err.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    if err:
        raise err[0]
    return out
