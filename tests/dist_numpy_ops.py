"""TEST INFRASTRUCTURE: a NumPy stand-in for CudaTileOps, so the multi-rank host logic of
paper_2503_04424_b200.distributed runs under gloo on CPU (the container has no GPU).  Tiles are
plain 128x128 row-major blocks here; only the tile-op semantics must match the device ones."""

import numpy as np
import torch
from scipy.linalg import cholesky

from paper_2503_04424_b200.distributed import INT64_MAX, RowCyclic

T = 128


class NumpyTileOps:
    def __init__(self, dist: RowCyclic, m: int, panel_tiles: int = 8):
        self.dist, self.m, self.W = dist, m, panel_tiles
        nt, ml = dist.nt, dist.maxloc
        self.grid = torch.zeros((ml, nt, T, T), dtype=torch.float64)
        self.inv = torch.zeros((T, T), dtype=torch.float64)
        self.diag_buffer = torch.zeros((self.W, T, T), dtype=torch.float64)
        self.panel_loc = torch.zeros((ml, self.W, T, T), dtype=torch.float64)
        self.panel_all = torch.zeros((dist.world * ml, self.W, T, T), dtype=torch.float64)
        self.ell = torch.zeros(nt * T, dtype=torch.float64)
        self.fail = INT64_MAX

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

    def potrf(self, li, p):
        t = self.grid[li, p].numpy()
        try:
            low = cholesky(np.tril(t) + np.tril(t, -1).T, lower=True)
        except np.linalg.LinAlgError:
            self.fail = min(self.fail, p * T)
            low = np.eye(T)
        self.grid[li, p] = torch.from_numpy(low)
        self.inv.copy_(torch.from_numpy(np.linalg.inv(low)))
        self.ell[p * T:(p + 1) * T] = torch.from_numpy(2.0 * np.log(np.diagonal(low)))

    def trsm(self, p):
        for i in self.dist.rows:
            if i > p:
                li = self.dist.local(i)
                self.grid[li, p] = self.grid[li, p] @ self.inv.T

    def fill_diag_buffer(self, p, k0, ke):
        self.diag_buffer.zero_()
        for j in range(p + 1, ke):
            if self.dist.owner(j) == self.dist.rank:
                self.diag_buffer[j - k0] = self.grid[self.dist.local(j), p]

    def update_intra(self, p, k0, ke):
        for i in self.dist.rows:
            li = self.dist.local(i)
            for j in range(p + 1, min(ke, i + 1)):
                self.grid[li, j] -= self.grid[li, p] @ self.diag_buffer[j - k0].T

    def local_panel(self, k0, ke):
        self.panel_loc.zero_()
        self.panel_loc[:, : ke - k0] = self.grid[:, k0:ke]
        return self.panel_loc

    def update_trailing(self, k0, ke):
        P, ml = self.dist.world, self.dist.maxloc
        for i in self.dist.rows:
            li = self.dist.local(i)
            for j in range(ke, i + 1):
                g = self.panel_all[(j % P) * ml + j // P]
                for p in range(k0, ke):
                    self.grid[li, j] -= self.grid[li, p] @ g[p - k0].T

    def fail_tensor(self):
        return torch.tensor([self.fail], dtype=torch.int64)

    def fail_value(self, fail):
        v = int(fail.item())
        return -1 if v == INT64_MAX else v

    def prefix(self):
        return torch.cumsum(self.ell[: self.m], 0)
