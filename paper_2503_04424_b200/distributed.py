"""Multi-GPU MEMDET: one process per GPU, tile rows distributed row-cyclically, panels exchanged
with NCCL collectives over NVLink.

Layout.  The n_pad x n_pad lower tile triangle (128-wide tiles) is split by tile
row: rank r owns tile rows i = r, r + P, r + 2P, ...  (row i holds i + 1 tiles, so the cyclic
deal balances the triangle).  Each rank stores its rows as a local grid [maxloc][nt] of tiles.

Step (outer panel of W tile-columns [k0, ke)), for p in the panel:
  1. the owner of tile row p factors the diagonal tile (potrf + inverse, fused 2 log L_pp);
  2. broadcast of L_pp^{-1} (128 KB) from the owner;
  3. every rank solves its tiles (i, p), i > p (DMMA TRSM against the inverse);
  4. the solved tiles L(j, p), j in (p, ke), meet in a W-tile buffer (all-reduce of disjoint
     contributions: exact) and every rank updates its tiles in the panel columns (p, ke).
After the panel: all-gather of the panel (each rank's rows x W tiles) and the trailing Schur
update of every rank's own tiles with K = 128*W (DMMA).  The 2 log L_ii values meet in one
all-reduce at the end and every rank scans the prefix.

The driver is written against a small tile-ops interface so the same host logic runs on the
GPUs (`CudaTileOps`, the C ABI's tile-level entry points on device buffers, NCCL) and in the
multi-process CPU tests (a NumPy stand-in under tests/, gloo).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native

T = 128
TILE_ELEMS = T * T
TILE_BYTES = TILE_ELEMS * 8
INT64_MAX = 2 ** 63 - 1


@dataclass(frozen=True)
class RowCyclic:
    """Tile row i lives on rank i % world, at local row i // world."""

    nt: int
    world: int
    rank: int

    @property
    def rows(self) -> range:
        return range(self.rank, self.nt, self.world)

    @property
    def nloc(self) -> int:
        return len(self.rows)

    @property
    def maxloc(self) -> int:
        return -(-self.nt // self.world)

    def owner(self, i: int) -> int:
        return i % self.world

    def local(self, i: int) -> int:
        return i // self.world


def factor_distributed(ops, comm, dist: RowCyclic, panel_tiles: int = 8):
    """Factor the distributed lower tile triangle held by `ops`; returns (prefix, fail) on
    every rank (fail = first non-positive pivot's global row, or -1)."""
    nt, P, W = dist.nt, dist.world, panel_tiles
    ops.begin()
    for k0 in range(0, nt, W):
        ke = min(k0 + W, nt)
        for p in range(k0, ke):
            owner = dist.owner(p)
            if dist.rank == owner:
                ops.potrf(dist.local(p), p)
            comm.broadcast(ops.inv, src=owner)
            ops.trsm(p)
            if p + 1 < ke:
                ops.fill_diag_buffer(p, k0, ke)
                comm.all_reduce(ops.diag_buffer)
                ops.update_intra(p, k0, ke)
        if ke >= nt:
            break
        comm.all_gather_into_tensor(ops.panel_all, ops.local_panel(k0, ke))
        ops.update_trailing(k0, ke)
    comm.all_reduce(ops.ell)
    fail = ops.fail_tensor()
    comm.all_reduce(fail, op=comm.ReduceOp.MIN)
    return ops.prefix(), ops.fail_value(fail)


class CudaTileOps:
    """Per-rank device state and the C-ABI tile kernels (all enqueued on torch's current
    stream).  Local grid [maxloc][nt] tiles; gathered panel [P][maxloc][W] tiles."""

    def __init__(self, dist: RowCyclic, m: int, panel_tiles: int = 8, device=None):
        import torch

        self.torch = torch
        self.dist = dist
        self.m = m
        self.W = panel_tiles
        self.dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        f64 = dict(dtype=torch.float64, device=self.dev)
        nt, ml = dist.nt, dist.maxloc
        self.grid = torch.empty(ml * nt * TILE_ELEMS, **f64)
        self.inv = torch.empty(TILE_ELEMS, **f64)
        self.diag_buffer = torch.empty(self.W * TILE_ELEMS, **f64)
        self.panel_loc = torch.empty(ml * self.W * TILE_ELEMS, **f64)
        self.panel_all = torch.empty(dist.world * ml * self.W * TILE_ELEMS, **f64)
        npad = nt * T
        self.ell = torch.zeros(npad, **f64)
        self.diag = torch.zeros(npad, **f64)
        self.prefix_buf = torch.empty(npad, **f64)
        self.fail = torch.empty(1, dtype=torch.int64, device=self.dev)
        self.lib = _native.load()
        self.launches = 0  # engine kernels enqueued (potrf / gemm / pack / prefix calls)

    # -------------------------------------------------------------------- helpers
    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.dev).cuda_stream)

    def _grid_map(self):
        return _native.TileMapC(self.grid.data_ptr(), self.dist.nt, 0, 0, 0)

    def _set(self, j0, j1, row_off=0):
        d = self.dist
        return _native.TileSetC(0, d.nloc, j0, j1, 1, row_off, d.world, d.rank)

    def _tile_ptr(self, li, j):
        return self.grid.data_ptr() + (li * self.dist.nt + j) * TILE_BYTES

    # -------------------------------------------------------------------- interface
    def load(self, a, lda: int | None = None):
        """Pack this rank's tiles from a row-major CUDA matrix (every rank holds or maps it)."""
        torch = self.torch
        dcode = _native.B2D_F64 if a.dtype == torch.float64 else _native.B2D_F32
        lda = lda or a.stride(0)
        _native.check(self.lib.b2d_pack_tiles(ctypes.c_void_p(a.data_ptr()), lda, dcode, 0, self.m,
                                              ctypes.byref(self._grid_map()),
                                              ctypes.byref(self._set(0, self.dist.nt)), self._stream()),
                      "b2d_pack_tiles")
        self.launches += 1

    def begin(self):
        self.ell.zero_()
        self.diag.zero_()
        self.fail.fill_(-1)  # all ones = UINT64_MAX for the kernel's atomicMin

    def potrf(self, li: int, p: int):
        _native.check(self.lib.b2d_tile_potrf_inv(
            ctypes.c_void_p(self._tile_ptr(li, p)), ctypes.c_void_p(self.inv.data_ptr()),
            ctypes.c_void_p(self.ell.data_ptr()), ctypes.c_void_p(self.diag.data_ptr()),
            ctypes.c_void_p(self.fail.data_ptr()), p * T, self.m, self._stream()), "potrf")
        self.launches += 1

    def trsm(self, p: int):
        s = self._set(p, p + 1, row_off=1)
        _native.check(self.lib.b2d_tile_gemm(1, None, None, ctypes.byref(self._grid_map()),
                                             ctypes.c_void_p(self.inv.data_ptr()), ctypes.byref(s),
                                             0, 0, p, self._stream()), "trsm")
        self.launches += 1

    def fill_diag_buffer(self, p: int, k0: int, ke: int):
        self.diag_buffer.zero_()
        buf = self.diag_buffer.view(self.W, TILE_ELEMS)
        grid = self.grid.view(self.dist.maxloc, self.dist.nt, TILE_ELEMS)
        for j in range(p + 1, ke):
            if self.dist.owner(j) == self.dist.rank:
                buf[j - k0].copy_(grid[self.dist.local(j), p])

    def _gemm_update(self, bmap, j0, j1, p0, p1):
        s = self._set(j0, j1)
        g = self._grid_map()
        _native.check(self.lib.b2d_tile_gemm(0, ctypes.byref(g), ctypes.byref(bmap), ctypes.byref(g), None,
                                             ctypes.byref(s), p0, p1, 0, self._stream()), "update")
        self.launches += 1

    def update_intra(self, p: int, k0: int, ke: int):
        # B(j, p) = diag_buffer[j - k0]: base shifted so tile(j, p) = base + (j + p) tiles
        base = self.diag_buffer.data_ptr() - (k0 + p) * TILE_BYTES
        self._gemm_update(_native.TileMapC(base, 1, 0, 0, 0), p + 1, ke, p, p + 1)

    def local_panel(self, k0: int, ke: int):
        grid = self.grid.view(self.dist.maxloc, self.dist.nt, TILE_ELEMS)
        loc = self.panel_loc.view(self.dist.maxloc, self.W, TILE_ELEMS)
        loc[:, : ke - k0].copy_(grid[:, k0:ke])
        return self.panel_loc

    def update_trailing(self, k0: int, ke: int):
        # gathered panel [P][maxloc][W]: tile (j, p) at ((j % P) * maxloc + j // P) * W + p - k0
        base = self.panel_all.data_ptr() - k0 * TILE_BYTES
        bmap = _native.TileMapC(base, self.W, 0, self.dist.world, self.dist.maxloc)
        self._gemm_update(bmap, ke, self.dist.nt, k0, ke)

    def fail_tensor(self):
        # the kernel's "no failure" is UINT64_MAX (int64 -1); make it the largest int64 for MIN
        f = self.fail.clone()
        f[f == -1] = INT64_MAX
        return f

    def fail_value(self, fail) -> int:
        v = int(fail.item())
        return -1 if v == INT64_MAX else v

    def prefix(self):
        _native.check(self.lib.b2d_prefix_scan(ctypes.c_void_p(self.ell.data_ptr()), self.m,
                                               ctypes.c_void_p(self.prefix_buf.data_ptr()), self._stream()),
                      "prefix")
        self.launches += 1
        return self.prefix_buf[: self.m]


class TorchComm:
    """torch.distributed collectives.  With NCCL the CUDA buffers go over NVLink directly; with
    gloo (tests, or hosts without NCCL) device buffers are staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist_mod

        self.d = dist_mod
        self.group = group
        self.ReduceOp = dist_mod.ReduceOp
        self.staged = dist_mod.get_backend(group) == "gloo"

    def _run(self, fn, *tensors):
        if not self.staged or not any(t.is_cuda for t in tensors):
            fn(*tensors)
            return
        host = [t.cpu() for t in tensors]
        fn(*host)
        for t, h in zip(tensors, host):
            t.copy_(h)

    def broadcast(self, t, src):
        self._run(lambda x: self.d.broadcast(x, src=src, group=self.group), t)

    def all_reduce(self, t, op=None):
        op = self.ReduceOp.SUM if op is None else op
        self._run(lambda x: self.d.all_reduce(x, op=op, group=self.group), t)

    def all_gather_into_tensor(self, out, inp):
        def gather(o, i):
            chunks = list(o.chunk(self.d.get_world_size(self.group)))
            self.d.all_gather(chunks, i, group=self.group)
        self._run(gather, out, inp)


class DistributedMemdet:
    """Reusable per-rank workspace for repeated distributed factorisations of order m."""

    def __init__(self, m: int, group=None, panel_tiles: int = 8, device=None):
        import torch.distributed as dist_mod

        self.group = group
        self.m = m
        self.panel_tiles = panel_tiles
        self.dist = RowCyclic(-(-m // T), dist_mod.get_world_size(group), dist_mod.get_rank(group))
        self.ops = CudaTileOps(self.dist, m, panel_tiles, device)
        self.comm = TorchComm(group)

    def run(self, a):
        """Enqueue pack + factorisation of the CUDA row-major matrix `a` (every rank passes the
        matrix; each packs its own tile rows).  Returns (device prefix view, fail)."""
        self.ops.load(a)
        return factor_distributed(self.ops, self.comm, self.dist, self.panel_tiles)


def memdet_cholesky_distributed(a, group=None, panel_tiles: int = 8):
    """Distributed logdet of a CUDA row-major SPD matrix visible to every rank (each rank packs
    only its own tile rows).  Returns (prefix as a NumPy array, fail index) on every rank."""
    import torch

    runner = DistributedMemdet(int(a.shape[0]), group, panel_tiles, a.device)
    prefix, fail = runner.run(a)
    torch.cuda.synchronize(a.device)
    return prefix.cpu().numpy(), fail
