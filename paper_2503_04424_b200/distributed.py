"""Multi-GPU MEMDET: one process per GPU, tile rows distributed row-cyclically, panels exchanged
with NCCL collectives over NVLink.

Layout.  The n_pad x n_pad lower tile triangle (128-wide tiles) is split by tile
row: rank r owns tile rows i = r, r + P, r + 2P, ...  (row i holds i + 1 tiles, so the cyclic
deal balances the triangle).  Each rank stores its rows as a local grid [maxloc][nt] of tiles.

Step s (outer panel of W tile-columns [k0, ke)), two collectives per panel:
  1. the W x W diagonal block meets on every rank (all-reduce of disjoint row contributions,
     exact) and every rank factors it redundantly (potrf + inverse per tile, intra-block
     solves and updates) -> identical L_blk, L_pp^{-1} and 2 log L_ii everywhere;
  2. every rank solves its own panel rows i >= ke against L_blk (DMMA TRSM + updates);
  3. the solved panel is exchanged.  Peer mode (default with NCCL): a stream-ordered barrier
     (an all-reduce of one word), after which the Schur-update kernels of every rank read the
     owners' panel tiles in place from their tile grids over NVLink peer memory (the grids are
     cudaMalloc'd and mapped into every rank with CUDA IPC; the kernel's producer warp bulk-
     copies remote tiles straight into shared memory), so the exchange overlaps the DMMA work
     tile by tile and no panel copy exists.  Gather mode: all-gather of the solved panel
     (each rank's rows x W tiles, double-buffered) into a local buffer;
  4. next-cols: every rank updates its tiles in the next panel's columns [ke, ke+W) (main
     stream, the critical path), then the rest [ke+W, nt) on a side stream that overlaps the
     next panel's steps 1-3 (one-panel look-ahead, as the single-GPU driver).
A solved panel column is final on its owner (later steps touch only columns to its right), so
peers may read it any time after the barrier.  Every rank holds every 2 log L_ii at the end
and scans the prefix itself.

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
    nt, W = dist.nt, panel_tiles
    ops.begin()
    steps = [(k0, min(k0 + W, nt)) for k0 in range(0, nt, W)]
    for s, (k0, ke) in enumerate(steps):
        ne = min(ke + W, nt)
        ops.wait_rest(s - 2)                    # columns [k0, ke) carry every earlier panel
        ops.fill_diag_block(k0, ke)
        comm.all_reduce(ops.diag_block)
        ops.factor_diag_block(k0, ke)
        if ke >= nt:
            break
        ops.solve_panel(k0, ke)
        if getattr(ops, "peers", None):
            comm.barrier()  # every rank's panel rows are solved: read in place from here on
        else:
            comm.all_gather_into_tensor(ops.panel_buffer(s), ops.local_panel(k0, ke))
        ops.update_trailing(s, k0, ke, ke, ne)                 # next panel's columns (main)
        ops.mark_panel(s)
        with ops.side():
            ops.wait_panel(s)
            ops.update_trailing(s, k0, ke, ne, nt)             # the rest (side stream)
            ops.mark_rest(s)
    ops.join()
    fail = ops.fail_tensor()
    comm.all_reduce(fail, op=comm.ReduceOp.MIN)
    return ops.prefix(), ops.fail_value(fail)


class CudaTileOps:
    """Per-rank device state and the C-ABI tile kernels (enqueued on torch's current stream;
    the rest updates on a side stream).  Local grid [maxloc][nt] tiles; W x W diagonal block;
    gathered panels [P][maxloc][W] tiles, double-buffered."""

    def __init__(self, dist: RowCyclic, m: int, panel_tiles: int = 8, device=None, grid=None):
        import torch

        self.torch = torch
        self.dist = dist
        self.m = m
        self.W = panel_tiles
        self.dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        f64 = dict(dtype=torch.float64, device=self.dev)
        nt, ml, W = dist.nt, dist.maxloc, self.W
        # the local tile grid (a peer-shareable buffer in peer mode, see DistributedMemdet)
        self.grid = grid if grid is not None else torch.empty(ml * nt * TILE_ELEMS, **f64)
        self.peers = None  # peer mode: every rank's grid address in this process, by rank
        self.diag_block = torch.empty(W * W * TILE_ELEMS, **f64)
        self.inv = torch.empty(W * TILE_ELEMS, **f64)
        self._panel_loc = None  # gather mode only (allocated on first use)
        self._panels = None
        npad = nt * T
        self.ell = torch.zeros(npad, **f64)
        self.diag = torch.zeros(npad, **f64)
        self.prefix_buf = torch.empty(npad, **f64)
        self.fail = torch.empty(1, dtype=torch.int64, device=self.dev)
        self.lib = _native.load()
        self.side_stream = torch.cuda.Stream(self.dev)
        nsteps = -(-nt // W)
        self.ev_panel = [torch.cuda.Event() for _ in range(nsteps)]
        self.ev_rest = [torch.cuda.Event() for _ in range(nsteps)]
        self.launches = 0  # engine kernels enqueued

    # -------------------------------------------------------------------- helpers
    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.dev).cuda_stream)

    def _grid_map(self):
        return _native.TileMapC(self.grid.data_ptr(), self.dist.nt, 0, 0, 0)

    def _blk_map(self, k0):
        # diag block tile (i, j), global indices in [k0, ke): base shifted so tile(i, j) lands at
        # ((i - k0) * W + (j - k0))
        base = self.diag_block.data_ptr() - (k0 * self.W + k0) * TILE_BYTES
        return _native.TileMapC(base, self.W, 0, 0, 0)

    def _rows_from(self, g):
        """First local row whose global row is >= g."""
        d = self.dist
        return max(0, -(-(g - d.rank) // d.world))

    def _gemm(self, mode, amap, bmap, cmap, binv, tset, p0, p1, k):
        _native.check(self.lib.b2d_tile_gemm(mode, None if amap is None else ctypes.byref(amap),
                                             None if bmap is None else ctypes.byref(bmap), ctypes.byref(cmap),
                                             None if binv is None else ctypes.c_void_p(binv), ctypes.byref(tset),
                                             p0, p1, k, self._stream()), "b2d_tile_gemm")
        self.launches += 1

    # -------------------------------------------------------------------- interface
    def load(self, a, lda: int | None = None):
        """Pack this rank's tiles from a row-major CUDA matrix (every rank holds or maps it)."""
        torch = self.torch
        dcode = _native.B2D_F64 if a.dtype == torch.float64 else _native.B2D_F32
        lda = lda or a.stride(0)
        d = self.dist
        s = _native.TileSetC(0, d.nloc, 0, d.nt, 1, 0, d.world, d.rank)
        _native.check(self.lib.b2d_pack_tiles(ctypes.c_void_p(a.data_ptr()), lda, dcode, 0, self.m,
                                              ctypes.byref(self._grid_map()), ctypes.byref(s), self._stream()),
                      "b2d_pack_tiles")
        self.launches += 1

    def load_host(self, a, lda: int | None = None):
        """Sharded ingest from a HOST row-major matrix (NumPy; pinned or pageable): this rank copies
        only its own tile rows -- tile row i is the file's column strip [128 i, 128 i + 128) over
        rows [0, 128 (i + 1)) (the upper triangle the reference reads) -- and packs them; no rank
        holds the matrix.  Returns the bytes copied."""
        import numpy as np

        torch = self.torch
        a = np.asarray(a)
        dcode = _native.B2D_F64 if a.dtype == np.float64 else _native.B2D_F32
        esz = a.itemsize
        lda = lda or a.strides[0] // esz
        d, m, nt = self.dist, self.m, self.dist.nt
        buf = torch.empty(nt * T * T * esz, dtype=torch.uint8, device=self.dev)
        moved = 0
        for li, i in enumerate(d.rows):
            c0 = i * T
            width, rows = max(0, min(T, m - c0)), min(m, (i + 1) * T)
            if width > 0:
                _native.check(self.lib.b2d_h2d_2d(ctypes.c_void_p(buf.data_ptr()), T * esz,
                                                  ctypes.c_void_p(a.ctypes.data + c0 * esz), lda * esz, width * esz,
                                                  rows, self._stream()), "b2d_h2d_2d")
                moved += width * rows * esz
            # element (R, C) of tile (i, J) is file[C][R]: the strip holds column R - 128 i of row C
            src = buf.data_ptr() - c0 * esz
            s = _native.TileSetC(li, li + 1, 0, i + 1, 0, 0, d.world, d.rank)
            _native.check(self.lib.b2d_pack_tiles(ctypes.c_void_p(src), T, dcode, 0, m,
                                                  ctypes.byref(self._grid_map()), ctypes.byref(s), self._stream()),
                          "b2d_pack_tiles")
            self.launches += 1
        self._keep = buf  # released with the next load (stream-ordered reuse)
        return moved

    def begin(self):
        self.ell.zero_()
        self.diag.zero_()
        self.fail.fill_(-1)  # all ones = UINT64_MAX for the kernel's atomicMin
        self.side_stream.wait_stream(self.torch.cuda.current_stream(self.dev))

    def wait_rest(self, s):
        if s >= 0:
            self.torch.cuda.current_stream(self.dev).wait_event(self.ev_rest[s])

    def fill_diag_block(self, k0, ke):
        self.diag_block.zero_()
        blk = self.diag_block.view(self.W, self.W, TILE_ELEMS)
        grid = self.grid.view(self.dist.maxloc, self.dist.nt, TILE_ELEMS)
        for i in range(k0, ke):
            if self.dist.owner(i) == self.dist.rank:
                blk[i - k0, : i - k0 + 1].copy_(grid[self.dist.local(i), k0:i + 1])

    def factor_diag_block(self, k0, ke):
        """Redundant on every rank: right-looking Cholesky of the W x W diagonal block."""
        bm = self._blk_map(k0)
        for p in range(k0, ke):
            invp = self.inv.data_ptr() + (p - k0) * TILE_BYTES
            _native.check(self.lib.b2d_tile_potrf_inv(
                ctypes.c_void_p(bm.base + ((p * self.W) + p) * TILE_BYTES), ctypes.c_void_p(invp),
                ctypes.c_void_p(self.ell.data_ptr()), ctypes.c_void_p(self.diag.data_ptr()),
                ctypes.c_void_p(self.fail.data_ptr()), p * T, self.m, self._stream()), "potrf")
            self.launches += 1
            if p + 1 < ke:
                self._gemm(1, None, None, bm, invp, _native.TileSetC(p + 1, ke, p, p + 1, 0, 0, 0, 0), 0, 0, p)
                self._gemm(0, bm, bm, bm, None, _native.TileSetC(p + 1, ke, p + 1, ke, 1, 0, 0, 0), p, p + 1, 0)

    def solve_panel(self, k0, ke):
        """Own rows i >= ke: X(i, [k0, ke)) = A L_blk^{-T}, right-looking over the block."""
        d = self.dist
        i0 = self._rows_from(ke)
        g, bm = self._grid_map(), self._blk_map(k0)
        for p in range(k0, ke):
            invp = self.inv.data_ptr() + (p - k0) * TILE_BYTES
            self._gemm(1, None, None, g, invp, _native.TileSetC(i0, d.nloc, p, p + 1, 0, 0, 0, 0), 0, 0, p)
            if p + 1 < ke:
                self._gemm(0, g, bm, g, None, _native.TileSetC(i0, d.nloc, p + 1, ke, 0, 0, 0, 0), p, p + 1, 0)

    def _gather_buffers(self):
        if self._panels is None:
            f64 = dict(dtype=self.torch.float64, device=self.dev)
            ml, W = self.dist.maxloc, self.W
            self._panel_loc = self.torch.empty(ml * W * TILE_ELEMS, **f64)
            self._panels = [self.torch.empty(self.dist.world * ml * W * TILE_ELEMS, **f64) for _ in range(2)]
        return self._panel_loc, self._panels

    def local_panel(self, k0: int, ke: int):
        panel_loc, _ = self._gather_buffers()
        grid = self.grid.view(self.dist.maxloc, self.dist.nt, TILE_ELEMS)
        loc = panel_loc.view(self.dist.maxloc, self.W, TILE_ELEMS)
        loc[:, : ke - k0].copy_(grid[:, k0:ke])
        return panel_loc

    def panel_buffer(self, s):
        return self._gather_buffers()[1][s % 2]

    def set_peers(self, ptrs):
        """Peer mode: `ptrs[r]` = rank r's tile grid as addressable from this process."""
        if len(ptrs) != self.dist.world or len(ptrs) > _native.MAX_PEERS:
            raise ValueError(f"need {self.dist.world} peer grids (at most {_native.MAX_PEERS})")
        self.peers = [int(p) for p in ptrs]

    def update_trailing(self, s, k0, ke, j0, j1):
        """Own tiles in columns [j0, j1) -= L(i, panel) L(j, panel)^T.  The panel rows L(j, .)
        are read in place from their owners' grids (peer mode) or from the gathered panel
        [P][maxloc][W] (gather mode), both through a row-cyclic tile map."""
        if j1 <= j0:
            return
        d = self.dist
        if self.peers:
            bmap = _native.peer_map(self.peers, d.nt)
        else:
            base = self._gather_buffers()[1][s % 2].data_ptr() - k0 * TILE_BYTES
            bmap = _native.TileMapC(base, self.W, 0, d.world, d.maxloc)
        g = self._grid_map()
        self._gemm(0, g, bmap, g, None, _native.TileSetC(0, d.nloc, j0, j1, 1, 0, d.world, d.rank), k0, ke, 0)

    def mark_panel(self, s):
        self.ev_panel[s].record(self.torch.cuda.current_stream(self.dev))

    def side(self):
        return self.torch.cuda.stream(self.side_stream)

    def wait_panel(self, s):
        self.side_stream.wait_event(self.ev_panel[s])

    def mark_rest(self, s):
        self.ev_rest[s].record(self.side_stream)

    def join(self):
        self.torch.cuda.current_stream(self.dev).wait_stream(self.side_stream)

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

    def barrier(self):
        """Stream-ordered barrier: an all-reduce of one word on the current CUDA stream (NCCL),
        so work enqueued after it starts only once every rank's earlier work has finished."""
        import torch

        if self.staged:  # host barrier: finish this rank's enqueued work first
            if torch.cuda.is_available() and torch.cuda.is_initialized():
                torch.cuda.current_stream().synchronize()
            self.d.barrier(group=self.group)
            return
        if getattr(self, "_token", None) is None:
            self._token = torch.zeros(1, dtype=torch.int32, device=torch.device("cuda", torch.cuda.current_device()))
        self.d.all_reduce(self._token, group=self.group)


class _DeviceArray:
    """A raw device allocation seen by torch through __cuda_array_interface__ (zero copy)."""

    def __init__(self, ptr: int, nelem: int):
        self.__cuda_array_interface__ = {"shape": (nelem,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerGrids:
    """Tile grids shared across the ranks of one node: this rank's grid is a cudaMalloc'd
    buffer; the others' are mapped in through CUDA IPC handles exchanged with
    all_gather_object.  `ptrs[r]` is rank r's grid in this process."""

    def __init__(self, nelem: int, group=None, device=None):
        import torch
        import torch.distributed as dist_mod

        self.lib = _native.load()
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev.index if dev.index is not None else torch.cuda.current_device()
        p = ctypes.c_void_p()
        _native.check(self.lib.b2d_dev_alloc(self.device, nelem * 8, ctypes.byref(p)), "b2d_dev_alloc")
        self.own = p.value
        self.tensor = torch.as_tensor(_DeviceArray(self.own, nelem), device=dev)
        h = ctypes.create_string_buffer(64)
        _native.check(self.lib.b2d_ipc_get_handle(ctypes.c_void_p(self.own), h), "b2d_ipc_get_handle")
        world, rank = dist_mod.get_world_size(group), dist_mod.get_rank(group)
        handles = [None] * world
        dist_mod.all_gather_object(handles, h.raw, group=group)
        self.opened, self.ptrs = [], []
        for r, hr in enumerate(handles):
            if r == rank:
                self.ptrs.append(self.own)
                continue
            q = ctypes.c_void_p()
            _native.check(self.lib.b2d_ipc_open_handle(self.device, ctypes.create_string_buffer(hr, 64),
                                                       ctypes.byref(q)), "b2d_ipc_open_handle")
            self.opened.append(q.value)
            self.ptrs.append(q.value)

    def close(self):
        for q in self.opened:
            self.lib.b2d_ipc_close_handle(ctypes.c_void_p(q))
        self.opened = []
        if self.own:
            self.tensor = None
            self.lib.b2d_dev_free(ctypes.c_void_p(self.own))
            self.own = None


def _peers_reachable(group=None, device=None) -> bool:
    """Every rank's device can map every other rank's memory (P2P over NVLink / NVSwitch)."""
    import torch
    import torch.distributed as dist_mod

    dev = device.index if device is not None and device.index is not None else torch.cuda.current_device()
    devs = [None] * dist_mod.get_world_size(group)
    dist_mod.all_gather_object(devs, dev, group=group)
    ok = all(a == b or torch.cuda.can_device_access_peer(dev, b) for a in [dev] for b in devs)
    flags = [None] * len(devs)
    dist_mod.all_gather_object(flags, ok, group=group)
    return all(flags)


class DistributedMemdet:
    """Reusable per-rank workspace for repeated distributed factorisations of order m.
    `peer` (default: with NCCL) reads the solved panels in place over NVLink peer memory
    instead of all-gathering them."""

    def __init__(self, m: int, group=None, panel_tiles: int = 8, device=None, peer=None):
        import torch.distributed as dist_mod

        self.group = group
        self.m = m
        self.panel_tiles = panel_tiles
        self.dist = RowCyclic(-(-m // T), dist_mod.get_world_size(group), dist_mod.get_rank(group))
        self.comm = TorchComm(group)
        if peer is None:
            peer = not self.comm.staged and self.dist.world <= _native.MAX_PEERS and _peers_reachable(group, device)
        self.shared = None
        grid = None
        if peer:
            self.shared = PeerGrids(self.dist.maxloc * self.dist.nt * TILE_ELEMS, group, device)
            grid = self.shared.tensor
        self.ops = CudaTileOps(self.dist, m, panel_tiles, device, grid=grid)
        if peer:
            self.ops.set_peers(self.shared.ptrs)

    def close(self):
        """Unmap the peers' grids and free this rank's (after every rank is done with it)."""
        if self.shared is not None:
            import torch

            torch.cuda.synchronize()
            self.comm.barrier()
            torch.cuda.synchronize()
            self.shared.close()
            self.shared = None

    def run(self, a):
        """Enqueue pack + factorisation of the row-major matrix `a` -- a CUDA tensor every rank can
        address, or a HOST array (NumPy) from which each rank copies only its own tile rows.
        Returns (device prefix view, fail)."""
        if hasattr(a, "is_cuda") and a.is_cuda:
            self.ops.load(a)
        else:
            self.h2d_bytes = self.ops.load_host(a)
        return factor_distributed(self.ops, self.comm, self.dist, self.panel_tiles)


def memdet_cholesky_distributed(a, group=None, panel_tiles: int = 8, peer=None, device=None):
    """Distributed logdet of a row-major SPD matrix: a CUDA tensor visible to every rank, or a host
    array (each rank copies and packs only its own tile rows).  Returns (prefix as a NumPy array,
    fail index) on every rank."""
    import torch

    if hasattr(a, "is_cuda") and a.is_cuda:
        device = a.device
    elif device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    runner = DistributedMemdet(int(a.shape[0]), group, panel_tiles, device, peer=peer)
    prefix, fail = runner.run(a)
    torch.cuda.synchronize(device)
    out = prefix.cpu().numpy()
    runner.close()
    return out, fail
