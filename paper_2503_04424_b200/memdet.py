"""Drop-in MEMDET drivers on the B200 engine (reference oocdet/memdet.py).

Same entry points, keyword arguments, result types and errors as the reference:

    memdet_cholesky(matrix, *, max_mem=None, num_blocks=None, scratch_dir=None, prefix_out=None)
        -> SpdResult            (reference memdet.py:415-433)
    memdet_ldl(matrix, *, max_mem=None, num_blocks=None, scratch_dir=None, prefix_out=None)
        -> SymmetricResult      (reference memdet.py:392-412)

`matrix` may be a MatrixFile, a MEMDET01 path, a NumPy array / memmap, or a torch tensor
(CUDA tensors are factored in place of residence, no host round trip).  The factorisation
runs in libmemdet_b200.so (hand-written sm_100a kernels); `num_blocks` / `max_mem` keep the
reference's meaning for the reported tiling and counters (memdet.py:249-255), while the engine
tiles HBM with its own 128-wide tiles — the unpivoted factorisation, and therefore every prefix,
is independent of the tiling up to rounding (reference tests/test_memdet.py:216-237).
There is no CPU fallback: without the engine or a GPU these raise EngineUnavailableError.
"""

from __future__ import annotations

import math
import os
import threading
import time
from contextlib import contextmanager
from dataclasses import dataclass, field, replace
from typing import Iterator, NamedTuple

import numpy as np

from . import _native
from .cost import predicted_reads, predicted_writes, scratch_slots
from .errors import IndefiniteBlockError, NotSpdError, StorageError
from .layout import BlockLayout
from .prefixio import PrefixWriter
from .storage import MatrixFile, MatrixSource


@dataclass(frozen=True)
class Budget:
    """Byte budget for resident tiles (reference memdet.py:50-60)."""

    max_mem: int
    dtype_bytes: int = 8

    def __post_init__(self):
        if self.max_mem < 3 * self.dtype_bytes:
            raise ValueError(f"budget {self.max_mem} B below minimum {3 * self.dtype_bytes} B")


def select_blocking(m: int, budget: Budget) -> tuple[int, BlockLayout]:
    """Budget -> n_b with r = m sqrt(beta / c), in exact integers (reference memdet.py:63-80):
    r <= 1 -> 1, r <= 2/sqrt(3) -> 2, else ceil(2r) = least q with q^2 c >= 4 m^2 beta."""
    if m < 1:
        raise ValueError(f"matrix dimension must be >= 1, got {m}")
    c, beta = budget.max_mem, budget.dtype_bytes
    msq = m * m * beta
    if msq <= c:
        n_b = 1
    elif 3 * msq <= 4 * c:
        n_b = 2
    else:
        q = math.isqrt(4 * msq // c)
        while q * q * c < 4 * msq:
            q += 1
        n_b = q
    lay = BlockLayout.from_grid(m, n_b, beta)
    return lay.n_b, lay


class _Visit(NamedTuple):
    i: int
    j: int
    load_b: bool
    load_c: bool
    next_diag: bool


def _symmetric_visits(n_b: int, k: int) -> Iterator[_Visit]:
    """Stage-k tile walk (0-based) of the reference schedule (memdet.py:124-145): columns right
    to left, each starting on its diagonal tile, then rows k+1..j-1; ends on (k+1, k+1)."""
    for j in range(n_b - 1, k, -1):
        first = True
        for i in (j, *range(k + 1, j)):
            yield _Visit(i, j, load_b=first and j == n_b - 1, load_c=i != j,
                         next_diag=(i == j == k + 1))
            first = False


@dataclass(frozen=True)
class ScheduleEntry:
    i: int
    j: int
    loads: tuple[str, ...]
    target: str


def _generic_visits(n_b: int, k: int):
    """Stage-k walk (0-based) of the generic case (memdet.py:97-121): rows bottom-up, the
    column direction alternating per row so one of B / C is reused between consecutive visits;
    yields (i, j, new_row, load_b, next_diag)."""
    for i in range(n_b - 1, k, -1):
        asc = (i - k) % 2 == 0
        js = range(k + 1, n_b) if asc else range(n_b - 1, k, -1)
        first = k + 1 if asc else n_b - 1
        for j in js:
            yield i, j, j == first, i == n_b - 1 or j != first, i == j == k + 1


def schedule(n_b: int, case: str, k: int) -> list[ScheduleEntry]:
    """Reference tile-visit order for stage k (1-based) with fresh-load annotations
    (memdet.py:156-177); the out-of-core engine walks the same order."""
    if case not in ("generic", "symmetric"):
        raise ValueError(f"case must be 'generic' or 'symmetric', got {case!r}")
    if not 1 <= k < n_b:
        raise ValueError(f"stage k must satisfy 1 <= k < n_b, got k={k}, n_b={n_b}")
    out = []
    if case == "generic":
        for i, j, new_row, load_b, nd in _generic_visits(n_b, k - 1):
            loads = tuple(x for x, on in (("B", load_b), ("C", new_row)) if on)
            out.append(ScheduleEntry(i + 1, j + 1, loads, "resident" if nd else "store"))
        return out
    for v in _symmetric_visits(n_b, k - 1):
        loads = tuple(x for x, on in (("B", v.load_b), ("C", v.load_c)) if on)
        out.append(ScheduleEntry(v.i + 1, v.j + 1, loads, "resident" if v.next_diag else "store"))
    return out


@dataclass(frozen=True)
class RunInfo:
    """Reference RunInfo fields (memdet.py:180-198) plus engine diagnostics.

    blocks_read / blocks_written / scratch_slots are the reference schedule's counts for the
    reported n_b (cost.py:79-101).  In-core runs keep the matrix resident in HBM and move
    h2d_bytes / d2h_bytes over PCIe instead; out-of-core runs walk the reference schedule on
    an ooc_blocks grid and report the block transfers they actually made (ooc_reads /
    ooc_writes / ooc_scratch — equal to the reference counters when ooc_blocks == n_b)."""

    m: int
    case: str
    n_b: int
    b: int
    blocks_read: int
    blocks_written: int
    scratch_slots: int
    wall_seconds: float
    device_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernel_launches: int = 0
    engine_tile: int = 128
    engine: str = "b200-sm100a"
    out_of_core: bool = False
    ooc_blocks: int = 0
    ooc_block: int = 0
    ooc_reads: int = 0
    ooc_writes: int = 0
    ooc_scratch: int = 0

    def to_json_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.__dataclass_fields__}


def _block_logdets(prefix: np.ndarray, b: int) -> np.ndarray:
    """Per-block log|det| contributions: prefix differences at the reference block
    boundaries q = k*b (prefixes agree across pivoting variants exactly there)."""
    ends = np.minimum(np.arange(b, len(prefix) + b, b), len(prefix)) - 1
    vals = np.asarray(prefix, dtype=np.float64)[ends]
    return np.diff(np.concatenate([[0.0], vals]))


@dataclass(frozen=True)
class SpdResult:
    """prefix[q-1] = logdet of the leading q x q principal submatrix (no pivoting)."""

    prefix: np.ndarray
    info: RunInfo
    d: np.ndarray | None = field(default=None, repr=False)

    @property
    def logabsdet(self) -> float:
        return float(self.prefix[-1])

    sign = 1

    @property
    def block_logdets(self) -> np.ndarray:
        return _block_logdets(self.prefix, self.info.b)


@dataclass(frozen=True)
class GenericResult:
    """log|det| and sign of a generic matrix (reference memdet.py:201-205)."""

    logabsdet: float
    sign: int
    info: RunInfo


@dataclass(frozen=True)
class SymmetricResult:
    """perm / prefix / prefix_signs as the reference (memdet.py:208-228): prefix[q-1] is
    log|det| of M[perm[:q], perm[:q]]."""

    perm: np.ndarray
    prefix: np.ndarray
    prefix_signs: np.ndarray
    info: RunInfo
    d: np.ndarray | None = field(default=None, repr=False)

    @property
    def logabsdet(self) -> float:
        return float(self.prefix[-1])

    @property
    def sign(self) -> int:
        return int(self.prefix_signs[-1])

    @property
    def block_logdets(self) -> np.ndarray:
        return _block_logdets(self.prefix, self.info.b)


def _pick_layout(m: int, itemsize: int, max_mem, num_blocks) -> BlockLayout:
    if num_blocks is not None:
        return BlockLayout.from_grid(m, num_blocks, itemsize)
    if max_mem is None:
        raise ValueError("either max_mem or num_blocks is required")
    return select_blocking(m, Budget(max_mem, itemsize))[1]


# Engine contexts (HBM workspaces) are leased, one run at a time: a run takes an idle context
# of its (device, m, mode, plan) key or creates one, and returns it to the idle pool when it has
# fetched its outputs, so repeated runs on the same order reuse their allocation (a plan cache)
# while concurrent runs -- distinct files may proceed in parallel -- each own
# their workspace.  Creating a context first frees every IDLE context (HBM); a context in use is
# never closed, and release_engine_cache() closes those only when they come back.
_ctx_idle: dict = {}
_ctx_lock = threading.Lock()
_ctx_generation = 0


def _ctx_matches(ctx: _native.Context, mode: int, num_blocks: int, max_mem: int) -> bool:
    # an in-core plan ignores the reference tiling (except the block-pivoted LDL and LU, which
    # pivot inside the reference's blocks); an out-of-core one is built from it
    tiled = ctx.out_of_core or mode in (_native.MODE_LDL_PIV, _native.MODE_LU)
    return not tiled or ctx.key[4:6] == (num_blocks, max_mem)


@contextmanager
def _lease(m: int, mode: int, device: int, hbm_budget=None, num_blocks=None, max_mem=None,
           out_of_core=None, emulation=False, f32_arith=False, devices=(),
           scratch_dir=None) -> Iterator[_native.Context]:
    global _ctx_generation
    kw = dict(hbm_budget=int(hbm_budget or 0), num_blocks=int(num_blocks or 0),
              max_mem=int(max_mem or 0), force_out_of_core=bool(out_of_core), emulation=bool(emulation),
              f32_arith=bool(f32_arith), devices=tuple(devices), scratch_dir=scratch_dir)
    base = (device, m, mode, kw["hbm_budget"], kw["force_out_of_core"], kw["emulation"], kw["f32_arith"],
            kw["devices"], scratch_dir)
    ctx = None
    stale = []
    with _ctx_lock:
        idle = _ctx_idle.get(base, [])
        for i, c in enumerate(idle):
            if _ctx_matches(c, mode, kw["num_blocks"], kw["max_mem"]):
                ctx = idle.pop(i)
                break
        if ctx is None:  # free the idle workspaces before allocating a new one
            for k in list(_ctx_idle):
                stale.extend(_ctx_idle.pop(k))
        gen = _ctx_generation
    for c in stale:
        c.close()
    if ctx is None:
        ctx = _native.Context(m, mode, device, **kw)
    try:
        yield ctx
    finally:
        with _ctx_lock:
            keep = gen == _ctx_generation
            if keep:
                _ctx_idle.setdefault(base, []).append(ctx)
        if not keep:
            ctx.close()


def release_engine_cache():
    """Free the idle HBM workspaces (contexts in use are freed when their run returns them)."""
    global _ctx_generation
    with _ctx_lock:
        _ctx_generation += 1
        stale = [c for v in _ctx_idle.values() for c in v]
        _ctx_idle.clear()
    for c in stale:
        c.close()


def _scratch_dir(scratch_dir):
    """The reference's scratch directory rule (storage.py:200-204) minus its final fallback: the
    argument, else $OOCDET_SCRATCH_DIR, else None -- then the engine keeps an out-of-core
    scratchpad in lazily touched host memory rather than a file."""
    d = scratch_dir if scratch_dir is not None else os.environ.get("OOCDET_SCRATCH_DIR")
    return os.fspath(d) if d else None


def _run_engine(src: MatrixSource, mode: int, device: int, lay: BlockLayout, max_mem, hbm_budget,
                out_of_core, emulation=False, devices=(), scratch_dir=None):
    dcode = _native.B2D_F64 if src.dtype == np.float64 else _native.B2D_F32
    m = src.m
    if len(devices) > 1:
        return _run_multi(src, mode, dcode, devices, hbm_budget, out_of_core, lay.n_b)
    # the out-of-core tile walk starts from the reference tiling (num_blocks / max_mem)
    ooc_kw = dict(hbm_budget=hbm_budget, num_blocks=lay.n_b, out_of_core=out_of_core, scratch_dir=scratch_dir)
    if src.device_ptr is not None and mode == _native.MODE_LU:
        # the generic walk streams reference blocks from host memory
        src.host, src.device_ptr = src.keepalive.cpu().numpy(), None
    if src.device_ptr is not None and out_of_core:
        raise ValueError("out_of_core=True needs a host matrix (the device copy already fits)")
    # float32 files under block pivoting factor in f32 with the reference's own rounding sequence
    # (memdet.py:337-338, _ldl.pyx `floating`, dense.py:73 eps of the file dtype): in core
    f32_arith = (mode == _native.MODE_LDL_PIV and src.dtype == np.float32
                 and os.environ.get("B2D_F32_ARITH", "1") != "0")
    if f32_arith and out_of_core:
        raise ValueError("float32 memdet_ldl factors in core (f32 arithmetic); out_of_core=True is not available")
    on_device = src.device_ptr is not None
    kw = ooc_kw if (not on_device or mode == _native.MODE_LDL_PIV) else {}
    if f32_arith:
        kw = dict(kw, out_of_core=None)
    with _lease(m, mode, src.device_index if on_device else device, emulation=emulation, f32_arith=f32_arith,
                **kw) as ctx:
        if on_device and mode == _native.MODE_LDL_PIV and ctx.out_of_core:
            # the block-pivoted LDL runs in core when the reference's blocks are tile-aligned and
            # fit; else the block walk, which streams reference blocks from host memory
            src.host, src.device_ptr, on_device = src.keepalive.cpu().numpy(), None, False
        if on_device:
            import torch

            stream = torch.cuda.current_stream(src.device_index).cuda_stream
            ctx.factor_device_async(src.device_ptr, src.lda, dcode, stream)
        else:
            a, lda = src.host_rowmajor()
            ctx.factor_host_async(a.ctypes.data, lda, dcode, 0)
        d = np.empty(m, np.float64)
        prefix = np.empty(m, np.float64)
        rc, fail, info = ctx.fetch(d, prefix)
        if rc == _native.B2D_ERR_NOT_SPD:
            raise NotSpdError(f"leading minor of order {fail + 1} is not positive-definite "
                              f"(global pivot {fail})")
        if rc == _native.B2D_ERR_INDEFINITE:
            raise IndefiniteBlockError(f"LDL pivot {fail} below tolerance: {_native.last_error()}")
        _native.check(rc, "memdet engine")
        perm = None
        if mode in (_native.MODE_LDL_PIV, _native.MODE_LU):
            perm = np.empty(m, np.int64)
            ctx.fetch_perm(perm)
        ooc = ctx.out_of_core
    if mode == _native.MODE_LU:
        return d, prefix, info, ooc, (perm, fail)
    return d, prefix, info, ooc, perm


def _run_multi(src: MatrixSource, mode: int, dcode: int, devices, hbm_budget, out_of_core, num_blocks):
    """Several devices in this process (engine multi-device context): each device
    ingests only its own outer panels -- from host memory, or read in place from a device tensor
    over NVLink peer access."""
    if out_of_core:
        raise ValueError("out_of_core=True is single-device (the multi-device plan shards the matrix in HBM)")
    m = src.m
    # the block-pivoted LDL's stages are the reference's blocks (num_blocks)
    with _lease(m, mode, devices[0], hbm_budget=hbm_budget, num_blocks=num_blocks, devices=devices) as ctx:
        if src.device_ptr is not None:
            import torch

            torch.cuda.synchronize(src.device_index)  # the engine orders its ranks after the legacy stream
            ctx.factor_device_async(src.device_ptr, src.lda, dcode, 0)
        else:
            a, lda = src.host_rowmajor()
            ctx.factor_host_async(a.ctypes.data, lda, dcode, 0)
        d = np.empty(m, np.float64)
        prefix = np.empty(m, np.float64)
        rc, fail, info = ctx.fetch(d, prefix)
        if rc == _native.B2D_ERR_NOT_SPD:
            raise NotSpdError(f"leading minor of order {fail + 1} is not positive-definite "
                              f"(global pivot {fail})")
        if rc == _native.B2D_ERR_INDEFINITE:
            raise IndefiniteBlockError(f"LDL pivot {fail} below tolerance: {_native.last_error()}")
        _native.check(rc, "memdet engine (multi-device)")
        perm = None
        if mode == _native.MODE_LDL_PIV:
            perm = np.empty(m, np.int64)
            ctx.fetch_perm(perm)
    return d, prefix, info, False, perm


def _memdet(matrix, mode, case_label, max_mem, num_blocks, device, assume, hbm_budget=None,
            out_of_core=None, schur="dmma", devices=None, scratch_dir=None):
    if schur not in ("dmma", "ozaki"):
        raise ValueError(f"schur must be 'dmma' or 'ozaki', got {schur!r}")
    t0 = time.perf_counter()
    src = MatrixSource(matrix, assume)
    if src.symmetry == "generic" and mode != _native.MODE_LU:
        raise ValueError("symmetric driver requires a symmetric or spd input file")
    lay = _pick_layout(src.m, src.dtype.itemsize, max_mem, num_blocks)
    sdir = _scratch_dir(scratch_dir)
    if sdir is not None and lay.n_b > 2 and not os.path.isdir(sdir):
        # the reference creates its scratchpad file there whenever it has slots (storage.py:147-165)
        raise StorageError(f"scratch directory {sdir!r} does not exist")
    devices = tuple(int(x) for x in devices) if devices else ()
    if len(devices) > 1 and schur != "dmma":
        raise ValueError("schur='ozaki' is single-device")
    d, prefix, cinfo, ooc, perm = _run_engine(src, mode, device, lay, max_mem, hbm_budget, out_of_core,
                                              schur == "ozaki", devices, sdir)
    nb = lay.n_b
    case = "generic" if mode == _native.MODE_LU else "symmetric"
    info = RunInfo(m=src.m, case=case_label, n_b=nb, b=lay.b,
                   blocks_read=predicted_reads(nb, case),
                   blocks_written=predicted_writes(nb, case),
                   scratch_slots=scratch_slots(nb, case),
                   wall_seconds=time.perf_counter() - t0, device_ms=float(cinfo.device_ms),
                   h2d_bytes=int(cinfo.h2d_bytes), d2h_bytes=int(cinfo.d2h_bytes),
                   kernel_launches=int(cinfo.kernel_launches), engine_tile=int(cinfo.tile),
                   out_of_core=ooc, ooc_blocks=int(cinfo.ooc_blocks), ooc_block=int(cinfo.ooc_block),
                   ooc_reads=int(cinfo.ooc_reads), ooc_writes=int(cinfo.ooc_writes),
                   ooc_scratch=int(cinfo.ooc_scratch))
    return d, prefix.astype(src.dtype, copy=False), info, perm


def memdet_cholesky(matrix, *, max_mem=None, num_blocks=None, scratch_dir=None, prefix_out=None,
                    device: int = 0, assume: str | None = None, hbm_budget: int | None = None,
                    out_of_core: bool | None = None, schur: str = "dmma", devices=None) -> SpdResult:
    """Prefix log-determinants of an SPD matrix (blocked Cholesky, no pivoting).

    prefix[q-1] = logdet of the leading q x q principal submatrix, summed from 2 log L_ii;
    NotSpdError on the first non-positive leading minor.  A matrix whose packed lower triangle
    exceeds `hbm_budget` (default: free HBM) — or any host matrix with out_of_core=True — runs
    the reference's out-of-core tile walk, blocks streamed between host memory and HBM.  Its
    scratchpad lives in a temp file under `scratch_dir` (else $OOCDET_SCRATCH_DIR; reference
    storage.py:147-204: capacity bounded by disk), or, with neither, in lazily touched host memory;
    either way transfers are staged through small pinned rings, so nothing is pinned up front.
    schur="ozaki" runs the in-core trailing Schur updates as FP64 emulated on the int8 tcgen05
    tensor cores (8-slice Ozaki scheme, error ~3 u relative to sum |a b|); the
    default "dmma" uses the FP64 tensor cores.  devices=[d0, d1, ...] shards the factorisation over
    several devices of this process (1-D block-cyclic outer panels, each device ingesting only its
    own panels, panels exchanged over NVLink); hbm_budget is then per device."""
    d, prefix, info, _ = _memdet(matrix, _native.MODE_CHOLESKY, "spd", max_mem, num_blocks, device, assume,
                                 hbm_budget, out_of_core, schur, devices, scratch_dir)
    res = SpdResult(prefix=prefix, info=info, d=d)
    if prefix_out is not None:
        with PrefixWriter(prefix_out) as w:
            w.append(prefix, np.ones(len(prefix), dtype=np.int64))
    return res


def _perm_parity(perm: np.ndarray) -> int:
    """Sign of a permutation (cycle decomposition)."""
    seen = np.zeros(len(perm), dtype=bool)
    swaps = 0
    for i in range(len(perm)):
        if not seen[i]:
            j, length = i, 0
            while not seen[j]:
                seen[j] = True
                j = int(perm[j])
                length += 1
            swaps += length - 1
    return -1 if swaps % 2 else 1


def memdet_lu(matrix, *, max_mem=None, num_blocks=None, scratch_dir=None, device: int = 0,
              assume: str | None = None, hbm_budget: int | None = None,
              out_of_core: bool | None = None) -> GenericResult:
    """log|det| and sign of a generic (non-symmetric) matrix via blocked LU with block-local
    partial pivoting over the reference's blocks (memdet.py:268-319): in core when its blocks
    start on tile boundaries and the matrix fits (the stages with the matrix resident), else
    the reference's generic block walk out of core.  A singular matrix returns (-inf, 0)
    rather than raising, as the reference.  Pivots are searched inside the reference's diagonal
    blocks, as the reference's (a block-local pivot search sees only its block, so the grid is
    never refined); blocks over 6144 rows raise NotImplementedError (the cluster panel kernel's
    reach) and a walk that does not fit the HBM budget raises MemoryError."""
    d, prefix, info, (perm, fail) = _memdet(matrix, _native.MODE_LU, "generic", max_mem, num_blocks, device,
                                            assume or "generic", hbm_budget, out_of_core, scratch_dir=scratch_dir)
    # the reference's counters for its walk (scratch = the peak number of distinct blocks
    # written, storage.py:265-267); it stops at a singular stage (memdet.py:293-294), whose
    # position the engine reports when its block grid is the reference's
    stage = info.n_b
    if fail >= 0 and info.ooc_blocks == info.n_b and info.ooc_block > 0:
        stage = fail // info.ooc_block
    elif fail >= 0 and not info.out_of_core:  # in core: the engine's blocks are the reference's
        stage = fail // info.b
    r, w, slots = _generic_counts_until(info.n_b, stage)
    info = replace(info, blocks_read=r, blocks_written=w, scratch_slots=slots)
    if fail >= 0 or not np.all(np.isfinite(d)) or np.any(d == 0):
        return GenericResult(-np.inf, 0, info)
    sign = _perm_parity(perm) * int(np.prod(np.sign(d)))
    return GenericResult(float(prefix[-1]), sign, info)


def _generic_counts_until(n_b: int, stage: int):
    """(reads, writes, scratch slots) of the reference generic walk when it stops while
    factoring the diagonal block of `stage` (memdet.py:283-319)."""
    reads, writes, keys = 1, 0, set()
    for k in range(min(stage, n_b - 1)):
        t = n_b - 1 - k
        for i, j, new_row, load_b, nd in _generic_visits(n_b, k):
            reads += int(new_row) + int(load_b) + 1
            if i == n_b - 1:  # the bottom row solves and stores the row-k blocks
                last = n_b - 1 if (i - k) % 2 == 0 else k + 1
                if t > 2 or j != last:
                    writes += 1
                    keys.add((k, j))
            if not nd:
                writes += 1
                keys.add((i, j))
    return reads, writes, len(keys)


def memdet_ldl(matrix, *, max_mem=None, num_blocks=None, scratch_dir=None, prefix_out=None,
               device: int = 0, assume: str | None = None, pivoting: str = "block",
               hbm_budget: int | None = None, out_of_core: bool | None = None,
               schur: str = "dmma", devices=None) -> SymmetricResult:
    """Prefix log-determinants of a symmetric matrix via blocked LDL^T.

    pivoting="block" reproduces the reference's block-local 1x1 diagonal pivoting
    (_ldl.pyx:30-46; perm and prefixes of the permuted minors).  pivoting="none" is the
    unpivoted LDL^T (D = L_ii^2 of the Cholesky factor, perm = identity): its prefixes are
    the natural-order leading minors and coincide with the pivoted ones at every block
    boundary q = k*b and at q = m.  schur and devices as memdet_cholesky."""
    if pivoting not in ("block", "none"):
        raise ValueError(f"pivoting must be 'block' or 'none', got {pivoting!r}")
    mode = _native.MODE_LDL_PIV if pivoting == "block" else _native.MODE_LDL_NOPIV
    d, prefix, info, perm = _memdet(matrix, mode, "symmetric", max_mem, num_blocks, device, assume, hbm_budget,
                                    out_of_core, schur, devices, scratch_dir)
    m = len(prefix)
    if mode == _native.MODE_LDL_NOPIV:
        perm = np.arange(m, dtype=np.int64)
        signs = np.ones(m, dtype=np.int64)
    else:  # memdet.py:407: cumprod(sign d)
        signs = np.cumprod(np.sign(d)).astype(np.int64)
    res = SymmetricResult(perm=perm, prefix=prefix, prefix_signs=signs, info=info, d=d)
    if prefix_out is not None:
        with PrefixWriter(prefix_out) as w:
            w.append(prefix, signs)
    return res


__all__ = ["Budget", "select_blocking", "schedule", "ScheduleEntry", "RunInfo", "SpdResult",
           "SymmetricResult", "memdet_cholesky", "memdet_ldl", "release_engine_cache", "MatrixFile"]
