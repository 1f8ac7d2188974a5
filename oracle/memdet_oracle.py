"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the reference's blocked symmetric MEMDET drivers:

* `memdet_symmetric`  <- `_memdet_symmetric`            memdet.py:322-389
* `memdet_cholesky`   <- `memdet_cholesky`              memdet.py:415-433
* `memdet_ldl`        <- `memdet_ldl`                   memdet.py:392-412
* `stage_visits`      <- `_symmetric_stage`             memdet.py:124-145
* `from_grid`         <- `BlockLayout.from_grid`        layout.py:35-51
* `select_blocking`   <- `select_blocking`              memdet.py:63-80
* `chol_tile`         <- `cholesky_inplace`             kernels/dense.py:84-91 (LAPACK ?potrf)
* `ldl_tile`          <- `ldl_inplace` + `ldl_factor`   kernels/dense.py:57-81, _ldl.pyx:21-61
* `perm_from_swaps`   <- `perm_from_swaps`              kernels/dense.py:25-30
* counters            <- `BlockStore` read/write counts storage.py:229-263

The reference streams tiles through an on-disk scratchpad; here the whole matrix lives in a
NumPy array and the block I/O is *counted* (one per whole-block read / scratch write, exactly
where the reference's BlockStore would move a block), so the counters equal the reference's.
Arithmetic per tile is the same third-party LAPACK/BLAS the reference calls (SciPy ?potrf and
?trtrs, NumPy matmul), and the pivoted LDL tile uses the C restatement in `ldl_tile.c`.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
from scipy.linalg import cholesky as _lapack_potrf
from scipy.linalg import solve_triangular as _lapack_trtrs

PIVOT_TOL_SCALE = 64.0  # kernels/dense.py:22

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_ldl.so")
_lib = None


class OracleNotSpd(Exception):
    """Stands for oocdet.errors.NotSpdError (errors.py:36-37)."""


class OracleIndefinite(Exception):
    """Stands for oocdet.errors.IndefiniteBlockError (errors.py:40-41)."""

    def __init__(self, msg, step):
        super().__init__(msg)
        self.step = step


_SRCS = ("ldl_tile.c", "ldl32_model.c")


def build_oracle_lib(force: bool = False) -> str:
    """Compile ldl_tile.c and ldl32_model.c with gcc into oracle/_build (test infrastructure).
    -ffp-contract=off: the restated roundings are the written ones (FMA only where fmaf says)."""
    srcs = [os.path.join(_HERE, f) for f in _SRCS]
    if force or not os.path.exists(_LIB_PATH) or any(os.path.getmtime(_LIB_PATH) < os.path.getmtime(f) for f in srcs):
        os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
        rc = os.system(f"gcc -O2 -ffp-contract=off -fPIC -shared -o {_LIB_PATH} {' '.join(srcs)} -lm")
        if rc != 0:
            raise RuntimeError("failed to build the oracle C sources")
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build_oracle_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        for name, ct in (("oracle_ldl_tile_f64", ctypes.c_double), ("oracle_ldl_tile_f32", ctypes.c_float)):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int64
            fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double]
        fn = lib.oracle_memdet_ldl32
        fn.restype = ctypes.c_int64
        fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                       ctypes.c_void_p]
        _lib = lib
    return _lib


# ----------------------------------------------------------------------------- geometry


@dataclass(frozen=True)
class Layout:
    m: int
    n_b: int
    b: int
    tail: int

    def size(self, k: int) -> int:
        return self.tail if k == self.n_b - 1 else self.b

    def span(self, k: int) -> slice:
        return slice(k * self.b, k * self.b + self.size(k))


def from_grid(m: int, n_b: int) -> Layout:
    """layout.py:35-51 — shrink n_b until ceil(m / b) == n_b, b = 1 + (m-1)//n_b."""
    if m < 1 or n_b < 1:
        raise ValueError("m and n_b must be >= 1")
    n_b = min(n_b, m)
    while True:
        b = 1 + (m - 1) // n_b
        need = -(-m // b)
        if need == n_b:
            return Layout(m, n_b, b, m - (n_b - 1) * b)
        n_b = need


def select_blocking(m: int, max_mem: int, beta: int = 8) -> int:
    """memdet.py:63-80 — exact-integer budget rule r = m*sqrt(beta/c)."""
    if max_mem < 3 * beta:
        raise ValueError("budget below minimum")
    msq = m * m * beta
    if msq <= max_mem:
        n_b = 1
    elif 3 * msq <= 4 * max_mem:
        n_b = 2
    else:
        q = math.isqrt((4 * msq) // max_mem)
        while q * q * max_mem < 4 * msq:
            q += 1
        n_b = q
    return from_grid(m, n_b).n_b


def stage_visits(n_b: int, k: int):
    """memdet.py:124-145 — stage-k visits (0-based) of the symmetric tile walk.

    Yields dicts with the same flags the reference's `_Visit` carries.  Columns run right
    to left; each column starts on its diagonal tile, then sweeps rows k+1..j-1.
    """
    for j in range(n_b - 1, k, -1):
        last_col = j == n_b - 1
        for pos, i in enumerate([j, *range(k + 1, j)]):
            off = i != j
            yield dict(i=i, j=j, col_start=pos == 0, load_b=pos == 0 and last_col,
                       load_c=off, solve_c=off and last_col,
                       write_c=off and last_col and n_b > 2 and i < j - 1,
                       next_diag=(i == k + 1 and j == k + 1))


def scratch_capacity(n_b: int) -> int:
    """cost.py:95-101 (symmetric case)."""
    return 0 if n_b <= 2 else (n_b * n_b + n_b - 8) // 2


def predicted_reads(n_b: int) -> int:
    """cost.py:79-83 (symmetric case)."""
    return (2 * n_b ** 3 - 3 * n_b ** 2 + 7 * n_b) // 6


def predicted_writes(n_b: int) -> int:
    """cost.py:86-92 (symmetric case)."""
    return 0 if n_b <= 2 else (n_b ** 3 + 3 * n_b ** 2 - 22 * n_b + 24) // 6


# ----------------------------------------------------------------------------- tile kernels


def perm_from_swaps(swaps) -> np.ndarray:
    """kernels/dense.py:25-30 — LAPACK swap list -> permutation vector."""
    perm = np.arange(len(swaps), dtype=np.int64)
    for r, t in enumerate(swaps):
        if t != r:
            perm[r], perm[t] = perm[t], perm[r]
    return perm


def chol_tile(a: np.ndarray) -> np.ndarray:
    """kernels/dense.py:84-91 — LAPACK ?potrf (lower); returns diag(L)."""
    try:
        low = _lapack_potrf(a, lower=True, check_finite=False)
    except np.linalg.LinAlgError as exc:
        raise OracleNotSpd(str(exc)) from exc
    a[:] = low
    return np.diagonal(a).copy()


def ldl_tile(a: np.ndarray):
    """kernels/dense.py:57-81 + _ldl.pyx:21-61 via the C restatement (ldl_tile.c)."""
    n = a.shape[0]
    amax = float(np.max(np.abs(a))) if n else 0.0
    if n and amax == 0.0:
        raise OracleIndefinite("LDL on an all-zero tile", 0)
    tol = PIVOT_TOL_SCALE * float(np.finfo(a.dtype).eps) * amax
    lib = _load()
    work_a = np.ascontiguousarray(a)
    swaps = np.empty(n, np.int64)
    d = np.empty(n, a.dtype)
    work = np.empty(n, a.dtype)
    fn = lib.oracle_ldl_tile_f64 if a.dtype == np.float64 else lib.oracle_ldl_tile_f32
    fail = fn(work_a.ctypes.data, n, n, swaps.ctypes.data, d.ctypes.data, work.ctypes.data, tol)
    if work_a is not a:
        a[:] = work_a
    if fail >= 0:
        raise OracleIndefinite(f"LDL pivot {fail} below tolerance {tol:.3e}", int(fail))
    return swaps, d


def lower_solve(l: np.ndarray, b: np.ndarray, unit: bool):
    """kernels/dense.py:94-99 — B <- L^{-1} B (LAPACK ?trtrs)."""
    b[:] = _lapack_trtrs(l, b, lower=True, unit_diagonal=unit, check_finite=False)


def schur_update(tile: np.ndarray, c: np.ndarray, b: np.ndarray):
    """kernels/dense.py:109-116 (form "ct_b") — T <- T - C^T B (NumPy matmul -> BLAS ?gemm)."""
    tile -= c.T @ b


# ----------------------------------------------------------------------------- driver


@dataclass
class OracleInfo:
    m: int
    n_b: int
    b: int
    blocks_read: int
    blocks_written: int
    scratch_slots: int


def memdet_symmetric(mat: np.ndarray, n_b: int, pivoted: bool, inplace: bool = False):
    """memdet.py:322-389 — blocked right-looking LDL^T (pivoted) or Cholesky (not).

    `mat` is the full symmetric matrix (row-major, as stored in a MEMDET01 file).  Tiles
    (i, j) with i <= j of the row-major upper triangle are the ones the reference reads;
    each stage factors the diagonal tile, lower-solves the row-k tiles once, scales them by
    D^{-1} for LDL, and applies `T -= C^T B` to every trailing (i <= j) tile.
    Returns (d, perm, info): d = D (LDL) or diag(L) (Cholesky), perm block-local pivots.
    inplace=True overwrites `mat` (full-size goldens whose copy would not fit host memory).
    """
    m = mat.shape[0]
    lay = from_grid(m, n_b)
    nb = lay.n_b
    work = mat if inplace else np.array(mat, copy=True)  # stands in for file + scratchpad
    d_all = np.empty(m, mat.dtype)
    perm_all = np.arange(m, dtype=np.int64)
    reads = 1  # tile (0, 0) loaded before stage 0 (memdet.py:345)
    writes = 0
    slots = set()
    for k in range(nb):
        sk = lay.span(k)
        akk = work[sk, sk]
        if pivoted:
            swaps, dk = ldl_tile(akk)
            pk = perm_from_swaps(swaps)
        else:
            dk = chol_tile(akk)
            pk = None
        off = k * lay.b
        d_all[off:off + len(dk)] = dk
        if pk is not None:
            perm_all[off:off + len(dk)] = off + pk
        if k == nb - 1:
            break
        lkk = akk  # ?trtrs reads only the lower triangle (unit diagonal for LDL)
        # solved (and for LDL unscaled) row-k tiles; reference solves each once
        solved = {}
        for v in stage_visits(nb, k):
            i, j = v["i"], v["j"]
            if v["load_b"]:
                reads += 1
            if v["load_c"]:
                reads += 1
            if v["write_c"]:
                writes += 1
                slots.add((k, i))
            for t in (i, j):
                if t not in solved:
                    blk = work[sk, lay.span(t)].copy()
                    if pk is not None:
                        blk = blk[pk]
                    lower_solve(lkk, blk, unit=pivoted)
                    solved[t] = blk
            reads += 1  # the target tile (memdet.py:384)
            c_t = solved[i]
            b_t = solved[j] / dk[:, None] if pivoted else solved[j]
            schur_update(work[lay.span(i), lay.span(j)], c_t, b_t)
            if not v["next_diag"]:
                writes += 1
                slots.add((i, j))
    info = OracleInfo(m=m, n_b=nb, b=lay.b, blocks_read=reads, blocks_written=writes,
                      scratch_slots=len(slots))
    return d_all, perm_all, info


def memdet_cholesky(mat: np.ndarray, n_b: int, inplace: bool = False):
    """memdet.py:415-433 — prefix[q-1] = sum_{i<q} 2 log L_ii (sequential cumsum)."""
    d, _, info = memdet_symmetric(mat, n_b, pivoted=False, inplace=inplace)
    return np.cumsum(2.0 * np.log(d)), info


def memdet_ldl(mat: np.ndarray, n_b: int, inplace: bool = False):
    """memdet.py:392-412 — (perm, prefix = cumsum log|d|, signs = cumprod sign d)."""
    d, perm, info = memdet_symmetric(mat, n_b, pivoted=True, inplace=inplace)
    prefix = np.cumsum(np.log(np.abs(d)))
    signs = np.cumprod(np.sign(d)).astype(np.int64)
    return perm, prefix, signs, info


def stage0_flops(m: int, n_b: int) -> float:
    """Exact flops (2 x FMA count, cost.py:104-137 per-op formulas) of stage 0 of the schedule."""
    lay = from_grid(m, n_b)
    b = lay.b
    t = lay.n_b - 1
    potrf = b ** 3 / 3.0
    trsm = t * b ** 3
    schur = (t * (t + 1) // 2) * 2.0 * b ** 3
    return potrf + trsm + schur


def run_stage0(mat: np.ndarray, n_b: int):
    """Stage 0 of memdet_cholesky's schedule (bounded CPU-baseline sample): factor tile (0,0),
    solve the row-0 tiles, apply every stage-0 Schur update (memdet.py:346-387, k = 0)."""
    lay = from_grid(mat.shape[0], n_b)
    s0 = lay.span(0)
    work = np.array(mat, copy=True)
    akk = work[s0, s0]
    chol_tile(akk)
    lkk = akk
    solved = {}
    for v in stage_visits(lay.n_b, 0):
        i, j = v["i"], v["j"]
        for t in (i, j):
            if t not in solved:
                blk = work[s0, lay.span(t)].copy()
                lower_solve(lkk, blk, unit=False)
                solved[t] = blk
        tile = work[lay.span(i), lay.span(j)]
        tile -= solved[i].T @ solved[j]
    return work


def memdet_ldl32(mat: np.ndarray, n_b: int):
    """memdet.py:392-412 on a float32 file, with the f32 roundings of the reference's own calls on
    the golden host (ldl32_model.c): (perm, d (float32), fail or -1).  prefix as the reference:
    np.cumsum(np.log(np.abs(d))) in float32."""
    m = mat.shape[0]
    lay = from_grid(m, n_b)
    work = np.array(mat, dtype=np.float32, order="C", copy=True)
    d = np.zeros(m, np.float32)
    perm = np.arange(m, dtype=np.int64)
    fail = _load().oracle_memdet_ldl32(work.ctypes.data, m, lay.n_b, lay.b, d.ctypes.data, perm.ctypes.data)
    return perm, d, int(fail)
