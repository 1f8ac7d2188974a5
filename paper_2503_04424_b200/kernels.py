"""The reference's tile-kernel module on the GPU: a drop-in for `oocdet.kernels`
(kernels/__init__.py:24-45, dense.py:57-116), so the reference's own driver can run on this
engine by binding these names (memdet.py:36-44 imports them by name):

    import oocdet.memdet as M, paper_2503_04424_b200.kernels as K
    for name in ("cholesky_inplace", "ldl_inplace", "solve_lower_inplace", "schur_update"):
        setattr(M, name, getattr(K, name))

Same signatures, in-place semantics and errors on host NumPy tiles (strided views included).  The
arithmetic runs in the tile's dtype on the GPU (libmemdet_b200.so b2d_tile_*_host, ldl32.cu) with
the golden host's LAPACK / BLAS rounding sequence: the pivoted LDL, the triangular solves and the
Schur update are bit-identical to the reference there (tests/test_tile_seam_gpu.py); the Cholesky
tile agrees to rounding.  Each call copies its tile to the device and back: this is the seam for
the reference's driver, not the engine's hot path (memdet_cholesky / memdet_ldl keep the matrix
in HBM).  The generic-LU kernels (lu_inplace, solve_upper_right_inplace) are not provided.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import IndefiniteBlockError, NotSpdError, NumericalError

PIVOT_TOL_SCALE = 64.0  # dense.py:22
HAVE_COMPILED_LDL = True


def _code(a: np.ndarray) -> int:
    if a.dtype == np.float64:
        return _native.B2D_F64
    if a.dtype == np.float32:
        return _native.B2D_F32
    raise ValueError(f"unsupported tile dtype {a.dtype}; use float64 or float32")


class _Tile:
    """A C-contiguous working copy of a (possibly strided) tile, written back on exit."""

    def __init__(self, view: np.ndarray, write: bool = True):
        self.view, self.write = view, write
        self.buf = np.ascontiguousarray(view)

    def __enter__(self):
        return self.buf

    def __exit__(self, exc_type, *_):
        if exc_type is None and self.write and self.buf is not self.view:
            self.view[...] = self.buf


def perm_from_swaps(swaps: np.ndarray) -> np.ndarray:
    """LAPACK-style interchanges (swaps[r] exchanged with r at step r) -> the permutation with
    (P^T A P)[i, j] == A[perm[i], perm[j]] (dense.py:25-30)."""
    perm = np.arange(len(swaps), dtype=np.int64)
    for r, t in enumerate(np.asarray(swaps)):
        if t != r:
            perm[[r, t]] = perm[[t, r]]
    return perm


def ldl_inplace(a: np.ndarray):
    """LDL^T with 1x1 diagonal pivoting (largest |a_ii|, lowest index on ties): the strict lower
    triangle becomes unit L, returns (swaps, d); IndefiniteBlockError below the tolerance
    PIVOT_TOL_SCALE * eps(dtype) * max|A| or on an all-zero tile (dense.py:57-81)."""
    n = a.shape[0]
    if a.ndim != 2 or a.shape[1] != n:
        raise ValueError(f"tile must be square, got {a.shape}")
    code = _code(a)
    amax = float(np.max(np.abs(a))) if n else 0.0
    if n and amax == 0.0:
        raise IndefiniteBlockError("LDL on an all-zero tile")
    tol = PIVOT_TOL_SCALE * float(np.finfo(a.dtype).eps) * amax
    swaps = np.empty(n, dtype=np.int64)
    d = np.empty(n, dtype=a.dtype)
    fail = ctypes.c_int64(-1)
    with _Tile(a) as t:
        _native.check(_native.load().b2d_tile_ldl_host(t.ctypes.data, n, t.strides[0] // t.itemsize, code, tol,
                                                       swaps.ctypes.data, d.ctypes.data, ctypes.byref(fail), 0),
                      "b2d_tile_ldl_host")
        if fail.value >= 0:
            raise IndefiniteBlockError(f"LDL pivot {fail.value}: below tolerance {tol:.3e}")
    return swaps, d


def cholesky_inplace(a: np.ndarray) -> np.ndarray:
    """A = L L^T, L written to the lower triangle (zeros above); returns diag(L); NotSpdError when
    a leading minor is not positive-definite (dense.py:84-91)."""
    n = a.shape[0]
    code = _code(a)
    diag = np.empty(n, dtype=a.dtype)
    fail = ctypes.c_int64(-1)
    with _Tile(a) as t:
        _native.check(_native.load().b2d_tile_cholesky_host(t.ctypes.data, n, t.strides[0] // t.itemsize, code,
                                                            diag.ctypes.data, ctypes.byref(fail), 0),
                      "b2d_tile_cholesky_host")
        if fail.value >= 0:
            raise NotSpdError(f"tile is not positive-definite: leading minor of order {fail.value + 1}")
    return diag


def solve_lower_inplace(l: np.ndarray, b: np.ndarray, unit_diag: bool = False):
    """B <- L^{-1} B for lower-triangular L (dense.py:94-99)."""
    if not unit_diag and np.any(np.diagonal(l) == 0.0):
        raise NumericalError("singular lower-triangular solve (zero diagonal)")
    code = _code(b)
    n, w = b.shape
    lc = np.ascontiguousarray(l, dtype=b.dtype)
    with _Tile(b) as t:
        _native.check(_native.load().b2d_tile_solve_lower_host(lc.ctypes.data, n, lc.shape[1], t.ctypes.data, w,
                                                               t.strides[0] // t.itemsize, code, int(bool(unit_diag)), 0),
                      "b2d_tile_solve_lower_host")


def schur_update(s: np.ndarray, c: np.ndarray, b: np.ndarray, form: str = "ct_b"):
    """S <- S - C^T B ("ct_b") or S <- S - C B ("c_b") (dense.py:109-116)."""
    if form == "ct_b":
        ct = np.ascontiguousarray(c, dtype=s.dtype)
    elif form == "c_b":
        ct = np.ascontiguousarray(np.asarray(c).T, dtype=s.dtype)
    else:
        raise ValueError(f"unknown form {form!r}")
    bb = np.ascontiguousarray(b, dtype=s.dtype)
    k, m = ct.shape
    if bb.shape[0] != k or s.shape != (m, bb.shape[1]):
        raise ValueError(f"shape mismatch: s {s.shape}, c {np.shape(c)}, b {np.shape(b)} ({form})")
    code = _code(s)
    with _Tile(s) as t:
        _native.check(_native.load().b2d_tile_schur_update_host(t.ctypes.data, m, bb.shape[1],
                                                                t.strides[0] // t.itemsize, ct.ctypes.data, m,
                                                                bb.ctypes.data, bb.shape[1], k, code, 0),
                      "b2d_tile_schur_update_host")


__all__ = ["HAVE_COMPILED_LDL", "PIVOT_TOL_SCALE", "cholesky_inplace", "ldl_inplace", "perm_from_swaps",
           "schur_update", "solve_lower_inplace"]
