"""MEMDET01 matrix files (reference storage.py:3-116) and matrix-argument normalisation.

Layout (little-endian): magic "MEMDET01", u32 version (1), u8 dtype (0 f64, 1 f32),
u8 symmetry (0 generic, 1 symmetric, 2 spd), 2 pad bytes, u64 m, pad to 64 bytes, then m*m
row-major elements.  The file length must be exactly 64 + m*m*itemsize."""

from __future__ import annotations

import os
import struct

import numpy as np

from .errors import StorageError

MAGIC = b"MEMDET01"
HEADER_SIZE = 64
VERSION = 1
_HEAD = struct.Struct("<8sIBBxxQ")
DTYPE_CODES = {"f64": 0, "f32": 1}
DTYPE_BY_CODE = {0: np.dtype(np.float64), 1: np.dtype(np.float32)}
SYMMETRY_CODES = {"generic": 0, "symmetric": 1, "spd": 2}
SYMMETRY_BY_CODE = {v: k for k, v in SYMMETRY_CODES.items()}


def _dtype_key(dtype) -> str:
    if isinstance(dtype, str) and dtype in DTYPE_CODES:
        return dtype
    try:
        dt = np.dtype(dtype)
    except TypeError:
        dt = None
    if dt == np.float64:
        return "f64"
    if dt == np.float32:
        return "f32"
    raise ValueError(f"unsupported dtype {dtype!r}; use f64 or f32")


class MatrixFile:
    """A dense m x m matrix in the MEMDET01 format."""

    def __init__(self, path, m: int, dtype, symmetry: str):
        self.path = str(path)
        self.m = int(m)
        self.dtype = np.dtype(dtype)
        self.symmetry = symmetry

    @classmethod
    def create(cls, path, m: int, dtype="f64", symmetry: str = "generic") -> "MatrixFile":
        if m < 1:
            raise ValueError(f"matrix dimension must be >= 1, got {m}")
        key = _dtype_key(dtype)
        if symmetry not in SYMMETRY_CODES:
            raise ValueError(f"unknown symmetry {symmetry!r}")
        npdt = DTYPE_BY_CODE[DTYPE_CODES[key]]
        head = _HEAD.pack(MAGIC, VERSION, DTYPE_CODES[key], SYMMETRY_CODES[symmetry], m)
        try:
            with open(path, "wb") as f:
                f.write(head.ljust(HEADER_SIZE, b"\0"))
                f.truncate(HEADER_SIZE + m * m * npdt.itemsize)
        except OSError as exc:
            raise StorageError(f"cannot create matrix file {path}: {exc}") from exc
        return cls(path, m, npdt, symmetry)

    @classmethod
    def open(cls, path) -> "MatrixFile":
        try:
            with open(path, "rb") as f:
                head = f.read(HEADER_SIZE)
        except OSError as exc:
            raise StorageError(f"cannot open matrix file {path}: {exc}") from exc
        if len(head) < HEADER_SIZE:
            raise StorageError(f"{path}: truncated header")
        magic, version, dcode, scode, m = _HEAD.unpack_from(head)
        if magic != MAGIC:
            raise StorageError(f"{path}: bad magic {magic!r}")
        if version != VERSION:
            raise StorageError(f"{path}: unsupported version {version}")
        if dcode not in DTYPE_BY_CODE:
            raise StorageError(f"{path}: unknown dtype code {dcode}")
        if scode not in SYMMETRY_BY_CODE:
            raise StorageError(f"{path}: unknown symmetry code {scode}")
        dt = DTYPE_BY_CODE[dcode]
        want = HEADER_SIZE + m * m * dt.itemsize
        got = os.path.getsize(path)
        if got != want:
            raise StorageError(f"{path}: length {got} != expected {want}")
        return cls(path, int(m), dt, SYMMETRY_BY_CODE[scode])

    def memmap(self, mode: str = "r") -> np.memmap:
        return np.memmap(self.path, dtype=self.dtype, mode=mode, offset=HEADER_SIZE,
                         shape=(self.m, self.m))


def write_matrix(path, values: np.ndarray, symmetry: str) -> MatrixFile:
    """Create a MEMDET01 file holding `values`."""
    values = np.asarray(values)
    mf = MatrixFile.create(path, values.shape[0], values.dtype, symmetry)
    mm = mf.memmap("r+")
    mm[:] = values
    mm.flush()
    del mm
    return mf


class MatrixSource:
    """Normalised matrix argument: MatrixFile / path (MEMDET01) / ndarray / memmap / torch tensor.

    `host` is a row-major 2-D array view (never copied unless its rows are not contiguous);
    `device_ptr` is set for CUDA tensors (row-major, contiguous rows)."""

    def __init__(self, matrix, assume: str | None = None):
        self.keepalive = None
        self.device_ptr = None
        self.device_index = None
        if isinstance(matrix, (str, os.PathLike)):
            matrix = MatrixFile.open(matrix)
        if isinstance(matrix, MatrixFile):
            self.symmetry = matrix.symmetry
            arr = matrix.memmap("r")
            self.dtype = matrix.dtype
            self.m = matrix.m
            self.host = arr
            return
        self.symmetry = assume or "symmetric"
        mod = type(matrix).__module__
        if mod.startswith("torch"):
            t = matrix
            if t.dim() != 2 or t.shape[0] != t.shape[1]:
                raise ValueError(f"matrix must be square, got shape {tuple(t.shape)}")
            import torch

            if t.dtype not in (torch.float64, torch.float32):
                raise ValueError(f"unsupported dtype {t.dtype}; use float64 or float32")
            self.dtype = np.dtype(np.float64 if t.dtype == torch.float64 else np.float32)
            self.m = int(t.shape[0])
            if t.stride(1) != 1:
                t = t.contiguous()
            self.keepalive = t
            self.lda = int(t.stride(0))
            if t.is_cuda:
                self.device_ptr = int(t.data_ptr())
                self.device_index = t.device.index or 0
                self.host = None
            else:
                self.host = t.numpy()
            return
        arr = np.asarray(matrix)
        if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
            raise ValueError(f"matrix must be square, got shape {arr.shape}")
        if arr.dtype not in (np.float64, np.float32):
            raise ValueError(f"unsupported dtype {arr.dtype}; use float64 or float32")
        self.dtype = arr.dtype
        self.m = int(arr.shape[0])
        self.host = arr

    def host_rowmajor(self):
        """(array, lda) with unit column stride."""
        a = self.host
        if a.strides[1] != a.itemsize or a.strides[0] % a.itemsize:
            a = np.ascontiguousarray(a)
            self.keepalive = a
        return a, a.strides[0] // a.itemsize
