"""ctypes binding of libmemdet_b200.so (the C ABI in include/memdet_b200.h).

Loading is lazy and loud: if the library or a CUDA device is missing, calls raise
EngineUnavailableError.  There is no CPU fallback anywhere in the product path."""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libmemdet_b200.so")
# A/B experiments only (tools/): another build of the same library
LIB_PATH = os.environ.get("B2D_LIB_OVERRIDE", LIB_PATH)

B2D_OK = 0
B2D_ERR_USAGE = 2
B2D_ERR_NOT_SPD = 3
B2D_ERR_INDEFINITE = 4
B2D_ERR_CUDA = 5
B2D_ERR_NOMEM = 6
B2D_ERR_UNSUPPORTED = 7
B2D_ERR_STORAGE = 8

B2D_F64, B2D_F32 = 0, 1
MODE_CHOLESKY, MODE_LDL_NOPIV, MODE_LDL_PIV, MODE_LU = 0, 1, 2, 3


class RunInfoC(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "m", "n_b", "b", "tail", "blocks_read", "blocks_written", "scratch_slots", "tile",
        "n_tiles", "h2d_bytes", "d2h_bytes", "kernel_launches")] + [
        ("device_ms", ctypes.c_double), ("wall_seconds", ctypes.c_double)] + [
        (name, ctypes.c_int64) for name in ("ooc_blocks", "ooc_block", "ooc_reads", "ooc_writes",
                                            "ooc_scratch")]


class OptionsC(ctypes.Structure):
    _fields_ = [("hbm_budget", ctypes.c_int64), ("num_blocks", ctypes.c_int64),
                ("max_mem", ctypes.c_int64), ("force_out_of_core", ctypes.c_int32),
                ("host_scratch", ctypes.c_int32), ("emulation", ctypes.c_int32),
                ("f32_arith", ctypes.c_int32), ("ndev", ctypes.c_int32),
                ("devices", ctypes.c_int32 * 8), ("scratch_mode", ctypes.c_int32),
                ("scratch_dir", ctypes.c_char_p)]


MAX_PEERS = 8


class TileMapC(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("ld", ctypes.c_int64), ("packed_nt", ctypes.c_int32),
                ("rmod", ctypes.c_int32), ("rstride", ctypes.c_int64), ("npeer", ctypes.c_int32),
                ("peer", ctypes.c_void_p * MAX_PEERS)]


def peer_map(peers, ld: int) -> TileMapC:
    """Row-cyclic map over the ranks' own grids: tile (i, j) at peers[i % P] + (i // P, j)."""
    m = TileMapC(None, ld, 0, len(peers), 0, len(peers))
    for r, p in enumerate(peers):
        m.peer[r] = p
    return m


class TileSetC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("i0", "i1", "j0", "j1", "lower", "row_off", "stride", "off")]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double

# symbol -> (restype, argtypes); every symbol declared in include/memdet_b200.h
SIGNATURES = {
    "b2d_version": (_I, []),
    "b2d_last_error": (ctypes.c_char_p, []),
    "b2d_device_count": (_I, []),
    "b2d_memdet_sym": (_I, [_P, _I64, _I64, _I, _I, _I64, _I64, ctypes.POINTER(ctypes.c_int), _I, _P, _P, _P,
                            _P, ctypes.POINTER(RunInfoC), ctypes.POINTER(_I64)]),
    "b2d_ctx_create": (_I, [_I, _I64, _I, ctypes.POINTER(_P)]),
    "b2d_ctx_create_ex": (_I, [_I, _I64, _I, ctypes.POINTER(OptionsC), ctypes.POINTER(_P)]),
    "b2d_ctx_is_out_of_core": (_I, [_P]),
    "b2d_ctx_destroy": (_I, [_P]),
    "b2d_ctx_factor_device_async": (_I, [_P, _P, _I64, _I, _P]),
    "b2d_ctx_factor_host_async": (_I, [_P, _P, _I64, _I, _P]),
    "b2d_ctx_fetch": (_I, [_P, _P, _P, ctypes.POINTER(_I64), ctypes.POINTER(RunInfoC)]),
    "b2d_ctx_device_prefix": (_P, [_P]),
    "b2d_ctx_fetch_perm": (_I, [_P, _P]),
    "b2d_ctx_set_profiling": (_I, [_P, _I]),
    "b2d_ctx_update_stats": (_I, [_P, ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_I64)]),
    "b2d_gen_rbf": (_I, [_P, _I64, _I, _D, _D, _P, _P]),
    "b2d_ctx_packed_init": (_I, [_P, _D, _P]),
    "b2d_ctx_gram_accumulate": (_I, [_P, _P, _I64, _I64, _D, _P]),
    "b2d_ctx_factor_packed_async": (_I, [_P, _P]),
    "b2d_probe_fp64_peak": (_I, [_I, _D, ctypes.POINTER(_D)]),
    "b2d_tile_ldl_host": (_I, [_P, _I64, _I64, _I, _D, _P, _P, ctypes.POINTER(_I64), _I]),
    "b2d_tile_cholesky_host": (_I, [_P, _I64, _I64, _I, _P, ctypes.POINTER(_I64), _I]),
    "b2d_tile_solve_lower_host": (_I, [_P, _I64, _I64, _P, _I64, _I64, _I, _I, _I]),
    "b2d_tile_schur_update_host": (_I, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _I64, _I, _I]),
    "b2d_tile_potrf_inv": (_I, [_P, _P, _P, _P, _P, _I64, _I64, _P]),
    "b2d_tile_gemm": (_I, [_I, ctypes.POINTER(TileMapC), ctypes.POINTER(TileMapC),
                           ctypes.POINTER(TileMapC), _P, ctypes.POINTER(TileSetC), ctypes.c_int32,
                           ctypes.c_int32, ctypes.c_int32, _P]),
    "b2d_pack_tiles": (_I, [_P, _I64, _I, _I64, _I64, ctypes.POINTER(TileMapC),
                            ctypes.POINTER(TileSetC), _P]),
    "b2d_prefix_scan": (_I, [_P, _I64, _P, _P]),
    "b2d_h2d_2d": (_I, [_P, _I64, _P, _I64, _I64, _I64, _P]),
    "b2d_dev_alloc": (_I, [_I, _I64, ctypes.POINTER(_P)]),
    "b2d_dev_free": (_I, [_P]),
    "b2d_ipc_get_handle": (_I, [_P, _P]),
    "b2d_ipc_open_handle": (_I, [_I, _P, ctypes.POINTER(_P)]),
    "b2d_ipc_close_handle": (_I, [_P]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load (once) and bind every exported symbol; raise loudly if the engine is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise errors.EngineUnavailableError(
                f"native engine not built: {path} is missing (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def probe_fp64_peak(device: int = 0, seconds: float = 0.3) -> float:
    out = ctypes.c_double()
    check(load().b2d_probe_fp64_peak(device, seconds, ctypes.byref(out)), "probe_fp64_peak")
    return out.value


def last_error() -> str:
    return (load().b2d_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "engine call", fail_index: int | None = None):
    """Map a C return code to the reference exception classes (errors.py:8-51)."""
    if rc == B2D_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == B2D_ERR_NOT_SPD:
        raise errors.NotSpdError(f"matrix is not positive-definite: {msg}")
    if rc == B2D_ERR_INDEFINITE:
        raise errors.IndefiniteBlockError(msg)
    if rc == B2D_ERR_USAGE:
        raise ValueError(msg)
    if rc == B2D_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == B2D_ERR_NOMEM:
        raise MemoryError(msg)
    if rc == B2D_ERR_STORAGE:
        raise errors.StorageError(msg)
    if rc == B2D_ERR_CUDA and "no CUDA device" in msg:
        raise errors.EngineUnavailableError(msg)
    raise RuntimeError(msg)


class Context:
    """Owning wrapper of a b2d_ctx (HBM workspace for one matrix order)."""

    def __init__(self, m: int, mode: int = MODE_CHOLESKY, device: int = 0, hbm_budget: int = 0,
                 num_blocks: int = 0, max_mem: int = 0, force_out_of_core: bool = False,
                 host_scratch: bool = False, emulation: bool = False, f32_arith: bool = False,
                 devices=None, scratch_dir: str | None = None, scratch_mode: int = 0):
        lib = load()
        h = ctypes.c_void_p()
        opt = OptionsC(int(hbm_budget or 0), int(num_blocks or 0), int(max_mem or 0),
                       int(bool(force_out_of_core)), int(bool(host_scratch)), int(bool(emulation)),
                       int(bool(f32_arith)))
        opt.scratch_mode = int(scratch_mode)
        self._scratch_dir = os.fsencode(scratch_dir) if scratch_dir else None  # kept alive with opt
        opt.scratch_dir = self._scratch_dir
        devices = tuple(int(x) for x in devices) if devices else ()
        if len(devices) > 8:
            raise ValueError(f"at most 8 devices, got {len(devices)}")
        if len(devices) > 1:
            opt.ndev = len(devices)
            for i, dv in enumerate(devices):
                opt.devices[i] = dv
            device = devices[0]
        check(lib.b2d_ctx_create_ex(device, m, mode, ctypes.byref(opt), ctypes.byref(h)),
              "b2d_ctx_create_ex")
        self._h = h
        self.m = m
        self.mode = mode
        self.device = device
        self.key = (device, m, mode, int(hbm_budget or 0), int(num_blocks or 0), int(max_mem or 0),
                    bool(force_out_of_core), bool(host_scratch), bool(emulation), bool(f32_arith), devices,
                    scratch_dir, int(scratch_mode))
        self.devices = devices or (device,)

    @property
    def scratch_on_device(self) -> bool:
        return bool(load().b2d_ctx_is_out_of_core(self._h) == 2)

    @property
    def out_of_core(self) -> bool:
        return bool(load().b2d_ctx_is_out_of_core(self._h))

    @property
    def handle(self):
        return self._h

    def factor_device_async(self, dev_ptr: int, lda: int, dtype_code: int, stream: int = 0):
        check(load().b2d_ctx_factor_device_async(self._h, ctypes.c_void_p(dev_ptr), lda, dtype_code,
                                                   ctypes.c_void_p(stream)), "factor_device")

    def factor_host_async(self, host_ptr: int, lda: int, dtype_code: int, stream: int = 0):
        check(load().b2d_ctx_factor_host_async(self._h, ctypes.c_void_p(host_ptr), lda, dtype_code,
                                                 ctypes.c_void_p(stream)), "factor_host")

    def fetch(self, d_out=None, prefix_out=None):
        """Wait, then copy outputs (NumPy float64 arrays or None); returns (rc, fail, info)."""
        fail = ctypes.c_int64(-1)
        info = RunInfoC()
        rc = load().b2d_ctx_fetch(self._h, None if d_out is None else d_out.ctypes.data,
                                  None if prefix_out is None else prefix_out.ctypes.data,
                                  ctypes.byref(fail), ctypes.byref(info))
        return rc, fail.value, info

    def fetch_perm(self, perm_out):
        check(load().b2d_ctx_fetch_perm(self._h, perm_out.ctypes.data), "fetch_perm")

    def device_prefix_ptr(self) -> int:
        return load().b2d_ctx_device_prefix(self._h)

    def set_profiling(self, mode: int):
        """0 off; events on the trailing rest-update launches: 1 in a normal run, 2 in a
        serialised replay (b2d_ctx_set_profiling)."""
        check(load().b2d_ctx_set_profiling(self._h, int(mode)))

    def update_stats(self):
        f, ms, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        check(load().b2d_ctx_update_stats(self._h, ctypes.byref(f), ctypes.byref(ms), ctypes.byref(n)),
              "update_stats")
        return f.value, ms.value, n.value

    def close(self):
        if self._h:
            load().b2d_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
