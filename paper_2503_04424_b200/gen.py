"""Seeded synthetic inputs for the BASELINE.json configs (host side, NumPy).

These stand in for the paper's NTK / kernel Gram matrices, which are not available offline
(BASELINE.md §2).  Every generator returns a bit-symmetric row-major float64 matrix — the
MEMDET01 contract for `symmetric` / `spd` files (reference `storage.py:15-17`), enforced by
mirroring the lower triangle as the reference's own generator does (`kernelgen.py:136-149`).

Large instances (C2 and up) are generated on the device by the native library
(`b2d_gen_rbf`); the host versions here are for tests, fixtures and the CPU oracle.
"""

from __future__ import annotations

import numpy as np


def _mirror_lower(a: np.ndarray) -> np.ndarray:
    """Make `a` bit-symmetric by copying the strict lower triangle onto the upper (in row
    blocks, so no index arrays of the matrix's size)."""
    n, step = a.shape[0], 1024
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        blk = a[r0:r1, r0:r1]
        iu = np.triu_indices(r1 - r0, 1)
        blk[iu] = blk.T[iu]
        a[r0:r1, r1:] = a[r1:, r0:r1].T
    return a


def spd_wishart(n: int, k: int, seed: int = 0, shift: float = 1e-3, scale: float | None = None,
                dtype=np.float64) -> np.ndarray:
    """C1 / C4: A = G G^T / scale + shift I, G an n x k i.i.d. N(0,1) matrix (rows nested in n)."""
    g = np.random.default_rng(seed).standard_normal((n, k))
    a = g @ g.T
    a /= float(k if scale is None else scale)
    a[np.diag_indices(n)] += shift
    return _mirror_lower(a).astype(dtype, copy=False)


def rbf_points(n: int, d: int = 16, seed: int = 0) -> np.ndarray:
    """C2 inputs: x_i in R^d i.i.d. N(0,1), drawn row by row (nested in n)."""
    return np.random.default_rng(seed).standard_normal((n, d))


def rbf(n: int, d: int = 16, ell: float = 4.0, jitter: float = 1e-6, seed: int = 0,
        x: np.ndarray | None = None, threads: int = 1) -> np.ndarray:
    """C2: K_ij = exp(-||x_i - x_j||^2 / (2 ell^2)) + jitter * delta_ij.

    The squared distance is summed over coordinates in index order from exact differences,
    which is the order the device generator (`b2d_gen_rbf`) uses, so K is bit-symmetric and
    close to the device bytes (exp may differ in the last ulp).  `threads` > 1 computes the
    1024-row chunks concurrently (NumPy releases the GIL): the bytes do not change.
    """
    if x is None:
        x = rbf_points(n, d, seed)
    out = np.empty((n, n))
    inv = 1.0 / (2.0 * ell * ell)
    step = 1024

    def chunk(r0):
        r1 = min(n, r0 + step)
        sq = np.zeros((r1 - r0, n))
        for c in range(x.shape[1]):
            diff = x[r0:r1, c][:, None] - x[None, :, c]
            sq += diff * diff
        out[r0:r1] = np.exp(-sq * inv)

    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(chunk, range(0, n, step)))
    else:
        for r0 in range(0, n, step):
            chunk(r0)
    out[np.diag_indices(n)] += jitter
    return _mirror_lower(out)


def ntk_like(n: int, p: int, alpha: float, jitter: float = 1e-8, seed: int = 0) -> np.ndarray:
    """C3 / C5 (small host version): K = Z diag(s)^2 Z^T / p + jitter I, s_j = j^-alpha."""
    z = np.random.default_rng(seed).standard_normal((n, p))
    s = np.arange(1, p + 1, dtype=np.float64) ** (-alpha)
    j = z * s[None, :]
    a = j @ j.T / p
    a[np.diag_indices(n)] += jitter
    return _mirror_lower(a)


def random_symmetric(n: int, seed: int = 0, diag_shift: float = 4.0) -> np.ndarray:
    """Symmetric indefinite matrix with a boosted mixed-sign diagonal (1x1 pivoting stays
    well defined); the same construction as the reference fixture (tests/conftest.py:18-29)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    a = np.tril(g) + np.tril(g, -1).T
    signs = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    a[np.diag_indices(n)] += diag_shift * signs
    return a


def random_spd(n: int, seed: int = 0, shift: float = 1.0) -> np.ndarray:
    """G G^T / n + shift I, symmetrised from the lower triangle (tests/conftest.py:32-35)."""
    g = np.random.default_rng(seed).standard_normal((n, n))
    a = g @ g.T / n + shift * np.eye(n)
    return np.tril(a) + np.tril(a, -1).T


CONFIGS = {
    # BASELINE.json configs; tiling (`num_blocks`) is the reference's, the engine's own
    # internal tile is independent of it for the unpivoted path.
    "C1": dict(n=4096, num_blocks=4, kind="wishart", k=4096, shift=1e-3, tol=1e-10),
    "C2": dict(n=32768, num_blocks=8, kind="rbf", d=16, ell=4.0, jitter=1e-6, tol=1e-10),
    "C3": dict(n=65536, num_blocks=16, kind="ntk", p=131072, alpha=0.75, jitter=1e-8, tol=1e-6),
    "C4": dict(n=131072, num_blocks=128, kind="wishart", k=131072, shift=1e-4, tol=1e-10),
    "C5": dict(n=196608, num_blocks=5, kind="ntk", p=262144, alpha=1.0, jitter=1e-8, tol=1e-6),
}


def ntk_like_device(n: int, p: int, alpha: float, jitter: float = 1e-8, seed: int = 0,
                    chunk: int = 8192, device: str = "cuda"):
    """C3 / C5 on the device: K = Z diag(s)^2 Z^T / p + jitter I, s_j = j^-alpha, with Z drawn
    chunk by chunk of columns from torch's counter-based (Philox) CUDA generator and the rank-k
    updates done by cuBLAS (input formation is off the timed path).  Returns a bit-symmetric
    row-major CUDA tensor."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    k = torch.zeros((n, n), dtype=torch.float64, device=device)
    for c0 in range(0, p, chunk):
        c1 = min(p, c0 + chunk)
        z = torch.randn((n, c1 - c0), dtype=torch.float64, device=device, generator=g)
        s = torch.arange(c0 + 1, c1 + 1, dtype=torch.float64, device=device).pow_(-alpha)
        z.mul_(s)
        k.addmm_(z, z.T)
        del z
    k.div_(p)
    k.diagonal().add_(jitter)
    # bit-symmetric: mirror the lower triangle onto the upper (kernelgen.py:136-149 precedent),
    # block column by block column so no n x n temporary is needed
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        blk = k[c0:c1, c0:c1]
        blk.copy_(torch.tril(blk) + torch.tril(blk, -1).T)
        if c1 < n:
            k[c0:c1, c1:].copy_(k[c1:, c0:c1].T)
    return k


def gram_into_context(ctx, n: int, k: int, scale: float, jitter: float, seed: int = 0, chunk: int = 8192,
                      col_scale=None):
    """Form K = scale * G diag(col_scale)^2 G^T + jitter I directly in an in-core engine
    context's packed tiles (G: n x k i.i.d. N(0,1) from torch's Philox CUDA generator, drawn
    chunk by chunk of columns; the rank-k updates run on the engine's DMMA Schur kernel).
    C4: col_scale=None, scale=1/n; C3/C5: col_scale(j) = j^-alpha, scale = 1/p."""
    import ctypes

    import torch

    from . import _native

    lib = _native.load()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native.check(lib.b2d_ctx_packed_init(ctx.handle, jitter, stream), "packed_init")
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    for c0 in range(0, k, chunk):
        c1 = min(k, c0 + chunk)
        z = torch.randn((n, c1 - c0), dtype=torch.float64, device="cuda", generator=g)
        if col_scale is not None:
            z.mul_(col_scale(torch.arange(c0 + 1, c1 + 1, dtype=torch.float64, device="cuda")))
        _native.check(lib.b2d_ctx_gram_accumulate(ctx.handle, ctypes.c_void_p(z.data_ptr()), c1 - c0, c1 - c0,
                                                  scale, stream), "gram_accumulate")
        torch.cuda.current_stream().synchronize()  # z is freed next iteration
        del z


# Full-size parity configs (BASELINE.json configs[2..4]) formed on the device.  C3 is configs[2]
# itself; "C4L" is C4's leading 65536 x 65536 principal block (rows of C4's own G, so its prefixes
# are C4's leading prefixes); "C5S" is C5's recipe at half the order (n = 98304, the reference's
# n_b = 5 with a ragged tail at a 16 GB budget, as C5 at 64 GB), which fits one GPU box's host.
BIG_CONFIGS = {
    "C3": dict(n=65536, num_blocks=16, kind="ntk", p=131072, alpha=0.75, jitter=1e-8, tol=1e-6),
    "C4L": dict(n=65536, num_blocks=64, kind="wishart_lead", n_full=131072, shift=1e-4, tol=1e-10),
    "C5S": dict(n=98304, num_blocks=5, kind="ntk", p=262144, alpha=1.0, jitter=1e-8, tol=1e-6),
}


def wishart_lead_device(lead: int, n: int, shift: float, seed: int = 0, chunk: int = 8192):
    """Leading lead x lead block of A = G G^T / n + shift I, G n x n i.i.d. N(0,1) drawn chunk by
    chunk of columns from torch's Philox CUDA generator (the same stream as C4's full G,
    tools/c4_run.py), rank-k updates by cuBLAS; bit-symmetric row-major CUDA tensor."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    k = torch.zeros((lead, lead), dtype=torch.float64, device="cuda")
    for c0 in range(0, n, chunk):
        z = torch.randn((n, min(n, c0 + chunk) - c0), dtype=torch.float64, device="cuda", generator=g)
        zl = z[:lead]
        k.addmm_(zl, zl.T)
        del z, zl
    k.div_(n)
    k.diagonal().add_(shift)
    for c0 in range(0, lead, chunk):
        c1 = min(lead, c0 + chunk)
        blk = k[c0:c1, c0:c1]
        blk.copy_(torch.tril(blk) + torch.tril(blk, -1).T)
        if c1 < lead:
            k[c0:c1, c1:].copy_(k[c1:, c0:c1].T)
    return k


def big_config_device(name: str):
    """The CUDA tensor of BIG_CONFIGS[name] (deterministic: same bytes on every B200 with this
    image; the parity tests check the SHA-256 against the golden's)."""
    c = BIG_CONFIGS[name]
    if c["kind"] == "ntk":
        return ntk_like_device(c["n"], c["p"], c["alpha"], c["jitter"], seed=0)
    return wishart_lead_device(c["n"], c["n_full"], c["shift"], seed=0)


def sha_rows(a: np.ndarray, rows: int = 1024, threads: int = 0) -> str:
    """SHA-256 over the SHA-256 digests of consecutive `rows`-row chunks of a host matrix (a
    checksum of checksums, hashed in parallel: hashlib releases the GIL on large buffers)."""
    import hashlib
    import os
    from concurrent.futures import ThreadPoolExecutor

    def one(r0):
        return hashlib.sha256(np.ascontiguousarray(a[r0:r0 + rows]).data).digest()

    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        digests = list(ex.map(one, range(0, a.shape[0], rows)))
    return hashlib.sha256(b"".join(digests)).hexdigest()
