"""Out-of-core cold (first call of a fresh context) vs warm times per scratchpad mode, on the C3
bytes (n = 65536, num_blocks = 4, 24 GB HBM budget) and optionally scaled C5 (--c5)."""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import gen

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
nb = 4 if name == "C3" else 5
budget = int(24e9)
a = gen.big_config_device(name)
n = a.shape[0]
host = np.empty((n, n))
cr = torch.cuda.cudart()
t0 = time.perf_counter()
cr.cudaHostRegister(host.ctypes.data, host.nbytes, 0)
print(f"{name}: host register {time.perf_counter() - t0:.1f} s", flush=True)
torch.from_numpy(host).copy_(a)
del a
torch.cuda.empty_cache()
flops = n ** 3 / 3
for mode in ("staged", "pinned", "file"):
    os.environ["B2D_SCRATCH"] = mode
    eng.release_engine_cache()
    kw = dict(num_blocks=nb, hbm_budget=budget, out_of_core=True)
    if mode == "file":
        kw["scratch_dir"] = "/tmp"
    t0 = time.perf_counter()
    r = eng.memdet_cholesky(host, **kw)
    cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    r2 = eng.memdet_cholesky(host, **kw)
    warm = time.perf_counter() - t0
    print(f"{name} mode={mode}: cold {cold:.2f} s ({flops / cold / 1e12:.1f} TF)  warm {warm:.2f} s "
          f"({flops / warm / 1e12:.1f} TF)  h2d {r2.info.h2d_bytes / 1e9:.1f} GB d2h {r2.info.d2h_bytes / 1e9:.1f} GB "
          f"equal={np.array_equal(r.prefix, r2.prefix)} logdet={r2.logabsdet:.12e}", flush=True)
eng.release_engine_cache()
