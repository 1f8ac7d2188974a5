"""One factorisation of the C2 matrix (or --n) through the engine's device path; for ncu."""
import argparse, ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_04424_b200 import _native, gen

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--host", action="store_true", help="pinned host input (e2e path)")
args = ap.parse_args()
n = args.n
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
torch.cuda.synchronize()
ctx = _native.Context(n)
pre = np.empty(n)
if args.host:
    h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    h.copy_(a)
    del a
    torch.cuda.empty_cache()
for s in range(args.steps):
    t0 = time.perf_counter()
    if args.host:
        ctx.factor_host_async(h.data_ptr(), n, _native.B2D_F64, 0)
    else:
        ctx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, 0)
    rc, fail, info = ctx.fetch(None, pre)
    _native.check(rc)
    dt = time.perf_counter() - t0
    print(f"n={n} step={s} {dt*1e3:.1f} ms  {n**3/3/dt/1e12:.2f} TF/s device_ms={info.device_ms:.1f} launches={info.kernel_launches} logdet={pre[-1]:.10e}", flush=True)
