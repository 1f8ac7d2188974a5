"""Out-of-core throughput: an n x n RBF Gram in pinned host memory, factored (a) in-core from the
host and (b) out of core under an HBM budget that forces the reference tile walk."""
import argparse, ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_04424_b200 import _native, gen

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--nb", type=int, default=4)
ap.add_argument("--budget-gb", type=float, default=24.0)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--skip-incore", action="store_true")
args = ap.parse_args()
n = args.n
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
h.copy_(a); torch.cuda.synchronize()
del a; torch.cuda.empty_cache()
flops = n ** 3 / 3
pre_in = None
if not args.skip_incore:
    ctx = _native.Context(n)
    pre_in = np.empty(n)
    for s in range(args.steps):
        t0 = time.perf_counter(); ctx.factor_host_async(h.data_ptr(), n, 0, 0); rc, f, info = ctx.fetch(None, pre_in); _native.check(rc)
        dt = time.perf_counter() - t0
        print(f"in-core  n={n}: {dt*1e3:.1f} ms {flops/dt/1e12:.2f} TF/s h2d={info.h2d_bytes/1e9:.1f} GB", flush=True)
    ctx.close()
ctx = _native.Context(n, hbm_budget=int(args.budget_gb * 1e9), num_blocks=args.nb, force_out_of_core=True)
pre = np.empty(n)
for s in range(args.steps):
    t0 = time.perf_counter(); ctx.factor_host_async(h.data_ptr(), n, 0, 0); rc, f, info = ctx.fetch(None, pre); _native.check(rc)
    dt = time.perf_counter() - t0
    print(f"out-of-core n={n} blocks={info.ooc_blocks} b={info.ooc_block}: {dt*1e3:.1f} ms {flops/dt/1e12:.2f} TF/s "
          f"reads={info.ooc_reads} writes={info.ooc_writes} scratch={info.ooc_scratch} "
          f"h2d={info.h2d_bytes/1e9:.1f} GB d2h={info.d2h_bytes/1e9:.1f} GB", flush=True)
if pre_in is not None:
    print("max rel diff in-core vs ooc:", float(np.max(np.abs(pre - pre_in) / np.maximum(1, np.abs(pre_in)))))
