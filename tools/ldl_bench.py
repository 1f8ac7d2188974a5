"""memdet_ldl (block-pivoted) timing on an RBF Gram (C2 family)."""
import argparse, ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import _native, gen
ap = argparse.ArgumentParser(); ap.add_argument("--n", type=int, default=32768); ap.add_argument("--nb", type=int, default=8)
ap.add_argument("--steps", type=int, default=2)
args = ap.parse_args(); n = args.n
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
h = torch.empty((n, n), dtype=torch.float64, pin_memory=True); h.copy_(a); del a; torch.cuda.empty_cache()
hn = h.numpy()
for s in range(args.steps):
    t0 = time.perf_counter(); r = eng.memdet_ldl(hn, num_blocks=args.nb); dt = time.perf_counter() - t0
    print(f"memdet_ldl block-pivoted n={n} nb={args.nb}: {dt*1e3:.1f} ms {n**3/3/dt/1e12:.2f} TF/s logdet={r.logabsdet:.12e} "
          f"perm!=id {int(np.sum(r.perm != np.arange(n)))} device_ms={r.info.device_ms:.1f} reads={r.info.ooc_reads}", flush=True)
t0 = time.perf_counter(); c = eng.memdet_cholesky(hn, num_blocks=args.nb); dt = time.perf_counter() - t0
print(f"memdet_cholesky n={n}: {dt*1e3:.1f} ms logdet={c.logabsdet:.12e}; block-boundary prefix max rel diff "
      f"{np.max(np.abs(c.prefix[r.info.b-1::r.info.b] - r.prefix[r.info.b-1::r.info.b]) / np.maximum(1, np.abs(c.prefix[r.info.b-1::r.info.b]))):.2e}")
