"""memdet_ldl on one reference block larger than the cluster panel's smem limit (16 x 384 rows):
the one-CTA panel path (or the big-block cluster path), device-resident RBF input."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import _native, gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 19661
lib = _native.load()
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(lib.b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
torch.cuda.synchronize()
for name, fn in (("ldl", eng.memdet_ldl), ("cholesky", eng.memdet_cholesky)):
    fn(a, num_blocks=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn(a, num_blocks=1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{os.environ.get('TAG','')} n={n} {name} one block: {dt*1e3:.1f} ms logdet {r.logabsdet:.12e}", flush=True)
