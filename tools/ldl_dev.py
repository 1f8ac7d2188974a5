"""memdet_ldl (block-pivoted) on a device-resident C2 / C3 matrix: CUDA-event time per call."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import _native, gen
ap = argparse.ArgumentParser(); ap.add_argument("--cfg", default="C2"); ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--chol", action="store_true")
args = ap.parse_args()
if args.cfg == "C2":
    n, nb = 32768, 8
    x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
    a = torch.empty((n, n), dtype=torch.float64, device="cuda")
    _native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
else:
    a = gen.big_config_device(args.cfg); n = a.shape[0]; nb = gen.BIG_CONFIGS[args.cfg]["num_blocks"]
torch.cuda.synchronize()
fn = eng.memdet_cholesky if args.chol else eng.memdet_ldl
fn(a, num_blocks=nb)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(args.steps):
    e0.record(); r = fn(a, num_blocks=nb); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
print(f"{args.cfg} {'chol' if args.chol else 'ldl'} env={[k + '=' + v for k, v in os.environ.items() if k.startswith('B2D_')]}: "
      f"{ms:.1f} ms {n**3/3/ms/1e9:.2f} TF/s logdet={r.logabsdet:.12e}", flush=True)
