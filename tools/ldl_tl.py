"""C2 memdet_ldl (device-resident input, as bench.py's `ldl` line) with the per-launch panel /
bulk timeline (B2D_LDL_TL) and the per-stage trace (B2D_LDL_TRACE); prints a summary.
   python tools/ldl_tl.py [--n 32768] [--nb 8] [--out gpurun_out/ldl_tl.txt]
Extra environment (B2D_*) is passed through, so A/B switches can be compared in one call."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_04424_b200 import _native, gen

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--nb", type=int, default=8)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--out", default="gpurun_out/ldl_tl.txt")
ap.add_argument("--tag", default="")
args = ap.parse_args()
n = args.n
lib = _native.load()
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(lib.b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
torch.cuda.synchronize()
ctx = _native.Context(n, _native.MODE_LDL_PIV, 0, num_blocks=args.nb)
prefix = np.empty(n)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, s.cuda_stream)
_native.check(ctx.fetch(None, prefix)[0], "warm")
times = []
for _ in range(args.steps):
    e0.record(s)
    ctx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, s.cuda_stream)
    e1.record(s)
    _native.check(ctx.fetch(None, prefix)[0], "step")
    times.append(e0.elapsed_time(e1))
ms = float(np.median(times))
print(f"{args.tag} n={n} nb={args.nb} memdet_ldl device: median {ms:.1f} ms ({n**3/3/ms/1e9:.2f} TF/s) "
      f"steps {['%.1f' % t for t in times]} logdet {prefix[-1]:.12e}", flush=True)
# timeline run
if os.path.exists(args.out):
    os.remove(args.out)
os.environ["B2D_LDL_TL"] = args.out
os.environ["B2D_LDL_TRACE"] = "1"
ctx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, s.cuda_stream)
_native.check(ctx.fetch(None, prefix)[0], "tl")
del os.environ["B2D_LDL_TL"], os.environ["B2D_LDL_TRACE"]
ctx.close()
rows = np.loadtxt(args.out, comments="#").reshape(-1, 4)
t0 = rows[:, 2].min()
b = n // args.nb
print(f"{'stage':>5} {'span_ms':>8} {'panel_ms':>8} {'bulk_ms':>8} {'gap_p_ms':>8} {'gap_b_ms':>8}  (per stage sums)")
for k in range(args.nb):
    sel = (rows[:, 0] >= k * b) & (rows[:, 0] < (k + 1) * b)
    p = rows[sel & (rows[:, 1] == 0)]
    q = rows[sel & (rows[:, 1] == 1)]
    p = p[np.argsort(p[:, 0])]
    q = q[np.argsort(q[:, 0])]
    span = (max(p[:, 3].max(), q[:, 3].max() if len(q) else 0) - p[:, 2].min()) / 1e6
    pan = (p[:, 3] - p[:, 2]).sum() / 1e6
    blk = (q[:, 3] - q[:, 2]).sum() / 1e6
    # gaps: panel i start - bulk i-1 end; bulk i start - panel i end
    qe = {int(r[0]): r for r in q}
    gp = gb = 0.0
    for r in p:
        prev = qe.get(int(r[0]) - 32)
        if prev is not None:
            gp += (r[2] - prev[3]) / 1e6
        cur = qe.get(int(r[0]))
        if cur is not None:
            gb += (cur[2] - r[3]) / 1e6
    print(f"{k:5d} {span:8.2f} {pan:8.2f} {blk:8.2f} {gp:8.2f} {gb:8.2f}   start {(p[:, 2].min() - t0) / 1e6:8.2f} ms")
