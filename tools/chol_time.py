"""C2 memdet_cholesky step time (device-resident input, as bench.py's value), for A/B builds
(B2D_LIB_OVERRIDE) and switches."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_04424_b200 import _native, gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
lib = _native.load()
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(lib.b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
ctx = _native.Context(n, _native.MODE_CHOLESKY, 0, num_blocks=nb)
prefix = np.empty(n)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    ctx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, s.cuda_stream)
    ctx.fetch(None, prefix)
ts = []
for _ in range(5):
    e0.record(s)
    ctx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, s.cuda_stream)
    e1.record(s)
    ctx.fetch(None, prefix)
    ts.append(e0.elapsed_time(e1))
print(f"{os.environ.get('TAG','')} n={n} cholesky: median {np.median(ts):.1f} ms ({n**3/3/np.median(ts)/1e9:.2f} TF/s) {['%.1f' % t for t in ts]} logdet {prefix[-1]:.10e}")
