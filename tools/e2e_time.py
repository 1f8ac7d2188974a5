"""C2 memdet_cholesky (or memdet_ldl with FN=ldl) end to end from pinned host memory: median of 3
(after one warm call); env switches apply per process (tools/e2e_trace.py has the per-step trace).
   [FN=ldl] [NB=8] python tools/e2e_time.py [n]"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import _native, gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
lib = _native.load()
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(lib.b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
h.copy_(a)
del a
torch.cuda.empty_cache()
hn = h.numpy()
fn = eng.memdet_ldl if os.environ.get("FN", "cholesky") == "ldl" else eng.memdet_cholesky
nb = int(os.environ.get("NB", "8"))
fn(hn, num_blocks=nb)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    r = fn(hn, num_blocks=nb)
    ts.append(time.perf_counter() - t0)
dt = float(np.median(ts))
print(f"{os.environ.get('TAG', '')} e2e {dt*1e3:.1f} ms ({n**3/3/dt/1e12:.2f} TF/s) device_ms {r.info.device_ms:.1f}", flush=True)
