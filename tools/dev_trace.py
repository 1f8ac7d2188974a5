"""C2 memdet_cholesky from a device tensor with the per-step trace (B2D_TRACE), for comparison with
tools/e2e_trace.py."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import _native, gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
lib = _native.load()
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(lib.b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
torch.cuda.synchronize()
eng.memdet_cholesky(a, num_blocks=8)
os.environ["B2D_TRACE"] = "1"
eng.release_engine_cache()
eng.memdet_cholesky(a, num_blocks=8)
r = eng.memdet_cholesky(a, num_blocks=8)
print(f"device_ms {r.info.device_ms:.1f}")
