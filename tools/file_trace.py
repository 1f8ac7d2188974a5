"""Band arrival / step timeline (B2D_TRACE) for a MEMDET01-file input at C2."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import _native, gen
from paper_2503_04424_b200.storage import MatrixFile
n = 32768
path = "/dev/shm/c2t.mdm"
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
h = a.cpu().numpy(); del a
mf = MatrixFile.create(path, n, "f64", "spd"); mm = mf.memmap("r+"); mm[:] = h; mm.flush(); del mm, h
for it in range(3):
    t0 = time.perf_counter(); r = eng.memdet_cholesky(path, num_blocks=8); dt = time.perf_counter() - t0
    print(f"file run {it}: {dt*1e3:.1f} ms device_ms={r.info.device_ms:.1f}", file=sys.stderr, flush=True)
os.remove(path)
