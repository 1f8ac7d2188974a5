"""memdet_cholesky / memdet_ldl from a MEMDET01 file (the reference's own input form: the file is
memory-mapped, i.e. pageable host memory) vs from pinned host memory, C2 (n = 32768)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import _native, gen
from paper_2503_04424_b200.storage import MatrixFile

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
path = sys.argv[2] if len(sys.argv) > 2 else "/dev/shm/c2.mdm"
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
host.copy_(a)
del a
torch.cuda.empty_cache()
t0 = time.perf_counter()
mf = MatrixFile.create(path, n, "f64", "spd")
mm = mf.memmap("r+")
hn = host.numpy()
for r0 in range(0, n, 2048):
    mm[r0:r0 + 2048] = hn[r0:r0 + 2048]
mm.flush()
del mm
print(f"wrote {path} ({n*n*8/1e9:.1f} GB) in {time.perf_counter() - t0:.1f} s", flush=True)
for name, f in (("cholesky", eng.memdet_cholesky), ("ldl", eng.memdet_ldl)):
    for src, arg in (("pinned host", hn), ("MEMDET01 file", path)):
        for it in range(2):
            t0 = time.perf_counter()
            r = f(arg, num_blocks=8)
            dt = time.perf_counter() - t0
            print(f"memdet_{name} from {src}: {dt*1e3:.1f} ms {n**3/3/dt/1e12:.2f} TFLOP/s logdet={r.logabsdet:.12e}", flush=True)
        eng.release_engine_cache()
os.remove(path)
