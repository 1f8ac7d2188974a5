"""Distributed driver at world size 1 (NCCL) on C2: per-GPU efficiency of the multi-GPU path."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2503_04424_b200 import _native, gen
from paper_2503_04424_b200.distributed import DistributedMemdet
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
x = torch.from_numpy(gen.rbf_points(n, 16, 0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
r = DistributedMemdet(n, None, 8, torch.device("cuda", 0))
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    p, f = r.run(a); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"distributed driver world=1 n={n}: {dt*1e3:.1f} ms {n**3/3/dt/1e12:.2f} TF/s logdet={float(p[-1]):.10e} launches={r.ops.launches}", flush=True)
dist.destroy_process_group()
