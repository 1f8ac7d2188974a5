import sys, numpy as np, torch, ctypes
sys.path.insert(0, '.')
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import gen, _native
n = 32768
x = torch.from_numpy(gen.rbf_points(n, 16, seed=0)).cuda()
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
_native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(x.data_ptr()), n, 16, 4.0, 1e-6, ctypes.c_void_p(a.data_ptr()), None))
torch.cuda.synchronize()
print(torch.cuda.mem_get_info())
for devs in ([0, 0], [0, 0, 0]):
    try:
        r = eng.memdet_ldl(a, num_blocks=8, devices=devs)
        print(devs, r.logabsdet, r.info.device_ms)
    except Exception as e:
        print(devs, "ERR", e)
    eng.release_engine_cache()
    print(torch.cuda.mem_get_info())
