"""The reference's block walk (forced out of core) vs in core, n = 32768, 8 blocks: generic LU,
pivoted LDL and Cholesky from pinned host memory."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
g = torch.Generator(device="cuda"); g.manual_seed(0)
a = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
gen_m = a + 2.0 * n ** 0.5 * torch.eye(n, device="cuda", dtype=torch.float64)
sym = torch.tril(a) + torch.tril(a, -1).T
sym.diagonal().add_(torch.where(torch.rand(n, device="cuda", generator=g) < 0.5, -4.0, 4.0) * n ** 0.5)
del a
for name, f, mat in (("lu", eng.memdet_lu, gen_m), ("ldl", eng.memdet_ldl, sym)):
    h = torch.empty((n, n), dtype=torch.float64, pin_memory=True); h.copy_(mat); hn = h.numpy()
    for ooc in (False, True):
        f(hn, num_blocks=8, out_of_core=ooc)
        t0 = time.perf_counter(); r = f(hn, num_blocks=8, out_of_core=ooc); dt = time.perf_counter() - t0
        print(f"{name} n={n} out_of_core={ooc}: {dt*1e3:.1f} ms logabsdet={r.logabsdet:.12e}", flush=True)
        eng.release_engine_cache()
    del h, hn
