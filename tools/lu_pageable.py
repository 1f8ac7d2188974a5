"""memdet_lu at n = 32768 from pinned vs pageable host memory (in core)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
n = 32768
g = torch.Generator(device="cuda"); g.manual_seed(0)
a = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
a.diagonal().add_(2.0 * n ** 0.5)
h = torch.empty((n, n), dtype=torch.float64, pin_memory=True); h.copy_(a); del a
pinned = h.numpy(); pageable = np.array(pinned)
for name, x in (("pinned", pinned), ("pageable", pageable)):
    eng.memdet_lu(x, num_blocks=8)
    t0 = time.perf_counter(); r = eng.memdet_lu(x, num_blocks=8); dt = time.perf_counter() - t0
    print(f"memdet_lu from {name}: {dt*1e3:.1f} ms logabsdet={r.logabsdet:.12e}", flush=True)
