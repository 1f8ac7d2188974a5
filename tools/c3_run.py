"""C3 (BASELINE.json configs[2]): n=65536 NTK-like Gram K = Z S^2 Z^T / p + 1e-8 I, p=131072,
s_j = j^-0.75, formed on the device; logdet + prefixes at n_k = 2^k through the engine, checked
against an independent GPU factorisation (cuSOLVER via torch, checker only) at 1e-6."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_04424_b200 as eng
from paper_2503_04424_b200 import gen

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--p", type=int, default=131072)
ap.add_argument("--alpha", type=float, default=0.75)
ap.add_argument("--nb", type=int, default=16)
ap.add_argument("--ldl", action="store_true")
args = ap.parse_args()
n = args.n
t0 = time.perf_counter()
a = gen.ntk_like_device(n, args.p, args.alpha, 1e-8, seed=0)
torch.cuda.synchronize()
print(f"formation: {time.perf_counter() - t0:.1f} s ({n*n*args.p/1e12:.1f} TFMA via cuBLAS)", flush=True)
for it in range(2):
    t0 = time.perf_counter()
    res = eng.memdet_cholesky(a, num_blocks=args.nb)
    dt = time.perf_counter() - t0
    print(f"engine memdet_cholesky C3 (device input): {dt*1e3:.1f} ms  {n**3/3/dt/1e12:.2f} TFLOP/s  logdet={res.logabsdet:.12e}", flush=True)
ks = [2 ** k for k in range(int(np.log2(n)) + 1)]
print("prefix at n_k=2^k:", {q: float(res.prefix[q - 1]) for q in ks}, flush=True)
eng.release_engine_cache()


def torch_block_cholesky_logdiag(a, blk=32768):
    # independent check (cuSOLVER potrf + cuBLAS trsm/gemm through torch, 2x2 blocks; torch's
    # potrf faults on > 2^31-element matrices, so the 65536 order is split)
    n = a.shape[0]
    out = []
    s = a[:blk, :blk].clone()
    l11 = torch.linalg.cholesky(s)
    out.append(torch.diagonal(l11).clone())
    if n > blk:
        l21 = torch.linalg.solve_triangular(l11, a[blk:, :blk].T.contiguous(), upper=False).T
        del l11, s
        s22 = a[blk:, blk:] - l21 @ l21.T
        del l21
        out.append(torch.diagonal(torch.linalg.cholesky(s22)).clone())
    return torch.cat(out)


dg = torch_block_cholesky_logdiag(a)
ref = torch.cumsum(2.0 * torch.log(dg), 0).cpu().numpy()
rel = np.abs(res.prefix - ref) / np.maximum(1, np.abs(ref))
print(f"vs cuSOLVER: max rel over all prefixes {rel.max():.3e}, at 2^k {rel[np.array(ks) - 1].max():.3e}", flush=True)
if args.ldl:
    # the 16x16-block pivoted LDL of configs[2]: device-resident input (in core, factored where
    # it lives), then end to end from pinned host memory (17 GB of the upper triangle over PCIe)
    def report(tag, r2, dt):
        b = r2.info.b
        bd = np.abs(r2.prefix[b - 1::b] - ref[b - 1::b]) / np.maximum(1, np.abs(ref[b - 1::b]))
        print(f"memdet_ldl block-pivoted C3 ({tag}): {dt*1e3:.1f} ms {n**3/3/dt/1e12:.2f} TFLOP/s "
              f"logdet={r2.logabsdet:.12e} block-boundary rel vs cholesky {bd.max():.3e} "
              f"perm!=id {int(np.sum(r2.perm != np.arange(n)))}", flush=True)
    for it in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r2 = eng.memdet_ldl(a, num_blocks=args.nb)
        report("device input", r2, time.perf_counter() - t0)
    eng.release_engine_cache()
    host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    host.copy_(a)
    del a
    torch.cuda.empty_cache()
    hn = host.numpy()
    for it in range(2):
        t0 = time.perf_counter()
        r2 = eng.memdet_ldl(hn, num_blocks=args.nb)
        report("pinned host input", r2, time.perf_counter() - t0)
