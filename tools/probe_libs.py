"""Library calibration (off the hot path): cuBLAS DGEMM and cuSOLVER DPOTRF rates on this B200."""
import time, torch
dev = "cuda"
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2): torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps): torch.matmul(a, b)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS DGEMM n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)", flush=True)
for n in (4096, 16384, 32768):
    g = torch.randn(n, 64, dtype=torch.float64, device=dev)
    x = g @ g.T / 64 + torch.eye(n, dtype=torch.float64, device=dev)
    torch.linalg.cholesky(x); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L = torch.linalg.cholesky(x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"cuSOLVER DPOTRF n={n}: {n**3/3/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)", flush=True)
    del L, x, g
