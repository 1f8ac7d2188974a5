import numpy as np, time, os, sys, torch
from concurrent.futures import ThreadPoolExecutor
n = 32768
path = "/dev/shm/probe.bin"
a = np.lib.format.open_memmap if False else None
mm = np.memmap(path, dtype=np.float64, mode="w+", shape=(n, n))
for r0 in range(0, n, 2048):
    mm[r0:r0+2048] = 1.0
mm.flush(); del mm
buf = torch.empty(64 << 17, dtype=torch.float64, pin_memory=True).numpy()  # 64 MB
anon = np.ones((n, n))
def run(src, threads, label):
    rows_per = 64 << 17 // n  # rows per 64 MB
    t0 = time.perf_counter()
    def job(r0):
        # copy 128-row strip (upper triangle) into a private slice of the pinned buffer
        r1 = min(n, r0 + 128)
        for r in range(r0, r1):
            w = n - r
            off = ((r // 128) % 8) * 128 * 0  # reuse
            buf[:w] = src[r, r:]
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(0, n, 128)))
    dt = time.perf_counter() - t0
    print(f"{label} threads={threads}: {dt*1e3:.0f} ms {n*n*4/dt/1e9:.1f} GB/s", flush=True)
for th in (1, 8, 16):
    mm = np.memmap(path, dtype=np.float64, mode="r", shape=(n, n))
    run(mm, th, "mmap first touch")
    run(mm, th, "mmap second pass")
    del mm
run(anon, 16, "anonymous")
os.remove(path)
