"""Benchmark: FP64 logdet TFLOP/s (n^3/3 flops per logdet) of the B200 MEMDET engine.

Headline workload (BASELINE.json configs[1], "C2"): n = 32768 RBF Gram, x_i in R^16 i.i.d.
N(0,1) (seed 0), l = 4, jitter 1e-6, reference tiling num_blocks = 8.  Synthetic (the paper's
NTK / kernel matrices are not available offline); generated on the device, untimed.

One step = one full logdet + all 32768 prefix log-determinants of that matrix:
  value : input row-major in HBM when the timed region starts; the step packs the upper tile
          triangle, factors, and scans the prefix (libmemdet_b200.so, CUDA events on the
          launching stream, barrier + synchronize around K steps, max over ranks).
  e2e   : the same metric through the public API memdet_cholesky(host pinned array,
          num_blocks=8): host->device copy of the upper triangle and device->host copy of the
          prefix and d are inside the timed region.
Beside it (same JSON line): memdet_ldl (block-pivoted, the north star's LDL^T) on C2; C3
(configs[2]: n = 65536 NTK-like, 16 blocks, formed on the device) for both drivers, device and
end to end from pinned host memory; the out-of-core walk on the C3 bytes, first (cold) and warm
calls, against max(compute, PCIe); the opt-in Ozaki line; a MEMDET01-file e2e line.
N > 1 (torchrun): C3 per step, factored across the N devices by the engine's multi-device
context (devices=[0..N-1]: 1-D block-cyclic outer panels, sharded ingest, panels over NVLink),
driven from rank 0 -> scaling "strong"; the other ranks hold their GPU for the launch contract
and join the barriers.

`--impl reference` times the reference's CPU path (oracle port of oocdet.memdet_cholesky: the
same SciPy LAPACK / NumPy BLAS calls, all host threads) on C2 itself (n = 32768, num_blocks = 8,
b = 4096): each step is stage 0 of its 8-stage walk (one 4096 potrf, 7 TRSMs, 28 GEMMs of
4096^3 -- the block shapes of every stage), rate = that stage's exact flops / its time.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

METRIC = "FP64 logdet TFLOP/s (n^3/3)"
UNIT = "TFLOP/s"
INT8_PEAK_TOPS = 4500.0  # nominal B200 dense int8 tensor throughput (TOPS), for the opt-in Ozaki line
C2 = dict(n=32768, num_blocks=8, d=16, ell=4.0, jitter=1e-6, seed=0)
OOC = dict(n=65536, num_blocks=4, hbm_budget=int(24e9))  # out-of-core line: C3-sized RBF, forced walk
PROFILE_SUMMARY = os.path.join(REPO, "profiles", "r02_gemm_update_ncu.json")


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------ clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------ CPU sample


def c2_host_matrix():
    """The C2 matrix on the host (NumPy, threaded; bit-identical to tests/golden/c2.json's input)."""
    from paper_2503_04424_b200 import gen

    return gen.rbf(C2["n"], C2["d"], C2["ell"], C2["jitter"], C2["seed"], threads=os.cpu_count() or 1)


def run_cpu_reference(a: np.ndarray, steps: int, warmup: int):
    """The reference's CPU path (oracle port of memdet_cholesky's walk, the same LAPACK / BLAS
    calls, all host threads) on C2 at full size: each step is stage 0 of the num_blocks = 8 walk
    (memdet.py:346-387, k = 0: the block shapes of every stage).  Returns (TFLOP/s, seconds per
    step, threads, stage flops)."""
    from oracle import memdet_oracle as O

    try:
        from threadpoolctl import threadpool_info, threadpool_limits

        threads = os.cpu_count()
        ctx = threadpool_limits(limits=threads)
        info = threadpool_info()
        threads = max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:  # pragma: no cover
        ctx = None
        threads = os.cpu_count()
    nb = C2["num_blocks"]
    flops = O.stage0_flops(a.shape[0], nb)
    for _ in range(warmup):
        O.run_stage0(a, nb)
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.run_stage0(a, nb)
        t.append(time.perf_counter() - t0)
    sec = float(np.mean(t))
    del ctx
    return flops / sec / 1e12, sec, threads, flops


def cpu_sample_text(sec, steps):
    return (f"oracle port of oocdet.memdet_cholesky (SciPy LAPACK potrf/trtrs + NumPy BLAS, as the reference "
            f"calls them) on C2 itself (n=32768, num_blocks=8, b=4096): stage 0 of the 8-stage walk per step "
            f"(1 potrf + 7 TRSM + 28 GEMM of 4096, incl. the block copies), rate = its exact flops / time; "
            f"mean of {steps} run(s), {sec:.2f} s each")


# ------------------------------------------------------------------------------ GPU arm


def generate_rbf_device(torch, dev_x, n):
    from paper_2503_04424_b200 import _native

    a = torch.empty((n, n), dtype=torch.float64, device=dev_x.device)
    _native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(dev_x.data_ptr()), n, C2["d"], C2["ell"],
                                             C2["jitter"], ctypes.c_void_p(a.data_ptr()),
                                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return a


def measure_int8_peak(torch, n=8192, reps=5):
    """Dense int8 tensor throughput for the opt-in Ozaki line's roofline: cuBLASLt's int8 GEMM
    (torch._int_mm, int8 x int8 -> int32) at n^3, best of `reps` by CUDA events (a library
    measurement of the denominator, as MEASURED_PEAKS.json's bf16 figure; not on the path)."""
    try:
        a = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda").t()
        torch._int_mm(a, b)
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del a, b
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12, f"measured: cuBLASLt int8 GEMM {n}^3, best of {reps}"
    except Exception as ex:  # noqa: BLE001
        return INT8_PEAK_TOPS, f"nominal (int8 GEMM probe failed: {type(ex).__name__})"


def measure_pcie(torch, nbytes=1 << 30, reps=3):
    """Pinned host <-> HBM copy rates (GB/s) for the out-of-core roofline."""
    h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    rates = []
    for src, dst in ((h, d), (d, h)):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        rates.append(reps * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del h, d
    return rates[0], rates[1]


def traffic_from_profile():
    try:
        with open(PROFILE_SUMMARY) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def pin_host(torch, arr: np.ndarray):
    """Page-lock an existing host array in place (exact size; torch's pinned allocator would
    round 34 GB up to 64 GB).  Returns an unregister callback."""
    cr = torch.cuda.cudart()
    rc = cr.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister failed: {rc}")
    return lambda: cr.cudaHostUnregister(arr.ctypes.data)


def timed_calls(torch, stream, fn, steps):
    """CUDA-event time per call of a public-API call on a device tensor (the engine enqueues on
    the current stream and the call returns after its fetch)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        res = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, res


def run_c3(args, torch, eng, gen, peak, e0, e1, stream):
    cfg = gen.BIG_CONFIGS["C3"]
    n, nb = cfg["n"], cfg["num_blocks"]
    flops = n ** 3 / 3.0
    t0 = time.perf_counter()
    a = gen.big_config_device("C3")
    torch.cuda.synchronize()
    t_form = time.perf_counter() - t0
    steps = max(1, min(args.steps, 2))
    out = {"config": {"workload": "C3 (BASELINE.json configs[2])", "n": n, "num_blocks": nb,
                      "kind": f"NTK-like Z S^2 Z^T/p + 1e-8 I, p={cfg['p']}, s_j=j^-{cfg['alpha']}",
                      "formation_s_untimed": t_form},
           "steps": steps}
    prefixes = {}
    for name, fn in (("cholesky", eng.memdet_cholesky), ("ldl", eng.memdet_ldl)):
        fn(a, num_blocks=nb)  # warm (allocates the workspace)
        ms, res = timed_calls(torch, stream, lambda: fn(a, num_blocks=nb), steps)
        eng.release_engine_cache()
        prefixes[name] = res.prefix
        out[name] = {"value": flops / (ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ms,
                     "frac_of_fp64_peak": flops / (ms * 1e-3) / 1e12 / peak, "logdet": res.logabsdet,
                     "gpu_launches": int(res.info.kernel_launches),
                     "api": f"paper_2503_04424_b200.memdet_{name}(CUDA tensor, num_blocks={nb})"}
        if name == "ldl":
            out[name]["interchanged_rows"] = int(np.sum(res.perm != np.arange(n)))
    ks = np.array([2 ** k for k in range(int(np.log2(n)) + 1)]) - 1
    out["prefix_at_2k"] = {int(q + 1): float(prefixes["cholesky"][q]) for q in ks}
    host = np.empty((n, n))
    at = torch.from_numpy(host)
    unpin = pin_host(torch, host)
    at.copy_(a)
    del a
    torch.cuda.empty_cache()
    for name, fn in (("cholesky", eng.memdet_cholesky), ("ldl", eng.memdet_ldl)):
        fn(host, num_blocks=nb)  # warm
        t0 = time.perf_counter()
        for _ in range(steps):
            res = fn(host, num_blocks=nb)
        sec = (time.perf_counter() - t0) / steps
        eng.release_engine_cache()
        out[name]["e2e"] = {"value": flops / sec / 1e12, "unit": UNIT, "seconds_per_step": sec,
                            "h2d_bytes_per_step": int(res.info.h2d_bytes), "d2h_bytes_per_step": int(res.info.d2h_bytes),
                            "api": f"paper_2503_04424_b200.memdet_{name}(pinned host ndarray, num_blocks={nb})"}
    out["_host"] = (host, unpin)
    return out


def run_ooc_line(torch, eng, host_unpin, peak, h2d_gbs, d2h_gbs):
    host, unpin = host_unpin
    on = host.shape[0]
    oflops = on ** 3 / 3.0
    budget = OOC["hbm_budget"]
    nb = OOC["num_blocks"]
    eng.release_engine_cache()
    t0 = time.perf_counter()  # cold: a fresh context (pins its scratchpad) -- the one-shot case
    cold = eng.memdet_cholesky(host, num_blocks=nb, hbm_budget=budget, out_of_core=True)
    cold_sec = time.perf_counter() - t0
    steps = 2
    t0 = time.perf_counter()
    for _ in range(steps):
        res = eng.memdet_cholesky(host, num_blocks=nb, hbm_budget=budget, out_of_core=True)
    sec = (time.perf_counter() - t0) / steps
    eng.release_engine_cache()
    unpin()
    oi = res.info
    roof = max(oflops / (peak * 1e12), oi.h2d_bytes / (h2d_gbs * 1e9), oi.d2h_bytes / (d2h_gbs * 1e9))
    return {"value": oflops / sec / 1e12, "unit": UNIT, "seconds_per_step": sec, "steps": steps,
            "cold": {"value": oflops / cold_sec / 1e12, "seconds": cold_sec, "roofline_frac": roof / cold_sec,
                     "note": "first call of a fresh context: includes allocating / pinning the scratchpad"},
            "config": {"workload": "C3 bytes (configs[2], n=65536 NTK-like) through the reference's out-of-core "
                                   "tile walk", "n": on, "num_blocks": nb, "b": int(oi.b), "hbm_budget_bytes": budget,
                       "out_of_core": bool(oi.out_of_core), "scratchpad": "pinned host"},
            "blocks_read": int(oi.blocks_read), "blocks_written": int(oi.blocks_written),
            "scratch_slots": int(oi.scratch_slots), "engine_reads": int(oi.ooc_reads),
            "engine_writes": int(oi.ooc_writes),
            "h2d_bytes_per_step": int(oi.h2d_bytes), "d2h_bytes_per_step": int(oi.d2h_bytes),
            "roofline": {"bound": "max(FP64 tensor, PCIe H2D, PCIe D2H)", "time_s": roof, "frac": roof / sec,
                         "peak_tflops": peak, "h2d_gbs": h2d_gbs, "d2h_gbs": d2h_gbs,
                         "pcie_source": "pinned 1 GiB cudaMemcpy each way, this run"},
            "logdet": res.logabsdet, "cold_equals_warm": bool(np.array_equal(cold.prefix, res.prefix)),
            "api": f"paper_2503_04424_b200.memdet_cholesky(pinned host ndarray, num_blocks={nb}, "
                   f"hbm_budget=24e9, out_of_core=True)"}


def run_engine(args):
    import torch
    import torch.distributed as dist

    import paper_2503_04424_b200 as eng
    from paper_2503_04424_b200 import _native, gen

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = C2["n"]
    flops = n ** 3 / 3.0
    x = gen.rbf_points(n, C2["d"], C2["seed"])
    dev_x = torch.from_numpy(x).cuda()
    a = generate_rbf_device(torch, dev_x, n)
    torch.cuda.synchronize()

    peak = _native.probe_fp64_peak(local, 0.3)

    ctx = _native.Context(n, _native.MODE_CHOLESKY, local)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    prefix = np.empty(n)

    def step():
        ctx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, sptr)

    # warm-up (also validates): W untimed steps
    for _ in range(args.warmup):
        step()
        rc, fail, info = ctx.fetch(None, prefix)
        _native.check(rc, "warmup")
    launches_per_step = int(info.kernel_launches)

    # timed region: K steps, barrier + synchronize on both sides, CUDA events on the stream
    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms_total = e0.elapsed_time(e1)
    rc, fail, _ = ctx.fetch(None, prefix)
    _native.check(rc, "timed steps")
    logdet = float(prefix[-1])
    t = torch.tensor([ms_total], device="cuda")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = ws * flops * args.steps / (ms_max * 1e-3) / 1e12

    # dominant kernel (Schur-update GEMM), two extra untimed steps with CUDA events per launch:
    # the trailing rest updates (1) inside a normal step, sharing the GPU with the panel streams,
    # and (2) in a serialised replay, each launch timed alone (what ncu's launch list sees)
    ctx.set_profiling(1)
    step()
    rc, _, _ = ctx.fetch(None, None)
    _native.check(rc)
    step_flops, step_ms, step_launches = ctx.update_stats()
    ctx.set_profiling(2)
    step()
    rc, _, _ = ctx.fetch(None, None)
    _native.check(rc)
    upd_flops, upd_ms, upd_launches = ctx.update_stats()
    ctx.set_profiling(0)
    ctx.close()

    # opt-in variant beside the headline (never as it): the same steps with the trailing Schur
    # updates emulated on the int8 tcgen05 tensor cores (schur="ozaki", 8-slice Ozaki scheme)
    ozaki = None
    if not args.no_ozaki:
        octx = _native.Context(n, _native.MODE_CHOLESKY, local, emulation=True)
        oprefix = np.empty(n)

        def ostep():
            octx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, sptr)

        for _ in range(max(1, args.warmup)):
            ostep()
            rc, _, _ = octx.fetch(None, oprefix)
            _native.check(rc, "ozaki warmup")
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            ostep()
        e1.record(stream)
        barrier()
        oms = e0.elapsed_time(e1) / args.steps
        rc, _, _ = octx.fetch(None, oprefix)
        _native.check(rc, "ozaki steps")
        diff = float(np.max(np.abs(oprefix - prefix) / np.maximum(1.0, np.abs(prefix))))
        octx.set_profiling(2)
        ostep()
        rc, _, _ = octx.fetch(None, None)
        _native.check(rc)
        oz_flops, oz_ms, oz_launches = octx.update_stats()
        octx.close()
        int8_tops, int8_src = measure_int8_peak(torch)
        oz_peak = int8_tops / 36.0
        oz_ach = oz_flops / (oz_ms * 1e-3) / 1e12 if oz_ms > 0 else None
        ozaki = {"value": flops / (oms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": oms,
                 "max_prefix_rel_diff_vs_fp64_dmma": diff, "logdet": float(oprefix[-1]),
                 "schur": "trailing updates as FP64 emulated on int8 tcgen05 MMAs: 8 balanced signed slices per "
                          "row-scaled operand, the 36 slice products with s+t <= 9 accumulated exactly in int32 "
                          "TMEM, FP64 reconstruction (error ~3 u relative to sum |a b|)",
                 "roofline": {"bound": "tensor (int8)", "kernel": "oz_expo + oz_slice + oz_update (rest updates)",
                              "achieved": oz_ach, "peak": oz_peak, "unit": UNIT,
                              "frac": (oz_ach / oz_peak) if oz_ach else None,
                              "peak_source": f"dense int8 {int8_tops / 1e3:.2f} POPS ({int8_src}) / 36 slice "
                                             "products per FP64 multiply-add",
                              "launches": oz_launches, "kernel_ms": oz_ms}}

    # the second entry point of the path: memdet_ldl with the reference's block-local 1x1 pivoting
    # (num_blocks=8: b = 4096, bit-identical pivots), in core, device-resident input
    ldl = None
    if not args.no_ldl:
        lctx = _native.Context(n, _native.MODE_LDL_PIV, local, num_blocks=C2["num_blocks"])
        lprefix = np.empty(n)

        def lstep():
            lctx.factor_device_async(a.data_ptr(), n, _native.B2D_F64, sptr)

        for _ in range(max(1, args.warmup)):
            lstep()
            rc, _, linfo = lctx.fetch(None, lprefix)
            _native.check(rc, "ldl warmup")
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            lstep()
        e1.record(stream)
        barrier()
        lms = e0.elapsed_time(e1) / args.steps
        rc, _, linfo = lctx.fetch(None, lprefix)
        _native.check(rc, "ldl steps")
        lperm = np.empty(n, np.int64)
        lctx.fetch_perm(lperm)
        l_in_core = not lctx.out_of_core
        lctx.close()
        ldl = {"value": flops / (lms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": lms,
               "frac_of_fp64_peak": flops / (lms * 1e-3) / 1e12 / peak,
               "config": {"num_blocks": C2["num_blocks"], "pivoting": "block-local 1x1 (reference _ldl.pyx)",
                          "in_core": l_in_core},
               "logdet": float(lprefix[-1]), "logdet_rel_diff_vs_cholesky": abs(float(lprefix[-1]) - logdet) / abs(logdet),
               "interchanged_rows": int(np.sum(lperm != np.arange(n))),
               "gpu_launches": int(linfo.kernel_launches) * args.steps}

    # e2e through the public API from pinned host memory
    pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    pinned.copy_(a)
    del a
    torch.cuda.empty_cache()
    host = pinned.numpy()
    e2e_steps = max(1, min(args.steps, 3))
    res = eng.memdet_cholesky(host, num_blocks=C2["num_blocks"])  # warm (allocates the workspace)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = eng.memdet_cholesky(host, num_blocks=C2["num_blocks"])
    torch.cuda.synchronize()
    e2e_sec = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([e2e_sec], device="cuda")
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_sec = float(te.item())
    e2e_logdet = res.logabsdet
    h2d, d2h = res.info.h2d_bytes, res.info.d2h_bytes
    eng.release_engine_cache()
    if ozaki is not None:  # the opt-in line through the same public call
        eng.memdet_cholesky(host, num_blocks=C2["num_blocks"], schur="ozaki")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ores = eng.memdet_cholesky(host, num_blocks=C2["num_blocks"], schur="ozaki")
        osec = (time.perf_counter() - t0) / e2e_steps
        eng.release_engine_cache()
        ozaki["e2e"] = {"value": flops / osec / 1e12, "unit": UNIT, "seconds_per_step": osec, "steps": e2e_steps,
                        "api": "paper_2503_04424_b200.memdet_cholesky(pinned host ndarray, num_blocks=8, schur='ozaki')",
                        "logdet": ores.logabsdet}
    if ldl is not None:
        eng.memdet_ldl(host, num_blocks=C2["num_blocks"])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            lres = eng.memdet_ldl(host, num_blocks=C2["num_blocks"])
        lsec = (time.perf_counter() - t0) / e2e_steps
        eng.release_engine_cache()
        ldl["e2e"] = {"value": flops / lsec / 1e12, "unit": UNIT, "seconds_per_step": lsec, "steps": e2e_steps,
                      "h2d_bytes_per_step": int(lres.info.h2d_bytes), "d2h_bytes_per_step": int(lres.info.d2h_bytes),
                      "api": "paper_2503_04424_b200.memdet_ldl(pinned host ndarray, num_blocks=8)",
                      "logdet": lres.logabsdet}

    # e2e from a MEMDET01 file (the reference's own input form: memory-mapped, pageable; staged
    # through pinned buffers by host threads), on tmpfs when there is one
    e2e_file = None
    if not args.no_file:
        from paper_2503_04424_b200.storage import MatrixFile
        fdir = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
        fpath = os.path.join(fdir, f"b2d_bench_c2_{os.getpid()}.mdm")
        try:
            mm = MatrixFile.create(fpath, n, "f64", "spd").memmap("r+")
            for r0 in range(0, n, 2048):
                mm[r0:r0 + 2048] = host[r0:r0 + 2048]
            mm.flush()
            del mm
            eng.memdet_cholesky(fpath, num_blocks=C2["num_blocks"])  # warm
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                fres = eng.memdet_cholesky(fpath, num_blocks=C2["num_blocks"])
            fsec = (time.perf_counter() - t0) / e2e_steps
            eng.release_engine_cache()
            e2e_file = {"value": flops / fsec / 1e12, "unit": UNIT, "seconds_per_step": fsec, "steps": e2e_steps,
                        "h2d_bytes_per_step": int(fres.info.h2d_bytes), "d2h_bytes_per_step": int(fres.info.d2h_bytes),
                        "api": "paper_2503_04424_b200.memdet_cholesky('<file>.mdm', num_blocks=8) (MEMDET01 file "
                               f"on {fdir}, memory-mapped)", "logdet": fres.logabsdet}
        finally:
            if os.path.exists(fpath):
                os.remove(fpath)

    # CPU baseline: the reference's CPU path on C2 itself (stage 0 of its walk), rank 0, N = 1
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        v, sec, threads, _ = run_cpu_reference(host, 1, 0)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "same_config": True,
               "sample": cpu_sample_text(sec, 1)}

    # C3 (configs[2]): n = 65536 NTK-like Gram formed on the device; both drivers at 16 blocks,
    # device-resident and end to end from pinned host memory; then the out-of-core walk on the
    # same host bytes (num_blocks = 4 under a 24 GB HBM budget), first call (pins its scratchpad)
    # and warm, against max(compute, PCIe)
    c3 = None
    ooc = None
    if not args.no_c3:
        h2d_gbs, d2h_gbs = measure_pcie(torch)
        del pinned, host
        torch.cuda.empty_cache()
        c3 = run_c3(args, torch, eng, gen, peak, e0, e1, stream)
        if not args.no_ooc:
            ooc = run_ooc_line(torch, eng, c3.pop("_host"), peak, h2d_gbs, d2h_gbs)
        c3.pop("_host", None)

    out = None
    if rank == 0:
        prof = traffic_from_profile()
        achieved = upd_flops / (upd_ms * 1e-3) / 1e12 if upd_ms > 0 else None
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: C2 RBF Gram generated on device (seeded), not the paper's NTKs",
            "config": {"workload": "C2", "n": n, "num_blocks": C2["num_blocks"], "kind": "rbf d=16 l=4 jitter=1e-6",
                       "engine_tile": 128, "l2": "inputs (8.6 GB) larger than L2 (126 MB)",
                       "parallelism": "replicas" if ws > 1 else "single"},
            "matrices_per_s": ws * args.steps / (ms_max * 1e-3),
            "frac_of_fp64_peak": value / (ws * peak),
            "logdet": logdet,
            "roofline": {"bound": "tensor",
                         "kernel": "gemm_kernel<MODE_UPDATE>, trailing Schur-update ('rest') launches of a step (DMMA)",
                         "achieved": achieved, "peak": peak, "unit": UNIT,
                         "frac": (achieved / peak) if achieved else None,
                         "peak_source": "live DMMA m8n8k4 microbenchmark (b2d_probe_fp64_peak), this run; "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "achieved_note": "algorithmic flops of the rest-update launches of one step "
                                          "(2*128^2*K per off-diagonal tile, 128*129*K per diagonal tile) / "
                                          "their summed CUDA-event time in a serialised replay of the step "
                                          "(each launch alone on the GPU, as in ncu's launch list, but warm)",
                         "in_step": {"achieved": (step_flops / (step_ms * 1e-3) / 1e12) if step_ms > 0 else None,
                                     "launches": step_launches, "kernel_ms": step_ms,
                                     "note": "the trailing 'rest' launches inside a normal step: their event "
                                             "span includes the time they share the SMs with the "
                                             "higher-priority panel streams, so this understates the kernel"},
                         "launches": upd_launches, "algorithmic_flops": upd_flops,
                         "kernel_ms": upd_ms,
                         "traffic": prof.get("dram_bytes_per_launch") if prof else None,
                         "traffic_launch": {k: prof[k] for k in ("kernel", "grid", "K", "duration_ms",
                                                                 "algorithmic_flops", "algorithmic_bytes_min",
                                                                 "dram_bytes_read", "dram_bytes_write")}
                         if prof else None},
            "cpu_baseline": cpu,
            "e2e": {"value": flops / e2e_sec / 1e12 * ws, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "seconds_per_step": e2e_sec, "steps": e2e_steps,
                    "api": "paper_2503_04424_b200.memdet_cholesky(pinned host ndarray, num_blocks=8)",
                    "logdet": e2e_logdet},
            "gpu_launches": launches_per_step * args.steps,
            "ozaki": ozaki,
            "ldl": ldl,
            "e2e_file": e2e_file,
            "c3": c3,
            "out_of_core": ooc,
            "clocks": clocks.summary(),
        }
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_engine_multi(args):
    """N > 1: C3 (configs[2], the north star's multi-GPU config) per step, factored across the N
    devices by the engine's multi-device context (devices=[0..N-1]), driven from
    rank 0; the other ranks keep their GPU for the launch contract and join the barriers.
    Strong scaling on a fixed C3 logdet; timed with CUDA events on rank 0's stream, which the
    multi-device call joins after every device's work (so the time is the max over devices)."""
    import torch
    import torch.distributed as dist

    import paper_2503_04424_b200 as eng
    from paper_2503_04424_b200 import _native, gen

    ws, rank, local = dist_env()
    backend = os.environ.get("B2D_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    import datetime

    kw = dict(device_id=torch.device("cuda", local)) if backend == "nccl" else {}
    # the other ranks wait in a barrier while rank 0 forms the matrix and drives every device
    dist.init_process_group(backend, timeout=datetime.timedelta(minutes=60), **kw)
    out = None
    if rank == 0:
        devices = [d % torch.cuda.device_count() for d in range(ws)]
        which = os.environ.get("B2D_BENCH_CONFIG", "C3")
        cfg = gen.BIG_CONFIGS[which] if which in gen.BIG_CONFIGS else None
        n = cfg["n"] if cfg else int(os.environ.get("B2D_BENCH_N", C2["n"]))
        nb = cfg["num_blocks"] if cfg else C2["num_blocks"]
        flops = n ** 3 / 3.0
        if cfg:
            a = gen.big_config_device(which)
        else:
            a = generate_rbf_device(torch, torch.from_numpy(gen.rbf_points(n, C2["d"], C2["seed"])).cuda(), n)
        torch.cuda.synchronize()
        peak = _native.probe_fp64_peak(local, 0.3)
        stream = torch.cuda.current_stream()
        lines = {}
        with ClockSampler(local) as clocks:
            for name, fn in (("cholesky", eng.memdet_cholesky), ("ldl", eng.memdet_ldl)):
                for _ in range(args.warmup if name == "cholesky" else 1):
                    fn(a, num_blocks=nb, devices=devices)
                ms, res = timed_calls(torch, stream, lambda: fn(a, num_blocks=nb, devices=devices),
                                      args.steps if name == "cholesky" else max(1, min(args.steps, 2)))
                lines[name] = (ms, res)
        eng.release_engine_cache()
        ms, res = lines["cholesky"]
        value = flops / (ms * 1e-3) / 1e12
        lms, lres = lines["ldl"]
        # e2e: pinned host -> each device ingests its own panels -> prefix on the host
        host = np.empty((n, n))
        unpin = pin_host(torch, host)
        torch.from_numpy(host).copy_(a)
        del a
        torch.cuda.empty_cache()
        eng.memdet_cholesky(host, num_blocks=nb, devices=devices)
        e2e_steps = max(1, min(args.steps, 2))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            eres = eng.memdet_cholesky(host, num_blocks=nb, devices=devices)
        e2e_sec = (time.perf_counter() - t0) / e2e_steps
        eng.release_engine_cache()
        unpin()
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic: {which} formed on the device (seeded), not the paper's NTKs",
            "config": {"workload": which, "n": n, "num_blocks": nb, "engine_tile": 128,
                       "l2": "inputs larger than L2 (126 MB)",
                       "parallelism": f"1-D block-cyclic outer panels (16 tile-columns) over {ws} devices, "
                                      f"sharded ingest, panels copied over NVLink (multi-device context driven "
                                      f"from rank 0)", "devices": devices},
            "matrices_per_s": 1.0 / (ms * 1e-3),
            "frac_of_fp64_peak": value / (ws * peak),
            "logdet": res.logabsdet,
            "roofline": {"bound": "tensor", "kernel": "all engine kernels, whole step, every device",
                         "achieved": value / ws, "peak": peak, "unit": UNIT, "frac": value / ws / peak,
                         "peak_source": "live DMMA m8n8k4 microbenchmark (b2d_probe_fp64_peak), device 0",
                         "achieved_note": "per-GPU share of the step's n^3/3 flops / step time", "traffic": None},
            "ldl": {"value": flops / (lms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": lms, "logdet": lres.logabsdet,
                    "api": f"memdet_ldl(CUDA tensor, num_blocks={nb}, devices={devices})"},
            "cpu_baseline": None,
            "e2e": {"value": flops / e2e_sec / 1e12, "unit": UNIT, "h2d_bytes_per_step": int(eres.info.h2d_bytes),
                    "d2h_bytes_per_step": int(eres.info.d2h_bytes), "seconds_per_step": e2e_sec, "steps": e2e_steps,
                    "api": f"paper_2503_04424_b200.memdet_cholesky(pinned host ndarray, num_blocks={nb}, "
                           f"devices={devices})", "logdet": eres.logabsdet},
            "gpu_launches": int(res.info.kernel_launches) * args.steps,
            "clocks": clocks.summary(),
        }
    dist.barrier()
    dist.destroy_process_group()
    return out


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    t0 = time.perf_counter()
    a = c2_host_matrix()
    t_gen = time.perf_counter() - t0
    v, sec, threads, flops = run_cpu_reference(a, args.steps, args.warmup)
    cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "same_config": True,
           "sample": cpu_sample_text(sec, args.steps)}
    return {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: C2 RBF Gram (host NumPy, seeded; the bytes of tests/golden/c2.json)",
            "config": {"workload": "C2", "n": C2["n"], "num_blocks": C2["num_blocks"], "b": 4096,
                       "step": "stage 0 of the reference walk (same block shapes as every stage)",
                       "stage_flops": flops, "parallelism": "cpu", "generation_s_untimed": t_gen},
            "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ozaki", action="store_true", help="skip the opt-in int8-emulated Schur line")
    ap.add_argument("--no-ldl", action="store_true", help="skip the memdet_ldl (block-pivoted) line")
    ap.add_argument("--no-ooc", action="store_true", help="skip the out-of-core line")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 lines (and the out-of-core line)")
    ap.add_argument("--no-file", action="store_true", help="skip the MEMDET01-file e2e line")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        out = run_reference(args)
    elif dist_env()[0] > 1:
        out = run_engine_multi(args)
    else:
        out = run_engine(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
