"""Benchmark: FP64 logdet TFLOP/s (n^3/3 flops per logdet) of the B200 MEMDET engine.

Workload (BASELINE.json configs[1], "C2"): n = 32768 RBF Gram, x_i in R^16 i.i.d. N(0,1)
(seed 0), l = 4, jitter 1e-6, reference tiling num_blocks = 8.  Synthetic (the paper's
NTK / kernel matrices are not available offline); generated on the device, untimed.

One step = one full logdet + all 32768 prefix log-determinants of that matrix:
  value : input row-major in HBM when the timed region starts; the step packs the upper tile
          triangle, factors, and scans the prefix (libmemdet_b200.so, CUDA events on the
          launching stream, barrier + synchronize around K steps, max over ranks).
  e2e   : the same metric through the public API memdet_cholesky(host pinned array,
          num_blocks=8): host->device copy of the upper triangle and device->host copy of the
          prefix and d are inside the timed region.
N > 1 (torchrun): one C2 logdet per step factored across all ranks (distributed.py: row-cyclic
tile rows, NCCL panel collectives) -> scaling "strong", value = n^3/3 per step / max time.

`--impl reference` times the reference's CPU path (oracle port of oocdet.memdet_cholesky: the
same SciPy LAPACK / NumPy BLAS calls, all host threads) on a bounded sample of the workload.
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
SAMPLE_N = 16384  # CPU baseline sample: leading principal 16384 submatrix of C2, b = 4096
PROFILE_SUMMARY = os.path.join(REPO, "profiles", "r01_gemm_update_ncu.json")


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


def cpu_sample_matrix(torch=None, dev_x=None):
    """Leading SAMPLE_N principal submatrix of the C2 matrix (the generator is nested)."""
    from paper_2503_04424_b200 import gen

    if torch is not None and dev_x is not None:
        a = generate_rbf_device(torch, dev_x[:SAMPLE_N].contiguous(), SAMPLE_N)
        out = a.cpu().numpy()
        del a
        return out
    return gen.rbf(SAMPLE_N, C2["d"], C2["ell"], C2["jitter"], C2["seed"])


def run_cpu_reference(a: np.ndarray, steps: int, warmup: int):
    """The reference's CPU path (oracle port of memdet_cholesky, same LAPACK/BLAS calls) on
    the sample; returns (TFLOP/s, seconds per step, threads)."""
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
    nb = SAMPLE_N // 4096
    for _ in range(warmup):
        O.memdet_cholesky(a, nb)
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.memdet_cholesky(a, nb)
        t.append(time.perf_counter() - t0)
    sec = float(np.mean(t))
    return SAMPLE_N ** 3 / 3.0 / sec / 1e12, sec, threads


# ------------------------------------------------------------------------------ GPU arm


def generate_rbf_device(torch, dev_x, n):
    from paper_2503_04424_b200 import _native

    a = torch.empty((n, n), dtype=torch.float64, device=dev_x.device)
    _native.check(_native.load().b2d_gen_rbf(ctypes.c_void_p(dev_x.data_ptr()), n, C2["d"], C2["ell"],
                                             C2["jitter"], ctypes.c_void_p(a.data_ptr()),
                                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return a


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
        oz_peak = INT8_PEAK_TOPS / 36.0
        oz_ach = oz_flops / (oz_ms * 1e-3) / 1e12 if oz_ms > 0 else None
        ozaki = {"value": flops / (oms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": oms,
                 "max_prefix_rel_diff_vs_fp64_dmma": diff, "logdet": float(oprefix[-1]),
                 "schur": "trailing updates as FP64 emulated on int8 tcgen05 MMAs: 8 balanced signed slices per "
                          "row-scaled operand, the 36 slice products with s+t <= 9 accumulated exactly in int32 "
                          "TMEM, FP64 reconstruction (error ~3 u relative to sum |a b|)",
                 "roofline": {"bound": "tensor (int8)", "kernel": "oz_expo + oz_slice + oz_update (rest updates)",
                              "achieved": oz_ach, "peak": oz_peak, "unit": UNIT,
                              "frac": (oz_ach / oz_peak) if oz_ach else None,
                              "peak_source": f"nominal B200 dense int8 {INT8_PEAK_TOPS / 1e3:.1f} POPS / 36 slice "
                                             "products per FP64 multiply-add (not measured)",
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

    # out-of-core (the north star's configs[4] schedule): the reference's tile walk on a C3-sized
    # RBF Gram (n = 65536, 34 GB in pinned host memory; the C2 points extended, nested) with
    # num_blocks=4 (b = 16384) under a 24 GB HBM budget -- 6 block slots in HBM, the 17 GB
    # scratchpad in pinned host memory -- against its roofline max(flops/peak, H2D/PCIe, D2H/PCIe)
    ooc = None
    if not args.no_ooc:
        h2d_gbs, d2h_gbs = measure_pcie(torch)
        del pinned, host
        on = OOC["n"]
        oflops = on ** 3 / 3.0
        ox = torch.from_numpy(gen.rbf_points(on, C2["d"], C2["seed"])).cuda()
        oa = generate_rbf_device(torch, ox, on)
        ohost_t = torch.empty((on, on), dtype=torch.float64, pin_memory=True)
        ohost_t.copy_(oa)
        del oa, ox
        torch.cuda.empty_cache()
        ohost = ohost_t.numpy()
        budget = OOC["hbm_budget"]
        eng.memdet_cholesky(ohost, num_blocks=OOC["num_blocks"], hbm_budget=budget, out_of_core=True)  # warm: pins the scratchpad
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ores2 = eng.memdet_cholesky(ohost, num_blocks=OOC["num_blocks"], hbm_budget=budget, out_of_core=True)
        osec2 = (time.perf_counter() - t0) / e2e_steps
        eng.release_engine_cache()
        oi = ores2.info
        roof = max(oflops / (peak * 1e12), oi.h2d_bytes / (h2d_gbs * 1e9), oi.d2h_bytes / (d2h_gbs * 1e9))
        ooc = {"value": oflops / osec2 / 1e12, "unit": UNIT, "seconds_per_step": osec2, "steps": e2e_steps,
               "config": {"workload": "RBF Gram n=65536 (C3 size; C2's recipe and points, nested)",
                          "n": on, "num_blocks": OOC["num_blocks"], "b": int(oi.b), "hbm_budget_bytes": budget,
                          "out_of_core": bool(oi.out_of_core), "scratchpad": "pinned host"},
               "blocks_read": int(oi.blocks_read), "blocks_written": int(oi.blocks_written),
               "scratch_slots": int(oi.scratch_slots), "engine_reads": int(oi.ooc_reads),
               "engine_writes": int(oi.ooc_writes),
               "h2d_bytes_per_step": int(oi.h2d_bytes), "d2h_bytes_per_step": int(oi.d2h_bytes),
               "roofline": {"bound": "max(FP64 tensor, PCIe H2D, PCIe D2H)", "time_s": roof, "frac": roof / osec2,
                            "peak_tflops": peak, "h2d_gbs": h2d_gbs, "d2h_gbs": d2h_gbs,
                            "pcie_source": "pinned 1 GiB cudaMemcpy each way, this run"},
               "logdet": ores2.logabsdet,
               "nested_prefix_rel_diff_vs_c2": float(np.max(np.abs(ores2.prefix[:n] - res.prefix)
                                                            / np.maximum(1.0, np.abs(res.prefix)))),
               "api": "paper_2503_04424_b200.memdet_cholesky(pinned host ndarray, num_blocks=4, hbm_budget=24e9, out_of_core=True)"}

    out = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            sample = cpu_sample_matrix(torch, dev_x)
            v, sec, threads = run_cpu_reference(sample, 1, 0)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": f"oracle port of oocdet.memdet_cholesky on the leading {SAMPLE_N}^2 "
                             f"principal submatrix of C2 (num_blocks=4, b=4096 = C2's tile), one run, "
                             f"{sec:.2f} s"}
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
            "out_of_core": ooc,
            "clocks": clocks.summary(),
        }
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_engine_multi(args):
    """N > 1: one C2 logdet per step, factored across all ranks (row-cyclic tile rows; per panel
    an NCCL all-reduce of the diagonal block and a stream-ordered barrier, after which every
    rank's Schur-update kernels read the solved panel tiles in place from their owners' grids
    over NVLink peer memory) -> strong scaling."""
    import torch
    import torch.distributed as dist

    from paper_2503_04424_b200 import _native, gen
    from paper_2503_04424_b200.distributed import DistributedMemdet

    ws, rank, local = dist_env()
    # B2D_DIST_BACKEND=gloo lets a functional check run several ranks on one GPU (collectives
    # staged through host memory); the measured configuration is NCCL, one rank per GPU
    backend = os.environ.get("B2D_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    kw = dict(device_id=torch.device("cuda", local)) if backend == "nccl" else {}
    dist.init_process_group(backend, **kw)
    n = int(os.environ.get("B2D_BENCH_N", C2["n"]))
    flops = n ** 3 / 3.0
    dev_x = torch.from_numpy(gen.rbf_points(n, C2["d"], C2["seed"])).cuda()
    a = generate_rbf_device(torch, dev_x, n)
    torch.cuda.synchronize()
    peak = _native.probe_fp64_peak(local, 0.3)
    peer_env = os.environ.get("B2D_DIST_PEER")  # default: peer mode with NCCL, gather with gloo
    runner = DistributedMemdet(n, None, 8, torch.device("cuda", local),
                               peer=None if peer_env is None else peer_env == "1")
    for _ in range(args.warmup):
        prefix, fail = runner.run(a)
        if fail != -1:
            raise RuntimeError(f"not SPD at {fail}")
    torch.cuda.synchronize()
    launches0 = runner.ops.launches
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            prefix, fail = runner.run(a)
        e1.record(stream)
        dist.barrier()
        torch.cuda.synchronize()
    launches = (runner.ops.launches - launches0) // max(1, args.steps)
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    logdet = float(prefix[-1].item())
    value = flops * args.steps / (ms_max * 1e-3) / 1e12
    # e2e: pinned host matrix -> each rank's device copy -> distributed factorisation -> prefix
    pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    pinned.copy_(a)
    e2e_steps = max(1, min(args.steps, 3))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        a.copy_(pinned, non_blocking=True)
        prefix, fail = runner.run(a)
        host_prefix = prefix.cpu()
    torch.cuda.synchronize()
    te = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_sec = float(te.item())
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: C2 RBF Gram generated on device (seeded), not the paper's NTKs",
            "config": {"workload": "C2", "n": n, "num_blocks": C2["num_blocks"], "kind": "rbf d=16 l=4 jitter=1e-6",
                       "engine_tile": 128, "l2": "inputs (8.6 GB) larger than L2 (126 MB)",
                       "parallelism": f"row-cyclic tile rows x{ws}, " + (
                           f"panels read in place over NVLink peer memory (CUDA IPC) after a {backend} barrier"
                           if runner.shared is not None else f"{backend} panel all-gather")},
            "matrices_per_s": args.steps / (ms_max * 1e-3),
            "frac_of_fp64_peak": value / (ws * peak),
            "logdet": logdet,
            "roofline": {"bound": "tensor", "kernel": "all engine kernels, whole step",
                         "achieved": value / ws, "peak": peak, "unit": UNIT, "frac": value / ws / peak,
                         "peak_source": "live DMMA m8n8k4 microbenchmark (b2d_probe_fp64_peak), rank 0",
                         "achieved_note": "per-GPU share of the step's n^3/3 flops / step time", "traffic": None},
            "cpu_baseline": None,
            "e2e": {"value": flops / e2e_sec / 1e12, "unit": UNIT, "h2d_bytes_per_step": int(n * n * 8 * ws),
                    "d2h_bytes_per_step": int(n * 8), "seconds_per_step": e2e_sec, "steps": e2e_steps,
                    "api": "paper_2503_04424_b200.distributed.DistributedMemdet.run after a pinned H2D copy per rank",
                    "logdet": float(host_prefix[-1])},
            "gpu_launches": launches * args.steps,
            "clocks": clocks.summary(),
        }
    runner.close()
    dist.barrier()
    dist.destroy_process_group()
    return out


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    a = cpu_sample_matrix()
    v, sec, threads = run_cpu_reference(a, args.steps, args.warmup)
    cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"oracle port of oocdet.memdet_cholesky (SciPy LAPACK potrf/trtrs + NumPy BLAS, "
                     f"as the reference calls them) on the leading {SAMPLE_N}^2 principal submatrix of "
                     f"C2 (num_blocks=4, b=4096); mean of {args.steps} runs, {sec:.2f} s each"}
    return {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: C2 RBF Gram (host, seeded), bounded sample",
            "config": {"workload": "C2", "n": C2["n"], "num_blocks": C2["num_blocks"],
                       "sample_n": SAMPLE_N, "parallelism": "cpu"},
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
