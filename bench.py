"""Benchmark: exact linear-memory DTW (arXiv 2008.02734) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

Default workload (BASELINE.json metric/configs[2]): one exact alignment of two
synthetic 12-dim chroma-like sequences, M = N = 100,000, fp32 accumulation
(bit-identical to the reference's precision=32), min_dim = 500.  A step is one
full alignment.  Metric: GCUPS = cells_processed / s (the reference's own
counter, ~2*M*N), plus seconds per alignment.

value  : inputs resident in HBM (device pointers through the C ABI), CUDA
         events on the library's stream, L2 flushed between steps.  Cells are
         the reference's cells_processed counter (both half passes of every
         node, ~2MN); the engine updates fewer (a child inherits one of its two
         half passes from its parent): config.cells_computed_per_step.  The
         timed steps run with the library's launch profiling off.
e2e    : the public drop-in call linmdtw(FeatureSeries, ...) on pinned host
         buffers: H2D copies, all kernels, path D2H and host stitching timed.
roofline: a separate profiled pass (CUDA events around every half-pass
         launch on the library's stream, read back at the engine's own sync
         points) gives the strip-wavefront kernel's time per step; achieved =
         the reference's half-pass cell updates per step over that time
         (achieved = GCUPS / R_fp32(d)), achieved_computed =
         the cells the kernel actually updates; peak = the FP32 cell-update
         roofline N_SM * 128 * f_max / (2d + 5).
cpu_baseline: the C oracle (oracle/, a restatement of the reference) with
         all host threads on the same workload (cfg4: a stated subsample).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "exact linear-mem DTW cell updates/s (GCUPS) at M=N=100k; sec/alignment"


# ------------------------------------------------------------------ inputs
def warp_positions(length, strength, rng):
    """Monotone warp of [0,1] (same construction as the reference's
    synth._warp_positions, synth.py:17-28)."""
    t = np.linspace(0.0, 1.0, length)
    if strength == 0.0:
        return t
    phase = rng.uniform(0, 2 * np.pi)
    w = np.sin(np.pi * t) / np.pi + 0.3 * np.sin(2 * np.pi * t + phase) / (2 * np.pi)
    u = t + 0.7 * strength * w
    return (u - u[0]) / (u[-1] - u[0])


def _latent_pair(M, N, d, seed):
    rng = np.random.default_rng(seed)
    w = np.cumsum(rng.standard_normal((M, d)), 0) / np.sqrt(M)
    u = warp_positions(N, 0.3, rng)
    t = np.linspace(0, 1, M)
    wy = np.stack([np.interp(u, t, w[:, c]) for c in range(d)], 1) + 0.01 * rng.standard_normal((N, d))
    return w, wy


def chroma(v):
    a = np.abs(v) + 1e-3
    return a / np.linalg.norm(a, axis=1, keepdims=True)


def chroma_pair(M, N, d=12, seed=2):
    """SURVEY.md 8(d) cfg2/cfg3 generator: 12-dim chroma-like sequences."""
    w, wy = _latent_pair(M, N, d, seed)
    return (np.ascontiguousarray(chroma(w), dtype=np.float32),
            np.ascontiguousarray(chroma(wy), dtype=np.float32))


def latent_pair(M, N, d=48, seed=5):
    """SURVEY.md 8(d) cfg5 generator: random-walk latent and its warped copy."""
    w, wy = _latent_pair(M, N, d, seed)
    return np.ascontiguousarray(w, dtype=np.float32), np.ascontiguousarray(wy, dtype=np.float32)


CONFIGS = {
    "cfg1": dict(workload="random-walk pair M=N=1000 d=2 (synth_pair seed 0)", M=1000, N=1000, d=2, prec=64),
    "cfg2": dict(workload="chroma-like M=N=20000 d=12 seed 2", M=20000, N=20000, d=12, seed=2, prec=32),
    "cfg3": dict(workload="chroma-like M=N=100000 d=12 seed 3", M=100000, N=100000, d=12, seed=3, prec=32),
    "cfg3x64": dict(workload="chroma-like M=N=100000 d=12 seed 3 (fp64)", M=100000, N=100000, d=12, seed=3,
                    prec=64),
    "cfg4": dict(workload="256 pairs M,N~U[5k,30k] d=12 chroma-like (rng 4)", batch=256, d=12, prec=32),
    "cfg5": dict(workload="M=200000 N=20000 d=48 latent walk seed 5 (fp64)", M=200000, N=20000, d=48, seed=5,
                 prec=64),
    # the reference extractor's feature width (mfcc-mod / DLNC0, d = 100): the WIDE kernels
    "d100": dict(workload="latent walk M=N=20000 d=100 seed 100 (fp32)", M=20000, N=20000, d=100, seed=100,
                 prec=32),
    "d100x64": dict(workload="latent walk M=N=20000 d=100 seed 100 (fp64)", M=20000, N=20000, d=100, seed=100,
                    prec=64),
}


def make_inputs(name):
    c = CONFIGS[name]
    if name == "cfg1":
        rng = np.random.default_rng(0)
        steps = rng.standard_normal((1000, 2))
        base = np.cumsum(steps, 0) / np.sqrt(1000)
        t = np.linspace(0, 1, 1000)
        u = warp_positions(1000, 0.3, rng)
        warped = np.stack([np.interp(u, t, base[:, q]) for q in range(2)], 1)
        return [(base.astype(np.float32), warped.astype(np.float32))]
    if name == "cfg4":
        rng = np.random.default_rng(4)
        MN = rng.integers(5000, 30001, size=(c["batch"], 2))
        return [chroma_pair(int(m), int(n), 12, seed=1000 + q) for q, (m, n) in enumerate(MN)]
    if name in ("cfg5", "d100", "d100x64"):
        return [latent_pair(c["M"], c["N"], c["d"], c["seed"])]
    return [chroma_pair(c["M"], c["N"], c["d"], c["seed"])]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    every 2 ms (pynvml), else nvidia-smi every 100 ms."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index=0):
        self.idx = gpu_index
        self.sm, self.mx, self.reasons = [], [], set()
        self.source = "unsampled"
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.idx)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
        while not self._stop.is_set():
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            self.mx.append(float(mx))
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            for nm, b in bits.items():
                if r & b:
                    self.reasons.add(nm)
            self._stop.wait(0.002)

    def _run_smi(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    r = [x.strip() for x in out.split(",")]
                    if r[1].replace(".", "").isdigit():
                        self.sm.append(float(r[1]))
                    if r[2].replace(".", "").isdigit():
                        self.mx.append(float(r[2]))
                    for q, nm in enumerate(self.NAMES):
                        if len(r) > 5 + q and r[5 + q].lower().startswith("active"):
                            self.reasons.add(nm)
            except Exception:
                pass
            self._stop.wait(0.1)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.source = "nvml"
            try:
                self._run_nvml(nv)
            finally:
                nv.nvmlShutdown()
        except Exception:
            self.source = "nvidia-smi"
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


# ------------------------------------------------------------------ helpers
def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def fp32_cell_roofline(d, n_sm, f_mhz):
    """cells/s = N_SM * 128 FP32 lanes * f / (2d + 5)."""
    return n_sm * 128 * f_mhz * 1e6 / (2 * d + 5)


# cfg4 on the CPU: a stated subsample of the batch (the whole batch is ~1.6e11 cells)
CPU_CFG4_PAIRS = 8


def cpu_workload(name, min_dim=500):
    """The CPU leg's sample of config `name`: the whole workload (the same
    inputs the GPU arm aligns) except cfg4, where the first CPU_CFG4_PAIRS
    pairs of the batch are aligned.  Returns (pairs, description)."""
    pairs = make_inputs(name)
    c = CONFIGS[name]
    if name == "cfg4":
        pairs = pairs[:CPU_CFG4_PAIRS]
        return pairs, f"first {len(pairs)} of the 256 cfg4 pairs (same inputs as the GPU arm)"
    return pairs, f"the whole {name} workload: {c['workload']} (same inputs as the GPU arm)"


def cpu_run(name, pairs, nthreads, min_dim=500):
    """The oracle (C restatement of the reference, test infrastructure) over
    `pairs` with `nthreads` host threads.  Returns (gcups, seconds, cells)."""
    from oracle import oracle as O
    O.build()
    prec = CONFIGS[name]["prec"]
    cells = 0
    t = time.perf_counter()
    for X, Y in pairs:
        cells += O.linmdtw(X, Y, min_dim=min_dim, precision=prec, nthreads=nthreads)["cells_processed"]
    dt = time.perf_counter() - t
    return cells / dt / 1e9, dt, cells


def numba_reference_cfg2():
    """The real reference (Python + numba, installed unmodified in
    baseline/_ref), JIT warmed on cfg1 first, SURVEY.md 8(d)'s repetitions
    where they fit a bench run: cfg1 x10 (fp64), cfg2 x3 (fp32, one core --
    numba holds the GIL), and cfg4 as an all-core multiprocessing pool (one
    pair per task) over the first 32 pairs.  None when it cannot be
    imported on this host."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "lmdtw")):
        return None
    code = (
        "import sys, time, json, os, multiprocessing as mp\n"
        f"sys.path.insert(0, {ref!r}); sys.path.insert(1, {ROOT!r})\n"
        "import lmdtw, bench\n"
        "X, Y = bench.make_inputs('cfg1')[0]\n"
        "lmdtw.linmdtw(X, Y, precision=32); lmdtw.linmdtw(X, Y, precision=64)\n"
        "t = time.perf_counter()\n"
        "for _ in range(10): r1 = lmdtw.linmdtw(X, Y, precision=64)\n"
        "dt1 = (time.perf_counter() - t) / 10\n"
        "X, Y = bench.make_inputs('cfg2')[0]\n"
        "ts = []\n"
        "for _ in range(3):\n"
        "    t = time.perf_counter(); r = lmdtw.linmdtw(X, Y, precision=32); ts.append(time.perf_counter() - t)\n"
        "def work(p):\n"
        "    return int(lmdtw.linmdtw(p[0], p[1], precision=32).cells_processed)\n"
        "pairs = bench.make_inputs('cfg4')[:32]\n"
        "n = os.cpu_count()\n"
        "with mp.get_context('fork').Pool(n) as pool:\n"
        "    pool.map(work, [bench.make_inputs('cfg1')[0]] * n, chunksize=1)\n"
        "    t = time.perf_counter(); c4 = pool.map(work, pairs, chunksize=1); dt4 = time.perf_counter() - t\n"
        "print(json.dumps({'cells': int(r.cells_processed), 'secs': sorted(ts)[1], 'all': ts, 'cost': float(r.cost),\n"
        "                  'cells1': int(r1.cells_processed), 'secs1': dt1, 'cost1': float(r1.cost),\n"
        "                  'cells4': sum(c4), 'secs4': dt4, 'n4': len(pairs), 'procs': n}))\n")
    env = dict(os.environ, NUMBA_CACHE_DIR="/tmp/lmdtw_numba_cache", PYTHONDONTWRITEBYTECODE="1")
    try:
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=420,
                             env=env, cwd="/tmp")
        r = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None
    return {"value": round(r["cells"] / r["secs"] / 1e9, 4), "unit": "GCUPS", "cores": 1, "kind": "reference",
            "seconds": round(r["secs"], 2), "seconds_all": [round(v, 2) for v in r["all"]], "cost": r["cost"],
            "sample": "unmodified reference lmdtw.linmdtw (baseline/_ref, numba) on cfg2 20000x20000 d=12 fp32, "
                      "median of 3",
            "cfg1": {"sec_per_alignment": round(r["secs1"], 5), "GCUPS": round(r["cells1"] / r["secs1"] / 1e9, 4),
                     "cost": r["cost1"], "reps": 10,
                     "sample": "the same reference on cfg1 (1000x1000 d=2 random walks, fp64), mean of 10"},
            "cfg4": {"GCUPS": round(r["cells4"] / r["secs4"] / 1e9, 4), "seconds": round(r["secs4"], 2),
                     "pairs_per_s": round(r["n4"] / r["secs4"], 3), "cores": r["procs"],
                     "sample": f"the same reference on the first {r['n4']} cfg4 pairs, fp32, multiprocessing "
                               f"pool of {r['procs']} processes, one pair per task (all cores)"}}


def host_threads() -> int:
    """All host threads this process may run on.  Not omp_get_max_threads():
    torchrun sets OMP_NUM_THREADS=1 in every rank, and the reference arm's
    rank 0 must still use the whole host (the oracle passes the count to
    its num_threads clause)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_desc():
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = "unknown"
    return model, os.cpu_count()


def _bench_device() -> int:
    if os.environ.get("LMDTW_BENCH_SAME_DEVICE") == "1":
        return 0
    return int(os.environ.get("LOCAL_RANK", "0"))


def _allreduce(v: float, op: str) -> float:
    """Scalar all-reduce over the bench ranks (device tensor under NCCL)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------------ arms
def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm on this host -- the C
    oracle restating it (the reference itself is Python + numba and holds
    the GIL, so it is effectively one core) with all host threads, on the same
    config, inputs and metric as our arm.  Each timed step is the whole
    workload (cfg4: a stated subsample); the warm-up steps run cfg1 (there is
    no JIT to warm).  The real numba reference is timed on cfg2 beside it."""
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    nthreads = host_threads()
    pairs, desc = cpu_workload(args.config, args.min_dim)
    warm = make_inputs("cfg1")
    for _ in range(args.warmup):
        cpu_run("cfg1", warm, nthreads)
    cells, secs = 0, 0.0
    for _ in range(args.steps):
        _, dt, c = cpu_run(args.config, pairs, nthreads, args.min_dim)
        cells += c
        secs += dt
    gcups = cells / secs / 1e9
    model, ncpu = cpu_desc()
    prec = CONFIGS[args.config]["prec"]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gcups, 4), "unit": "GCUPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs / args.steps, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if prec == 32 else "f64", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config]["workload"], "min_dim": args.min_dim, "precision": prec,
                   "cells_per_step": cells // args.steps, "same_config": args.config != "cfg4",
                   "sample": desc},
        "cpu_baseline": {"value": round(gcups, 4), "unit": "GCUPS", "cores": nthreads, "kind": "port",
                         "sample": f"oracle linmdtw (C restatement of the reference), {desc}, per step; "
                                   f"{model}, nproc={ncpu}"},
        "e2e": {"value": round(gcups, 4), "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu:
        nb = numba_reference_cfg2()
        line["reference_numba"] = nb if nb is not None else {"unavailable": "numba reference not importable"}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import ctypes as C
    import torch
    import paper_2008_02734_b200 as L
    from paper_2008_02734_b200 import _capi
    from paper_2008_02734_b200.divide import _c_config

    dev = _bench_device()
    torch.cuda.set_device(dev)
    L.set_device(dev)
    lib = _capi.load()
    cfgd = CONFIGS[args.config]
    prec = cfgd["prec"]
    pairs = make_inputs(args.config)
    n_total = len(pairs)
    d = pairs[0][0].shape[1]
    cfg = L.LinMdtwConfig(min_dim=args.min_dim, precision=prec)
    ccfg = _c_config(cfg)

    # device-resident inputs
    dX = [torch.from_numpy(X).cuda() for X, _ in pairs]
    dY = [torch.from_numpy(Y).cuda() for _, Y in pairs]
    stream = torch.cuda.ExternalStream(_capi.stream_handle(dev))
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    # N > 1: one alignment's recursion sharded over the ranks (strong scaling,
    # distributed.linmdtw_distributed); batches: pairs sharded longest-first
    dist_single = world > 1 and len(pairs) == 1
    if dist_single:
        from paper_2008_02734_b200.distributed import DeviceEngine, linmdtw_distributed
        resident = DeviceEngine(pairs[0][0], pairs[0][1], cfg, dev)
    if world > 1 and len(pairs) > 1:
        from paper_2008_02734_b200.distributed import lpt_assign
        own = lpt_assign([X.shape[0] * Y.shape[0] for X, Y in pairs], world)
        keep = [q for q in range(len(pairs)) if own[q] == rank]
        pairs = [pairs[q] for q in keep]
        dX = [dX[q] for q in keep]
        dY = [dY[q] for q in keep]

    def one_device():
        n = len(pairs)
        if dist_single:
            r = linmdtw_distributed(pairs[0][0], pairs[0][1], config=cfg, engine=resident)
            return r.cells_processed, None
        if n == 0:
            return 0, None
        if n == 1:
            h = C.c_void_p()
            _capi.check(lib.lmdtw_align(dev, C.c_void_p(dX[0].data_ptr()), pairs[0][0].shape[0],
                                        C.c_void_p(dY[0].data_ptr()), pairs[0][1].shape[0], d, C.byref(ccfg),
                                        _capi.MEM_DEVICE, _capi.PROGRESS_FN(), None, C.byref(h)))
            hs = [h]
        else:
            xp = (C.c_void_p * n)(*[t.data_ptr() for t in dX])
            yp = (C.c_void_p * n)(*[t.data_ptr() for t in dY])
            Ms = (C.c_int64 * n)(*[X.shape[0] for X, _ in pairs])
            Ns = (C.c_int64 * n)(*[Y.shape[0] for _, Y in pairs])
            arr = (C.c_void_p * n)()
            _capi.check(lib.lmdtw_align_batch(dev, n, xp, Ms, yp, Ns, d, C.byref(ccfg), _capi.MEM_DEVICE, arr))
            hs = [C.c_void_p(arr[q]) for q in range(n)]
        cells, info = 0, None
        for h in hs:
            info = _capi.AlignInfo()
            lib.lmdtw_result_info(h, C.byref(info))
            cells += info.cells_processed
            lib.lmdtw_result_free(h)
        return cells, info

    def timed(fn, steps):
        tot_ms, cells_all = [], 0
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            cells, info = fn()
            e1.record(stream)
            e1.synchronize()
            tot_ms.append(e0.elapsed_time(e1))
            cells_all += cells
        return tot_ms, cells_all, info

    for _ in range(args.warmup):
        one_device()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # timed steps with the library's launch profiling OFF (no events recorded
    # around the kernels); the kernel shares come from a separate pass below
    l0 = _capi.launch_count()
    with ClockSampler(dev) as clk:
        ms, cells, info = timed(one_device, args.steps)
    launches = _capi.launch_count() - l0
    clocks = clk.summary()
    # profiled pass (not timed for `value`): CUDA events around every wave
    # launch on the library's stream, read at the engine's own sync points
    psteps = max(1, min(args.steps, 3))
    _capi.profile(True)
    _capi.profile_reset()
    pms_prof, _, _ = timed(one_device, psteps)
    prof = _capi.profile_get()
    _capi.profile(False)
    step_ms = sum(ms) / len(ms)
    cells_rank = cells  # this rank's share (the roofline below is per GPU)
    if world > 1:
        step_ms = _allreduce(step_ms, "max")
        if not dist_single:  # sharded batch: every rank's pairs count
            cells = int(_allreduce(float(cells), "sum"))
    value = (cells / args.steps) / (step_ms / 1e3) / 1e9

    # e2e: the public drop-in API on pinned host buffers
    pin = []
    for X, Y in pairs:
        tx = torch.from_numpy(X).pin_memory()
        ty = torch.from_numpy(Y).pin_memory()
        pin.append((L.FeatureSeries(tx.numpy()), L.FeatureSeries(ty.numpy()), tx, ty))

    def one_e2e():
        if dist_single:
            r = linmdtw_distributed(pin[0][0], pin[0][1], config=cfg)
            return r.cells_processed, None
        if len(pin) == 0:
            return 0, None
        if len(pin) == 1:
            r = L.linmdtw(pin[0][0], pin[0][1], config=cfg)
            return r.cells_processed, None
        rs = L.align_batch([(a, b) for a, b, _, _ in pin], config=cfg)
        return sum(r.cells_processed for r in rs), None

    one_e2e()
    ems, ecells, _ = timed(one_e2e, max(1, min(args.steps, 3)))
    e2e_ms = sum(ems) / len(ems)
    if world > 1:
        e2e_ms = _allreduce(e2e_ms, "max")
        if not dist_single:
            ecells = int(_allreduce(float(ecells), "sum"))
    e2e_value = (ecells / len(ems)) / (e2e_ms / 1e3) / 1e9
    # the reference's natural inputs: pageable numpy arrays (FeatureSeries)
    page = [(L.FeatureSeries(X), L.FeatureSeries(Y)) for X, Y in pairs]

    def one_pageable():
        if dist_single:
            return linmdtw_distributed(page[0][0], page[0][1], config=cfg).cells_processed, None
        if len(page) == 0:
            return 0, None
        if len(page) == 1:
            return L.linmdtw(page[0][0], page[0][1], config=cfg).cells_processed, None
        return sum(r.cells_processed for r in L.align_batch(page, config=cfg)), None

    pms, pcells, _ = timed(one_pageable, max(1, min(args.steps, 3)))
    page_ms = sum(pms) / len(pms)
    if world > 1:
        page_ms = _allreduce(page_ms, "max")
        if not dist_single:
            pcells = int(_allreduce(float(pcells), "sum"))
    page_value = (pcells / len(pms)) / (page_ms / 1e3) / 1e9
    h2d = sum(X.nbytes + Y.nbytes for X, Y in pairs)
    K = sum(X.shape[0] + Y.shape[0] for X, Y in pairs)
    d2h = K * 16  # path (i,j) int64 pairs ~ M+N per alignment (upper bound)

    peaks, kind = measured_peaks()
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    f_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    roof = fp32_cell_roofline(d, n_sm, f_mhz)
    # per step of the profiled pass: half-pass wave kernel time, the cells it
    # updates, and the reference's count of the half-pass cells it stands for
    # (cells_processed minus the leaves' brute-force cells, SURVEY.md 8(d):
    # roofline.achieved = GCUPS / R_fp32(d) in the reference's cell count)
    wave_ms_step = prof["wave_ms"] / psteps
    wave_computed = prof["wave_cells"] / psteps
    wave_algo = (cells_rank / args.steps) - prof["leaf_cells"] / psteps
    wave_rate = wave_algo / (wave_ms_step / 1e3) if wave_ms_step > 0 else 0.0
    wave_rate_computed = wave_computed / (wave_ms_step / 1e3) if wave_ms_step > 0 else 0.0
    # dram bytes per launch of the dominant kernel (level-0 wave_kernel) from one
    # ncu --set full capture, committed under profiles/ (null if not captured)
    traffic, traffic_basis = None, None
    tp = os.path.join(ROOT, "profiles", "wave_kernel_traffic.json")
    if os.path.exists(tp):
        try:
            t = json.load(open(tp)).get(args.config)
            if t:
                traffic = t["per_launch_bytes"]
                traffic_basis = (f"{t['launch']}: dram read+write per launch for {t['cells']} cells; algorithmic: "
                                 f"X+Y features once + 6 output diagonals ~= {t.get('algorithmic_bytes', 'n/a')} B")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms, 3), "higher_is_better": True,
        "scaling": "strong" if dist_single else "weak", "vs_baseline": None,
        "dtype": "f32" if prec == 32 else "f64", "data": "synthetic",
        "config": {"workload": cfgd["workload"], "min_dim": args.min_dim, "precision": prec,
                   "cells_per_step": cells // args.steps,
                   "cells_computed_per_step": (prof["wave_cells"] + prof["leaf_cells"]) // psteps,
                   "sec_per_alignment": round(step_ms / 1e3 / n_total, 6),
                   "l2": "flushed (256 MiB write) between timed steps", "parallelism": ("single-gpu" if world == 1 else
                                   (f"level-sharded x{world} (one alignment, distributed.py)" if dist_single
                                    else f"pairs sharded longest-first over {world} ranks"))},
        "e2e": {"value": round(e2e_value, 3), "unit": "GCUPS", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
                "api": "paper_2008_02734_b200.linmdtw (pinned host FeatureSeries)"},
        "e2e_pageable": {"value": round(page_value, 3), "unit": "GCUPS", "ms_per_step": round(page_ms, 3),
                         "api": "paper_2008_02734_b200.linmdtw (pageable numpy FeatureSeries)"},
        "roofline": {"bound": "fp32", "kernel": "wave_kernel (half passes)", "achieved": round(wave_rate / 1e9, 2),
                     "peak": round(roof / 1e9, 2), "unit": "Gcell/s", "frac": round(wave_rate / roof, 4),
                     "achieved_basis": ("the reference's half-pass cell updates per step (cells_processed minus "
                                        "leaf cells) / the half-pass wave_kernel time per step (CUDA events, "
                                        "separate profiled pass); SURVEY 8(d)"),
                     # what the kernel actually updates: with half-pass reuse a child inherits one of
                     # its two half passes from its parent, so it updates ~0.76 of the reference count
                     "achieved_computed": round(wave_rate_computed / 1e9, 2),
                     "frac_computed": round(wave_rate_computed / roof, 4),
                     "traffic": traffic, "traffic_basis": traffic_basis,
                     "peak_basis": f"N_SM={n_sm} x 128 lanes x {f_mhz} MHz ({kind} sm_max_mhz) / (2d+5), d={d}",
                     "kernel_ms_share": round(prof["wave_ms"] / sum(pms_prof), 4) if sum(pms_prof) > 0 else None,
                     # the whole alignment (value, every kernel and host gap) against the same peak
                     "frac_alignment": round(value * 1e9 / roof, 4)},
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as O
        nthreads = host_threads()
        cpairs, desc = cpu_workload(args.config, args.min_dim)
        g, secs, ncell = cpu_run(args.config, cpairs, nthreads, args.min_dim)
        model, ncpu = cpu_desc()
        line["cpu_baseline"] = {"value": round(g, 4), "unit": "GCUPS", "cores": nthreads, "kind": "port",
                                "sample": f"oracle linmdtw (C restatement of the reference), {desc}: "
                                          f"{ncell} cells in {secs:.1f} s; {model}, nproc={ncpu}"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--min-dim", type=int, default=500)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(_bench_device())
        # LMDTW_BENCH_BACKEND=gloo + LMDTW_BENCH_SAME_DEVICE=1: exercise the
        # N > 1 path with every rank on cuda:0 (1-GPU boxes); timings then
        # measure contention, not scaling
        dist.init_process_group(os.environ.get("LMDTW_BENCH_BACKEND", "nccl"))
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
