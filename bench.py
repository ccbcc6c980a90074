"""Benchmark: exact linear-memory DTW (arXiv 2008.02734) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

Default workload (BASELINE.json metric/configs[2]): one exact alignment of two
synthetic 12-dim chroma-like sequences, M = N = 100,000, fp32 accumulation
(bit-identical to the reference's precision=32), min_dim = 500.  A step is one
full alignment.  Metric: GCUPS = cells_processed / s (the reference's own
counter, ~2*M*N), plus seconds per alignment.

value  : inputs resident in HBM (device pointers through the C ABI), CUDA
         events on the library's stream, L2 flushed between steps.
e2e    : the public drop-in call linmdtw(FeatureSeries, ...) on pinned host
         buffers: H2D copies, all kernels, path D2H and host stitching timed.
roofline: the strip-wavefront kernel's cell updates/s (CUDA events around
         every half-pass launch in the timed steps) against the FP32 cell-
         update roofline of SURVEY.md 8(d): N_SM * 128 * f_max / (2d + 5).
cpu_baseline: the C oracle (oracle/, a restatement of the reference) on a
         bounded sample, single-threaded.
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
    if name == "cfg5":
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


def cpu_sample(prec=32, nthreads=1, M=20000, N=20000, seed=3):
    """Oracle linmdtw on a bounded sample of the workload: a cfg3-generator pair
    at 20k x 20k (cfg2 shape).  Returns (gcups, seconds, cells)."""
    from oracle import oracle as O
    O.build()
    X, Y = chroma_pair(M, N, 12, seed=seed)
    t = time.perf_counter()
    r = O.linmdtw(X, Y, min_dim=500, precision=prec, nthreads=nthreads)
    dt = time.perf_counter() - t
    return r["cells_processed"] / dt / 1e9, dt, r["cells_processed"]


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
    """--impl reference: the reference's CPU algorithm (the C oracle restating
    it; the reference itself is Python+numba and is not shipped to the box)
    with all host threads, one bounded sample per step."""
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    nthreads = O.num_threads()
    X, Y = chroma_pair(20000, 20000, 12, seed=3)
    vals = []
    for s in range(args.warmup + args.steps):
        t = time.perf_counter()
        r = O.linmdtw(X, Y, min_dim=500, precision=32, nthreads=nthreads)
        dt = time.perf_counter() - t
        if s >= args.warmup:
            vals.append((r["cells_processed"], dt))
    cells = sum(c for c, _ in vals)
    secs = sum(t for _, t in vals)
    gcups = cells / secs / 1e9
    model, ncpu = cpu_desc()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gcups, 4), "unit": "GCUPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs / len(vals), 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "chroma-like 20000x20000 d=12 seed 3 (bounded sample of cfg3), min_dim=500"},
        "cpu_baseline": {"value": round(gcups, 4), "unit": "GCUPS", "cores": nthreads, "kind": "port",
                         "sample": f"oracle linmdtw 20000x20000 fp32 per step; {model}, nproc={ncpu}"},
        "e2e": {"value": round(gcups, 4), "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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
    _capi.profile(True)
    _capi.profile_reset()
    l0 = _capi.launch_count()
    with ClockSampler(dev) as clk:
        ms, cells, info = timed(one_device, args.steps)
    launches = _capi.launch_count() - l0
    prof = _capi.profile_get()
    _capi.profile(False)
    clocks = clk.summary()
    step_ms = sum(ms) / len(ms)
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
    h2d = sum(X.nbytes + Y.nbytes for X, Y in pairs)
    K = sum(X.shape[0] + Y.shape[0] for X, Y in pairs)
    d2h = K * 16  # path (i,j) int64 pairs ~ M+N per alignment (upper bound)

    peaks, kind = measured_peaks()
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    f_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    roof = fp32_cell_roofline(d, n_sm, f_mhz)
    wave_rate = prof["wave_cells"] / (prof["wave_ms"] / 1e3) if prof["wave_ms"] > 0 else 0.0
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
                   "cells_per_step": cells // args.steps, "sec_per_alignment": round(step_ms / 1e3 / n_total, 6),
                   "l2": "flushed (256 MiB write) between timed steps", "parallelism": ("single-gpu" if world == 1 else
                                   (f"level-sharded x{world} (one alignment, distributed.py)" if dist_single
                                    else f"pairs sharded longest-first over {world} ranks"))},
        "e2e": {"value": round(e2e_value, 3), "unit": "GCUPS", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
                "api": "paper_2008_02734_b200.linmdtw (pinned host FeatureSeries)"},
        "roofline": {"bound": "fp32", "kernel": "wave_kernel (half passes)", "achieved": round(wave_rate / 1e9, 2),
                     "peak": round(roof / 1e9, 2), "unit": "Gcell/s", "frac": round(wave_rate / roof, 4),
                     "traffic": traffic, "traffic_basis": traffic_basis,
                     "peak_basis": f"N_SM={n_sm} x 128 lanes x {f_mhz} MHz ({kind} sm_max_mhz) / (2d+5), d={d}",
                     "kernel_ms_share": round(prof["wave_ms"] / sum(ms), 4) if sum(ms) > 0 else None},
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        g, secs, ncell = cpu_sample(prec=32, nthreads=1)
        model, ncpu = cpu_desc()
        line["cpu_baseline"] = {"value": round(g, 4), "unit": "GCUPS", "cores": 1, "kind": "port",
                                "sample": f"oracle linmdtw chroma 20000x20000 d=12 fp32 ({ncell} cells, "
                                          f"{secs:.1f} s); {model}, nproc={ncpu}"}
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
