#!/usr/bin/env python
"""Benchmark: additive-kernel NFFT matvecs/s on BASELINE config 4.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[3], the one the metric is quoted on):
N = 1,000,000 points, d = 30 (seeded 5-component Gaussian mixture), 10
consecutive windows of 3 features, Gaussian kernel, ell = 1 (prescaled
1/sqrt(3)), sigma_f = 1, one RHS, reference default NFFT setup (m = 32,
n = 64, cutoff 6, Kaiser-Bessel).  A step is one full K v over all windows.

* ``value``: K v per second with v and the plan resident in HBM (device API).
* ``e2e``: the same through the public numpy API (fast_matvec with a host
  vector): H2D of v and D2H of K v inside every timed step.
* ``deriv``: (K v, dK/d ell v, dK/d sigma_f v) triples per second from one
  shared spread (fast_matvecs).
* ``roofline``: the dominant kernel (q=3 spread or interp) timed alone with
  CUDA events on the launching stream; FP64-FMA-bound, so achieved TFLOP/s of
  algorithmic FLOPs (2 * 12^3 per point per window) against the FP64 DFMA
  peak measured in this run (MEASURED_PEAKS.json has no FP64 entry).
* ``cpu_baseline``: the reference's OWN fast_matvec (numba, installed unmodified
  into baseline/_ref) on one window at full N, one core (its kernels are
  serial), scaled to 10 windows; the oracle port's single-core time on the same
  window is reported beside it.  Falls back to the port if baseline/_ref is absent.
* ``rel_err_vs_oracle``: the GPU K v against the oracle at full size, all ten
  windows (oracle/fullsize.py on every host thread); ``extras`` carry the same
  for configs 3 (all 8 RHS, K and dK/dl) and 5 (RHS 0 and 15: K, every dK/dl_w,
  dK/ds), per-kernel device times (ak_prof_* events) and per-kernel rooflines.

Multi-GPU (torchrun): --shard cell (default) splits the ranks into G window
groups x Q cell slabs (G from distributed.hybrid_layout: 2 x 4 on 8 GPUs for
config 4); each rank spreads the rows of its slab of whole grid cells of each
owned window (one row-masked plan), the band spectra are all-reduced within
the window group, each rank interpolates its slab rows, and one all-reduce of
the length-N partials assembles K v.  --shard hybrid uses row blocks instead
of cell slabs (same collectives; thinner cells per rank: per-rank device time
0.871 vs 0.812 ms at 4 ranks, 0.495 vs 0.488 at 8, equal at 2, tools/rank_emulate.py);
--shard point (G = 1) / window (Q = 1) are the two pure decompositions.
Timing is the max over ranks; the roofline is rank 0's local kernels.
``--gpus N`` without a torchrun environment re-launches itself under
torch.distributed.run with N local ranks (and fails if fewer devices exist);
under torchrun WORLD_SIZE must equal --gpus.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

L2_NOTE = "inputs larger than L2: per-step geometry stream 32 B x 1M x 10 windows = 320 MB (no flush needed)"
SHARD_NAMES = {"cell": "window groups x cell slabs", "hybrid": "window groups x row blocks",
               "point": "row blocks (band all-reduce)", "window": "windows (row all-reduce)"}
METRIC = "additive-kernel matvecs/sec at N=1M, 10 windows (+dK mvs); rel. err vs dense/oracle"
WORKLOAD = ("C4: N=1,000,000, d=30 seeded 5-component Gaussian mixture (means U[-1,1], std 0.3), "
            "min-max scaled, 10 consecutive windows of 3, gauss ell=1 (prescaled 1/sqrt(3)), sigma_f=1, "
            "1 RHS v~N(0,1), preset default (m=32, n=64, cutoff 6, Kaiser-Bessel)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=1_000_000, help="points (default: the config's 1M)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip extras (for profilers)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: functional check of the multi-rank path with several ranks on one device "
                         "(host-side collectives; its timings are not bench values)")
    ap.add_argument("--shard", choices=["cell", "hybrid", "point", "window"], default="cell",
                    help="multi-GPU decomposition (N > 1): window groups x cell slabs (default), x row blocks, "
                         "rows only, windows only")
    return ap.parse_args()


def config_dict(args) -> dict:
    """The workload description both arms print (identical dicts: the driver compares them)."""
    par = "single GPU" if args.gpus == 1 else f"{SHARD_NAMES[args.shard]} over {args.gpus} GPUs, NCCL"
    if args.gpus > 1 and getattr(args, "dist_backend", "nccl") == "gloo":
        par = f"{SHARD_NAMES[args.shard]} over {args.gpus} ranks on one device, gloo (functional check, not a bench value)"
    return {"workload": WORKLOAD, "N": args.n, "windows": 10, "rhs": 1, "parallelism": par, "l2": L2_NOTE}


def ensure_world(args) -> None:
    """--gpus N: under torchrun WORLD_SIZE must equal N; without a launcher, re-exec
    under torch.distributed.run with N local ranks (one process per GPU)."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            sys.stderr.write(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}\n")
            sys.exit(2)
        return
    if args.gpus <= 1:
        return
    if args.dist_backend == "nccl":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, {have} visible\n")
            sys.exit(2)
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# reference arm (CPU oracle port)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import restate as R
    from paper_2404_17344_b200 import configs

    wl = configs.config4(args.n)
    cores = len(os.sched_getaffinity(0))
    P = len(wl.window_set)
    # every host thread: split each window's rows into chunks so that the
    # P * chunks gridding tasks divide evenly over the threads
    chunks = max(1, cores // math.gcd(P, cores))
    cols = [wl.window_set.columns(w) for w in wl.window_set]
    fs = R.ChunkedFastSum("gauss", wl.spec.ell, wl.spec.sigma_f, cols, wl.data.features, chunks=chunks)
    v = wl.V[0]
    from concurrent.futures import ThreadPoolExecutor

    pool = ThreadPoolExecutor(max_workers=cores)

    def step():
        fs.matvec_pool(v, pool)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    pool.shutdown()
    value = 1.0 / dt
    T = cores
    sample = (f"all {P} windows at full N={wl.data.n_rows} per step (one complete K v), rows split into "
              f"{chunks} chunks per window, {P * chunks} gridding tasks on {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "matvecs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args), "execution": f"host CPU, {T} threads",
        "cpu_baseline": {"value": value, "unit": "matvecs/s", "cores": T, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the oracle/ port of the reference path (same algorithm: serial C gridding loops + numpy "
                "pocketfft), gridding spread over every host thread -- the strongest CPU arm available: the "
                "reference's own numba kernels are serial (one core; timed in our arm's cpu_baseline)",
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def cuda_time(torch, fn, reps):
    """Average ms of fn() over reps, CUDA events on the current stream."""
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def kernel_roofline(torch, plan, wl, peaks, reps=10):
    """Time the q=3 spread and interp kernels alone (ak_spread / ak_interp: the
    same kernels ak_op_apply launches) and express them against the FP64 peak."""
    import ctypes

    from paper_2404_17344_b200 import _native
    from paper_2404_17344_b200.nufft import _stream_ptr

    lib = _native.lib()
    geom = plan.geometries
    N = plan.n_rows  # this rank's rows (all of them on one GPU)
    T = plan.nufft_plans[3].taps
    V = torch.as_tensor(np.ascontiguousarray(wl.V[:1, :N]), device="cuda").contiguous()
    grids = torch.zeros(geom.canon_total, dtype=torch.float64, device="cuda")
    out = torch.zeros(N, dtype=torch.float64, device="cuda")
    scale = torch.ones(geom.n_windows, dtype=torch.float64, device="cuda")
    st = _stream_ptr(torch)

    def spread():
        _native.check(lib.ak_spread(geom.handle, V.data_ptr(), 1, N, grids.data_ptr(), st))

    def interp():
        _native.check(lib.ak_interp(geom.handle, grids.data_ptr(), 1, scale.data_ptr(), out.data_ptr(), N, 1, 0, st))

    for _ in range(2):
        spread()
        interp()
    t_spread = cuda_time(torch, spread, reps)
    t_interp = cuda_time(torch, interp, reps)
    # algorithmic: one FMA per tap per point per window (a cell-slab rank's windows hold
    # only their slab's rows)
    pw3 = sum(r for w, r in zip(plan.window_set, geom.rows_per_window) if len(w) == 3)
    flops = 2.0 * T ** 3 * pw3
    fp64 = peaks["fp64_tflops"]
    name, t = ("spread_q3", t_spread) if t_spread >= t_interp else ("interp_q3", t_interp)
    achieved = flops / (t * 1e-3) / 1e12
    alg_bytes = pw3 * (24 + 8)  # coordinates + value (spread) / output (interp), compulsory
    prof = profiled_traffic(name)
    return {
        "bound": "fp64", "bound_note": "FP64 datapath (hybrid DMMA + DFMA spread / FP64-DMMA interp share it): one FMA per tap, "
                                      "12.9 FLOP per compulsory byte vs a ridge of ~5.6 -- neither HBM- nor "
                                      "low-precision-tensor-bound; HBM figures below",
        "kernel": name, "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
        "frac": achieved / fp64, "traffic": prof["bytes"] if prof else None,
        "traffic_source": (f"ncu --set full, {prof['source']} ({prof['kernel'][:40]}); includes the cached "
                           "window-weight stream (288 B/point), see DESIGN.md") if prof else None,
        "peak_source": "ak_probe_fp64 DFMA microbenchmark in this run (MEASURED_PEAKS.json has no FP64 figure)",
        "flops_per_launch": flops, "ms_per_launch": t,
        "spread_ms": t_spread, "interp_ms": t_interp,
        "hbm_algorithmic_gbs": alg_bytes / (t * 1e-3) / 1e9, "hbm_peak_gbs": peaks.get("hbm_gbs"),
        "ncu": ncu_evidence(prof),
    }


def profiled_traffic(kernel: str):
    """dram read+write bytes per launch of `kernel` from the newest committed ncu
    full capture summary (profiles/*_summary.json), or None."""
    best = None
    # round tags sort by name: r1 < r1b < ... < r1e < r2
    for f in sorted((ROOT / "profiles").glob("*_summary.json"), key=lambda p: p.name):
        try:
            data = json.loads(f.read_text())
        except (OSError, ValueError):
            continue
        key = "spread3" if kernel.startswith("spread") else "interp3"
        for m in data.get("full", []):
            if key in m.get("kernel", "") and m.get("dram_bytes_per_launch"):
                best = {"bytes": m["dram_bytes_per_launch"], "source": f.name, "kernel": m["kernel"], "metrics": m}
    return best


def ncu_evidence(prof):
    """Memory-side evidence of the dominant kernel from the same committed ncu capture
    (the north_star asks for achieved HBM GB/s and L2/atomic throughput)."""
    if not prof:
        return None
    m = prof["metrics"]
    dur = m.get("duration_s") or 0.0
    out = {"source": prof["source"], "duration_ms": dur * 1e3 if dur else None,
           "dram_gbs": prof["bytes"] / dur / 1e9 if dur else None,
           "l2_throughput_pct": m.get("l2_throughput_pct"), "dram_throughput_pct": m.get("dram_throughput_pct"),
           "fp64_pipe_pct": m.get("fp64_pipe_pct"), "dmma_pipe_pct": m.get("dmma_pipe_pct")}
    if m.get("fp64_pipe_pct") is not None and m.get("dmma_pipe_pct") is not None:
        # DFMA / DMUL and FP64 DMMA issue to one FP64 datapath (tools/fp64_mix.cu): its busy
        # share, of which the useful-slot fraction is algorithmic work
        out["fp64_datapath_busy_pct"] = m["fp64_pipe_pct"] + m["dmma_pipe_pct"]
    red = m.get("red_sectors_to_l2")
    if red is not None and dur:
        out["red_sectors_per_s"] = red / dur
    return out


def fp64_peak(torch):
    import ctypes

    from paper_2404_17344_b200 import _native
    from paper_2404_17344_b200.nufft import _stream_ptr

    lib = _native.lib()
    best = 0.0
    dmma = 0.0
    for _ in range(3):
        v = ctypes.c_double()
        _native.check(lib.ak_probe_fp64(20000, _stream_ptr(torch), ctypes.byref(v)))
        best = max(best, v.value)
        _native.check(lib.ak_probe_dmma(5000, _stream_ptr(torch), ctypes.byref(v)))
        dmma = max(dmma, v.value)
    return best, dmma


def reference_window_time(wl, k=0):
    """The reference's own fast_matvec (baseline/_ref: the unmodified package, numba
    kernels, serial) on window k of the workload at full N, one core.  Returns
    (plan_s, matvec_s, output) or None when baseline/_ref is not installed."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "addkern").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    sys.path.insert(0, str(ref_dir))
    try:
        from addkern import dataset as rds
        from addkern import fastsum as rfs
        from addkern import kernels as rk
        from addkern import windows as rw
    finally:
        sys.path.remove(str(ref_dir))
    if not str(Path(rfs.__file__).resolve()).startswith(str(ref_dir.resolve())):
        return None
    X = wl.data.features
    names = tuple(f"x{i + 1}" for i in range(X.shape[1]))
    spec = rk.KernelSpec("gauss", wl.spec.ell, wl.spec.sigma_f)
    ws = rw.WindowSet((wl.window_set.windows[k],), d_max=wl.window_set.d_max)
    small = rds.Dataset(X[:500], np.zeros(500), names, scaling_state=rds.PRESCALED, d_max=wl.data.d_max)
    rfs.fast_matvec(rfs.build_plan(spec, ws, "default", small), wl.V[0][:500])   # numba JIT outside the timing
    ds = rds.Dataset(X, np.zeros(X.shape[0]), names, scaling_state=rds.PRESCALED, d_max=wl.data.d_max)
    t0 = time.perf_counter()
    plan = rfs.build_plan(spec, ws, "default", ds)
    t1 = time.perf_counter()
    out = rfs.fast_matvec(plan, wl.V[0])
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, out


def cpu_baseline(wl, gpu_window0):
    """cpu_baseline: the reference's own fast_matvec on window 1 at full N (one core,
    scaled x10 windows); the oracle port timed on the same window beside it.
    Returns (cpu_baseline dict, rel err of the GPU's window-1 product vs the reference)."""
    from oracle import restate as R

    P = len(wl.window_set)
    cols0 = [wl.window_set.columns(wl.window_set.windows[0])]
    t0 = time.perf_counter()
    port = R.FastSum("gauss", wl.spec.ell, wl.spec.sigma_f, cols0, wl.data.features).matvec(wl.V[0])
    t_port = time.perf_counter() - t0
    ref = reference_window_time(wl)
    if ref is None:
        err = float(np.linalg.norm(gpu_window0 - port) / np.linalg.norm(port))
        return ({"value": 1.0 / (P * t_port), "unit": "matvecs/s", "cores": 1, "kind": "port",
                 "sample": f"window 1 of {P} at full N={wl.data.n_rows}, scaled x{P}; {t_port:.2f} s; "
                           "baseline/_ref not installed"}, err)
    plan_s, mv_s, out = ref
    err = float(np.linalg.norm(gpu_window0 - out) / np.linalg.norm(out))
    return ({"value": 1.0 / (P * mv_s), "unit": "matvecs/s", "cores": 1, "kind": "reference",
             "host_cpu_count": os.cpu_count(), "host_affinity": len(os.sched_getaffinity(0)),
             "reference_build_plan_s": plan_s,
             "sample": f"the reference's own fastsum.fast_matvec (baseline/_ref, numba, serial) on window 1 of {P} "
                       f"at full N={wl.data.n_rows}: {mv_s:.2f} s per window product (build_plan {plan_s:.2f} s, "
                       f"excluded), scaled x{P}",
             "port_single_core_s": t_port, "reference_single_core_s": mv_s,
             "note": f"the oracle port runs the same window in {t_port:.2f} s on one core "
                     f"({mv_s / t_port:.2f}x the reference's time); the --impl reference arm runs the port on "
                     "every host thread"}, err)


# ---------------------------------------------------------------------------
# per-kernel rooflines (ak_prof_* device times)


def _kernel_q(name: str) -> int:
    if not name.startswith("k_"):
        return 0       # cuFFT transforms (library)
    if name.startswith(("k_spread3", "k_interp3")):
        return 3
    if name.startswith(("k_spread2", "k_interp2")) or "<2>" in name:
        return 2
    if name.startswith(("k_spread1", "k_interp1")) or "<1>" in name:
        return 1
    return 0


def kernel_rooflines(report: dict, lengths, rows_per_window, R: int, steps: int, peaks: dict) -> dict:
    """Per-kernel achieved rates from KernelTimer totals over `steps` steps.

    Algorithmic work per launch of a q-group (every window of length q, R RHS):
      FLOPs = 2 T^q per point x window x RHS (one FMA per tap)
      bytes = per point x window: 8 q (coordinates) + 8 R (one RHS value read by the
              spread / one output written by the interpolation, per RHS)
    Bound: whichever roof the kernel's arithmetic intensity hits first (ridge = FP64
    peak / HBM peak, ~5.6 FLOP/B): FP64 for q = 3 and for q = 2 with many RHS, HBM for
    q = 1."""
    T = 12
    out = {}
    for name, (cnt, ms) in report.items():
        q = _kernel_q(name)
        if not q or not cnt or ms <= 0:
            continue
        pw = sum(r for L, r in zip(lengths, rows_per_window) if L == q)
        t = ms / cnt * 1e-3                     # seconds per launch
        flops = 2.0 * T ** q * pw * R
        byts = pw * (8.0 * q + 8.0 * R)
        ent = {"launches_per_step": cnt / steps, "ms_per_launch": t * 1e3, "q": q,
               "flops_per_launch": flops, "alg_bytes_per_launch": byts,
               "achieved_tflops": flops / t / 1e12, "achieved_gbs": byts / t / 1e9}
        ridge = peaks["fp64_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
        ent["flop_per_byte"] = flops / byts
        if flops / byts >= ridge:
            ent.update(bound="fp64", frac=ent["achieved_tflops"] / peaks["fp64_tflops"],
                       hbm_frac=ent["achieved_gbs"] / peaks["hbm_gbs"])
        else:
            ent.update(bound="hbm", frac=ent["achieved_gbs"] / peaks["hbm_gbs"],
                       fp64_frac=ent["achieved_tflops"] / peaks["fp64_tflops"])
        out[name] = ent
    return out


def extra_workloads(torch, peaks, steps=5, warmup=2, check=True):
    """Batched-RHS / derivative configurations (BASELINE configs 3 and 5) on one GPU:
    device time per step of the whole product set the config asks for, per-kernel
    times and rooflines, and (check=True, after the timing) full-size parity against
    the oracle: C3 all 8 RHS (K, dK/dl), C5 RHS 0 and 15 (K, all dK/dl_w, dK/ds)."""
    from paper_2404_17344_b200 import _native, configs
    from paper_2404_17344_b200.fastsum import build_mixed_plan, build_plan, fast_matvecs, mixed_matvecs

    out = {}
    for name in ("C3", "C5"):
        wl = configs.CONFIGS[name]()
        t0 = time.perf_counter()
        if wl.mixed:
            plan = build_mixed_plan(wl.specs, wl.window_set, "default", wl.data)
            V = torch.as_tensor(wl.V, device="cuda")
            fn = lambda: mixed_matvecs(plan, V, dell=True, dsigma=True)  # noqa: E731
            n_products = V.shape[0] * (2 + len(wl.window_set))
            what = "K V + dK/dl_w V (per window) + dK/ds V"
        else:
            plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
            V = torch.as_tensor(wl.V, device="cuda")
            fn = lambda: fast_matvecs(plan, V, dell=wl.dell, dsigma=wl.dsigma)  # noqa: E731
            n_products = V.shape[0] * (1 + int(wl.dell) + int(wl.dsigma))
            what = "K V" + (" + dK/dl V" if wl.dell else "") + (" + dK/ds V" if wl.dsigma else "")
        torch.cuda.synchronize()
        plan_s = time.perf_counter() - t0
        for _ in range(warmup):
            fn()
        ms = cuda_time(torch, fn, steps)
        with _native.KernelTimer() as kt:
            for _ in range(2):
                fn()
        R = int(V.shape[0])
        ent = {"N": wl.data.n_rows, "windows": list(wl.window_set.lengths), "rhs": R,
               "products": what, "ms_per_step": ms, "products_per_s": n_products * 1000.0 / ms,
               "plan_build_s": plan_s, "plan": plan.geometries.describe,
               "kernels_ms_per_step": {k: t / 2 for k, (c, t) in kt.report.items()},
               "kernel_roofline": kernel_rooflines(kt.report, wl.window_set.lengths,
                                                   plan.geometries.rows_per_window, R, 2, peaks)}
        if check:
            from oracle.fullsize import config_products, max_rel_rows

            t1 = time.perf_counter()
            if wl.mixed:
                pick = [0, 15]
                res = fn()
                K = res["K"][pick].cpu().numpy()
                dK = res["dK_dell"][:, pick].cpu().numpy()
                dS = res["dK_dsigma"][pick].cpu().numpy()
                del res
                ref = config_products(wl, rhs=pick, dell=True, per_window_dell=True)
                errs = {"K": max_rel_rows(K, ref["K"]),
                        "dK_dell_w": max(max_rel_rows(dK[w], ref["dK_dell"][w]) for w in range(len(wl.window_set))),
                        "dK_dsigma": max_rel_rows(dS, (2.0 / wl.specs[0].sigma_f) * ref["K"])}
                scope = "RHS 0 and 15 at full size: K V, all 10 dK/dl_w V, dK/ds V (sum of single-window oracle plans)"
            else:
                res = fn()
                ref = config_products(wl, dell=True)
                errs = {"K": max_rel_rows(res["K"].cpu().numpy(), ref["K"]),
                        "dK_dell": max_rel_rows(res["dK_dell"].cpu().numpy(), ref["dK_dell"])}
                scope = f"all {R} RHS at full size: K V and dK/dl V"
            ent["rel_err_vs_oracle"] = {"max": max(errs.values()), "per_output": errs, "tolerance": 1e-8,
                                        "scope": scope, "oracle_s": time.perf_counter() - t1}
        out[name] = ent
        del plan, V
        torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            # communicator set-up lines on stderr (ranks, transport: NVLink / NVLS)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2404_17344_b200 import _native, configs
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvec, fast_matvecs
    from paper_2404_17344_b200.windows import WindowSet

    wl = configs.config4(args.n)
    N = wl.data.n_rows
    wins = wl.window_set.windows

    def barrier():
        if world > 1:
            dist.barrier()

    t0 = time.perf_counter()
    dplan = None
    if world > 1:
        from paper_2404_17344_b200.distributed import (CellShardedPlan, HybridShardedPlan, PointShardedPlan,
                                                           WindowShardedPlan)

        cls = {"cell": CellShardedPlan, "hybrid": HybridShardedPlan, "point": PointShardedPlan,
               "window": WindowShardedPlan}[args.shard]
        dplan = cls(wl.spec, wl.window_set, "default", wl.data)
        plan = dplan.plan
    else:
        plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t0

    # the caller's input lives in page-locked host memory (the e2e contract: H2D from
    # pinned host memory); fast_matvec uploads it with one stream-ordered DMA
    v_host = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
    v_host[:] = wl.V[0]
    v_pageable = np.array(wl.V[0])
    v_dev = torch.as_tensor(v_host, device="cuda")

    def step_dev():
        if world > 1:
            return dplan.matvec(v_dev)
        return fast_matvec(plan, v_dev)

    def e2e(vh):
        def step():
            if world > 1:
                out = dplan.matvec(torch.as_tensor(vh).cuda())
                host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
                host.copy_(out, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return host.numpy()
            return fast_matvec(plan, vh)
        return step

    def step_deriv():
        if world > 1:
            fams = ("gauss", "der_gauss")
            if args.shard in ("cell", "window"):
                return dplan.matvecs(v_dev.reshape(1, -1), fams)
            return dplan.matvecs_local(v_dev[dplan.lo:dplan.hi].reshape(1, -1), fams)
        return fast_matvecs(plan, v_dev, dell=True, dsigma=True)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = _native.launch_count()
        e0.record(st)
        for _ in range(steps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        barrier()
        launches = _native.launch_count() - l0
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms / steps, launches

    sampler = ClockSampler(local)
    sampler.start()
    ms_step, launches = timed(step_dev, args.steps, args.warmup)
    clocks = sampler.stop()

    result = {
        "metric": METRIC, "value": 1000.0 / ms_step, "unit": "matvecs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args), "plan": plan.geometries.describe if plan is not None else None,
        "clocks": clocks, "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "plan_build_s": plan_s,
    }
    if dplan is not None:
        result["sharding"] = {"kind": args.shard, "window_groups": getattr(dplan, "G", None),
                              "slabs_or_blocks": getattr(dplan, "Q", None), "rank0_owned_windows":
                              [int(w) + 1 for w in getattr(dplan, "owned", [])]}
        if hasattr(dplan, "stage_times"):
            result["stages_ms_per_step"] = dplan.stage_times(lambda: step_dev(), 5)

    if not args.quick:
        ms_e2e, _ = timed(e2e(v_host), max(3, args.steps // 2), 2)
        ms_e2e_pg, _ = timed(e2e(v_pageable), max(3, args.steps // 2), 2)
        result["e2e"] = {"value": 1000.0 / ms_e2e, "unit": "matvecs/s", "h2d_bytes_per_step": 8 * N,
                         "d2h_bytes_per_step": 8 * N, "ms_per_step": ms_e2e,
                         "api": "fastsum.fast_matvec(plan, numpy v in page-locked memory) -> numpy",
                         "pageable": {"value": 1000.0 / ms_e2e_pg, "ms_per_step": ms_e2e_pg,
                                      "api": "fastsum.fast_matvec(plan, plain numpy v) -> numpy"}}
        ms_d, _ = timed(step_deriv, max(3, args.steps // 2), 2)
        result["deriv"] = {"value": 1000.0 / ms_d, "unit": "(K v, dK/dl v, dK/ds v) triples/s",
                           "ms_per_step": ms_d, "matvecs_per_s": 3000.0 / ms_d}
        if rank == 0:
            peaks_file = ROOT / "MEASURED_PEAKS.json"
            peaks = json.loads(peaks_file.read_text()) if peaks_file.exists() else {"hbm_gbs": 6650.0}
            fp64, dmma = fp64_peak(torch)
            peaks["fp64_tflops"] = fp64
            result["fp64_probe"] = {"dfma_tflops": fp64, "dmma_tflops": dmma}
            if plan is not None and 3 in plan.nufft_plans:
                result["roofline"] = kernel_roofline(torch, plan, wl, peaks)
            if world == 1:
                # per-kernel device times of a step (every rank would have to join the
                # collectives of a sharded step: single GPU only)
                with _native.KernelTimer() as kt:
                    for _ in range(3):
                        step_dev()
                result["kernels_ms_per_step"] = {k: t / 3 for k, (c, t) in kt.report.items()}
            if world == 1:
                result["extras"] = extra_workloads(torch, peaks, check=not args.no_cpu_baseline)
            if world == 1 and not args.no_cpu_baseline:
                from oracle.fullsize import config_products, rel_err

                got = fast_matvec(plan, v_host)
                t1 = time.perf_counter()
                ref = config_products(wl)["K"][0]
                result["rel_err_vs_oracle"] = {"value": rel_err(got, ref), "tolerance": 1e-8,
                                               "scope": "all 10 windows at full N = 1M (oracle/fullsize.py, "
                                                        "every host thread)", "oracle_s": time.perf_counter() - t1}
                one = build_plan(wl.spec, WindowSet(tuple(wins[:1]), d_max=3), "default", wl.data)
                base, err = cpu_baseline(wl, fast_matvec(one, v_host))
                result["cpu_baseline"] = base
                result["rel_err_vs_reference"] = {"value": err, "tolerance": 1e-8,
                                                  "scope": "window 1 at full N against the reference's own "
                                                           "fast_matvec (cpu_baseline run)"}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        ensure_world(args)
        run_ours(args)


if __name__ == "__main__":
    main()
