"""Kernel-level timing of the C4 workload: spread / interp alone and the full K v.

    python tools/kbench.py [--n N] [--reps R] [--tuning cell_items3=2,chunk3=256]
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_17344_b200 import configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan, fast_matvec, fast_matvecs  # noqa: E402

def parse_tuning(text):
    """'cell_items3=1,chunk3=256' -> ak_tuning overrides (numbers parsed)."""
    out = {}
    for kv in filter(None, (text or "").split(",")):
        k, v = kv.split("=")
        out[k] = float(v) if "." in v or "e" in v else int(v)
    return out


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--config", default="C4")
ap.add_argument("--tuning", default="", help="ak_tuning overrides, e.g. cell_items3=1,chunk3=256")
args = ap.parse_args()
tun = parse_tuning(args.tuning)
wl = configs.CONFIGS[args.config](args.n) if args.config != "C5" else configs.config5(args.n, 16)
plan = build_plan(wl.spec, wl.window_set, "default", wl.data, tuning=tun)
peaks = {"fp64_tflops": 36.7, "hbm_gbs": 6553.3}
roof = bench.kernel_roofline(torch, plan, wl, peaks, reps=args.reps)
v = torch.as_tensor(wl.V[0], device="cuda")
fast_matvec(plan, v)  # operators + cuFFT plans created outside the timing
fast_matvecs(plan, v, dell=True)
ms = bench.cuda_time(torch, lambda: fast_matvec(plan, v), args.reps)
msd = bench.cuda_time(torch, lambda: fast_matvecs(plan, v, dell=True), args.reps)
print(json.dumps({"tuning": tun, "plan": plan.geometries.describe, "items": plan.geometries.n_items,
                  "spread_ms": roof["spread_ms"], "interp_ms": roof["interp_ms"],
                  "spread_frac": roof["flops_per_launch"] / (roof["spread_ms"] * 1e-3) / 36.7e12,
                  "interp_frac": roof["flops_per_launch"] / (roof["interp_ms"] * 1e-3) / 36.7e12,
                  "matvec_ms": ms, "K+dK_ms": msd}))
