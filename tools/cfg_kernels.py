"""Per-kernel device time of one step of a BASELINE config (ak_prof_* events around
every launch of the library), plus the step time without the events.

    python tools/cfg_kernels.py C5 [--reps 3] [--tuning cell_items2=8]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_17344_b200 import _native, configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_mixed_plan, build_plan, fast_matvecs, mixed_matvecs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--tuning", default="")
args = ap.parse_args()
tun = {}
for kv in filter(None, args.tuning.split(",")):
    k, v = kv.split("=")
    tun[k] = float(v) if "." in v or "e" in v else int(v)
wl = configs.CONFIGS[args.config](*([args.n] if args.n else []))
if wl.mixed:
    plan = build_mixed_plan(wl.specs, wl.window_set, "default", wl.data, tuning=tun)
    V = torch.as_tensor(wl.V, device="cuda")
    fn = lambda: mixed_matvecs(plan, V, dell=True, dsigma=True)  # noqa: E731
else:
    plan = build_plan(wl.spec, wl.window_set, "default", wl.data, tuning=tun)
    V = torch.as_tensor(wl.V, device="cuda")
    fn = lambda: fast_matvecs(plan, V, dell=wl.dell, dsigma=wl.dsigma)  # noqa: E731
fn()
ms = bench.cuda_time(torch, fn, args.reps)
with _native.KernelTimer() as kt:
    for _ in range(args.reps):
        fn()
per = {k: {"launches_per_step": c / args.reps, "ms_per_step": t / args.reps} for k, (c, t) in kt.report.items()}
print(json.dumps({"config": args.config, "plan": plan.geometries.describe, "tuning": tun, "ms_per_step": ms,
                  "kernels_ms_sum": sum(v["ms_per_step"] for v in per.values()), "kernels": per}, indent=1))
