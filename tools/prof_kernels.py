"""Profiling driver: C4 plan, then a few K v products (spread, FFT, interp kernels).

    python tools/prof_kernels.py [--reps R]
Used under ncu (one GPU); prints nothing performance-relevant itself.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2404_17344_b200 import configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan, fast_matvec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=1_000_000)
args = ap.parse_args()
wl = configs.config4(args.n)
plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
v = torch.as_tensor(wl.V[0], device="cuda")
for _ in range(args.reps):
    out = fast_matvec(plan, v)
torch.cuda.synchronize()
print("ok", float(out.norm()))
