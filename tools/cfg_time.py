"""Device time of one step of configs 2, 3 and 5, CUDA events.

    python tools/cfg_time.py [cell_items2=8,...]   (ak_tuning overrides)
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_17344_b200 import configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_mixed_plan, build_plan, fast_matvecs, mixed_matvecs  # noqa: E402



def timed(fn, reps):
    fn()
    return bench.cuda_time(torch, fn, reps)


tun = {}
for kv in filter(None, (sys.argv[1] if len(sys.argv) > 1 else "").split(",")):
    k, v = kv.split("=")
    tun[k] = float(v) if "." in v or "e" in v else int(v)
out = {"tuning": tun}
for name in ("C2", "C3"):
    wl = configs.CONFIGS[name]()
    plan = build_plan(wl.spec, wl.window_set, "default", wl.data, tuning=tun)
    V = torch.as_tensor(wl.V, device="cuda")
    out[name] = timed(lambda: fast_matvecs(plan, V, dell=True), 10)
wl = configs.config5()
plan = build_mixed_plan(wl.specs, wl.window_set, "default", wl.data, tuning=tun)
V = torch.as_tensor(wl.V, device="cuda")
out["C5"] = timed(lambda: mixed_matvecs(plan, V), 3)
print(json.dumps(out))
