"""RHS pairs vs cell density: config-4 data at N rows, R = 2 / 8 RHS, K V device time
with the plan's automatic supercell choice and with single-cell items forced
(tuning cell_items3=1, which the RHS-pair tensor-core spread needs).

    python tools/rhs_pair_density.py
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, str(ROOT))
    import torch

    from paper_2404_17344_b200 import configs
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs

    n, R = int(sys.argv[2]), int(sys.argv[3])
    wl = configs.config4(n)
    tun = {"cell_items3": 1} if len(sys.argv) > 4 and sys.argv[4] == "single_cell" else None
    plan = build_plan(wl.spec, wl.window_set, "default", wl.data, tuning=tun)
    import numpy as np

    V = torch.as_tensor(np.random.default_rng(0).normal(size=(R, n)), device="cuda")
    for _ in range(3):
        fast_matvecs(plan, V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fast_matvecs(plan, V)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"ms": e0.elapsed_time(e1) / 10}))
    sys.exit(0)

res = []
for n in (125_000, 250_000, 500_000):
    for R in (2, 8):
        row = {"N": n, "R": R}
        for tag in ("auto", "single_cell"):
            out = subprocess.run([sys.executable, __file__, "--one", str(n), str(R), tag], capture_output=True,
                                 text=True)
            row[tag] = json.loads(out.stdout.strip().splitlines()[-1])["ms"]
        res.append(row)
        print(json.dumps(row), flush=True)
