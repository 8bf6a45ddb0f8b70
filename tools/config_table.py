"""Per-config comparison on one box: GPU device time of one step (the products the
config asks for, all RHS) vs the CPU oracle port on every host thread for the same
step (configs 1-3; 4 is bench.py's headline, 5 is too large for the CPU here).

    python tools/config_table.py
"""
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import restate as R  # noqa: E402
from paper_2404_17344_b200 import configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs  # noqa: E402

cores = len(os.sched_getaffinity(0))
pool = ThreadPoolExecutor(cores)
rows = []
for name in ("C1", "C2", "C3"):
    wl = configs.CONFIGS[name]()
    plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
    V = torch.as_tensor(wl.V, device="cuda")
    fast_matvecs(plan, V, dell=wl.dell)
    gpu_ms = bench.cuda_time(torch, lambda: fast_matvecs(plan, V, dell=wl.dell), 20)
    cols = [wl.window_set.columns(w) for w in wl.window_set]
    P = len(cols)
    chunks = max(1, cores // math.gcd(P, cores))
    fams = [wl.spec.family] + (["der_" + wl.spec.family] if wl.dell else [])
    sums = [R.ChunkedFastSum(f, wl.spec.ell, wl.spec.sigma_f, cols, wl.data.features, chunks=chunks) for f in fams]
    t0 = time.perf_counter()
    for fs in sums:
        for r in range(wl.V.shape[0]):
            fs.matvec_pool(wl.V[r], pool)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    rows.append((name, wl.data.n_rows, P, wl.V.shape[0], "+".join(fams), gpu_ms, cpu_ms))

print(f"| config | N | windows | RHS | products | GPU ms/step | CPU oracle ms/step ({cores} threads) | ratio |")
print("|---|---|---|---|---|---|---|---|")
for name, n, p, r, f, g, c in rows:
    print(f"| {name} | {n} | {p} | {r} | {f} | {g:.3f} | {c:.0f} | {c / g:.0f}x |")
